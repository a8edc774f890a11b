// rd_api.cu — the C ABI of librd.so (include/rd.h): validation, host-side level
// tables, device scratch arena, launch sequence K1 -> K2 -> K3, and the pipelined
// host-buffer entry point.
#include <cmath>
#include <cstdio>
#include <cstring>
#include <algorithm>
#include <cstdlib>
#include <tuple>
#include <vector>

#include "rd.h"
#include "rd_internal.cuh"

namespace rd {
size_t k_ridges_smem(int Ks);
int k_ridges_slots(int n_sm);
cudaError_t launch_ridges(const void* frames, int64_t pitch, int64_t fstride, int n_frames, const Params& P,
                          cudaStream_t st);
cudaError_t launch_eigen(const double* abc, int64_t n, double* out, int* deg, cudaStream_t st);
size_t k_hough2_layout(Params& P, int G, int nt, int cb);
bool k_hough2_has_shape(int cb, int G, int nt, int minb);
cudaError_t launch_redo_reset(int n_frames, const Params& P, cudaStream_t st);
cudaError_t launch_hough2(int n_frames, const Params& P, bool wide, int G, int nt, int minb, int cb, int n_sm,
                          cudaStream_t st);
size_t k_fit_smem(const Params& P);
cudaError_t launch_fit(int n_frames, const Params& P, cudaStream_t st);
cudaError_t launch_emit(int n_frames, const Params& P, void* out, int out_cap, int* counts, int* offsets,
                        const int* base_in, int* base_out, int* flags_out, cudaStream_t st);
cudaError_t launch_rays(int n_frames, const Params& P, cudaStream_t st);
cudaError_t launch_members(const Params& P, int f, int write, int* offsets, uint32_t* members, cudaStream_t st);
constexpr int RD_NEV = 5;   // timing events per rd_detect: K1 | K1.5 | K2 | K3
}  // namespace rd

using namespace rd;

static thread_local char g_err[512] = "";

static rd_status cuda_fail(cudaError_t e, const char* where) {
  snprintf(g_err, sizeof g_err, "%s: %s", where, cudaGetErrorString(e));
  return RD_ERR_CUDA;
}
#define CK(call)                                   \
  do {                                             \
    cudaError_t e__ = (call);                      \
    if (e__ != cudaSuccess) return cuda_fail(e__, #call); \
  } while (0)

struct rd_detector {
  rd_config cfg;
  int device;
  int max_batch;
  Params P;
  bool wide;
  int G, k2_threads, k2_minb;   // Hough kernel launch shape (levels per step, threads, CTAs/SM)
  int k2_cb;                    // counter bytes of the main persistent pass (1: + 16-bit redo pass)
  Params P16;                   // redo pass (16-bit counters): its own layout and shape
  int G16, k2_threads16, k2_minb16;
  int n_sm;
  // device allocations
  void* d_tables = nullptr;
  void* d_bins_count = nullptr;
  void* d_bins_xy = nullptr;
  void* d_bins_d = nullptr;
  void* d_peaks = nullptr;
  void* d_ray_d = nullptr;     // K1.5 -> K2 ray lists per Hough tile
  void* d_ray_xy = nullptr;
  void* d_ray_r = nullptr;
  void* d_counters = nullptr;  // stats | peak_count | flags | dbg_count
  size_t counters_bytes = 0;
  void* d_rings_int = nullptr; // K3 output per frame, compacted into the caller's buffer by k_emit
  int* d_need = nullptr;       // [1 + RD_HOST_DEPTH][NEED_N + 1] capacities a call needed, then the
                               // checked-build flag: slot 0 rd_detect, slot 1 + j host call j
  void* d_dbg = nullptr;
  void* d_fpr = nullptr;       // debug: level fingerprints
  int* d_mem_off = nullptr;    // rd_ring_members scratch: offsets (ring_cap + 1)
  uint32_t* d_members = nullptr;
  int64_t members_cap = 0;
  cudaStream_t s_aux = nullptr;   // rd_ring_members / queries
  void* d_redo_list = nullptr;
  void* d_zeros = nullptr;      // zero block the K2 level buffers are cleared from
  // host path: each call in flight (rd_submit_host, at most RD_HOST_DEPTH) has its own mapped
  // pinned staging that the k_emit copies write straight into (only the rings found cross the
  // bus), its chunk cursors and its slot of d_need; the caller's buffers are filled at the wait
  struct HostCall {
    rd_ring* h_stage = nullptr;   // mapped pinned: the call's compacted rings (grown)
    int64_t stage_cap = 0;
    int* h_co = nullptr;          // mapped pinned: counts [n] | offsets [n + 1] | flags [n] (grown)
    int64_t co_cap = 0;
    int* d_cursor = nullptr;      // first output offset of each chunk (chained by k_scan)
    int cursor_cap = 0;
    cudaEvent_t ev_end = nullptr; // the call's work on every stream is done
    rd_ring* h_rings = nullptr;   // the caller's outputs
    int32_t cap = 0;
    int32_t* h_counts = nullptr;
    int32_t* h_offsets = nullptr;
    int n = 0;
  };
  HostCall hcall[RD_HOST_DEPTH];
  int n_pend = 0, pend_head = 0;    // calls in flight, FIFO
  uint64_t chunk_seq = 0;           // host-path chunks enqueued so far: stage and slot rotation
  int chunk = 0;                    // largest chunk of a call with the pipeline empty (ramped up to it)
  int chunk_pipe = 0;               // chunk of a call behind one in flight (stage buffer size)
  int room = 0;                     // frames of the internal buffers per slot: slot b owns [b room, (b+1) room)
  const int* last_co = nullptr;     // counts | offsets | flags of the last completed host call
  int* need_cur = nullptr;          // d_need slot of the last call (rd_query_overflow, check flag)
  cudaStream_t s_join = nullptr;    // joins a call's streams into its end event
  cudaEvent_t ev_start = nullptr, ev_tail[5] = {};
  static constexpr int NSTAGE = 4;   // host-path chunk buffers: copies run up to 3 chunks ahead
  void* d_stage[NSTAGE] = {};
  cudaStream_t s_comp = nullptr, s_h2d = nullptr, s_d2h = nullptr;
  cudaStream_t s_hc[4] = {};        // host path: chunk k computes on s_hc[k % n_slots] (tails overlap)
  static constexpr int NPART = 4;    // frame-view slots: rd_detect parts / host-path chunks
  cudaStream_t s_half[NPART] = {};   // rd_detect: the parts of a large batch
  cudaEvent_t ev_fork = nullptr, ev_join[NPART] = {};
  int n_slots = 1;                  // frame regions of the internal buffers used by concurrent chunks
  cudaEvent_t ev_h2d[NSTAGE], ev_done[NSTAGE], ev_d2h[NSTAGE];
  cudaEvent_t ev_last = nullptr;
  bool timing = false;
  std::vector<cudaEvent_t> tev;  // 4 per timed call
  int n_timed = 0;
  unsigned long long* d_prof = nullptr;
  bool have_last = false;
  bool last_host = false;           // the last call was rd_detect_host (internal buffers hold chunks)
  int last_n = 0;
};

extern "C" {

int32_t rd_abi_version(void) { return RD_ABI_VERSION; }

const char* rd_status_string(rd_status s) {
  switch (s) {
    case RD_OK: return "ok";
    case RD_ERR_PARAM: return "invalid parameter";
    case RD_ERR_DIM: return "unsupported frame dimensions";
    case RD_ERR_CONFIG: return "inconsistent configuration";
    case RD_ERR_CAPACITY: return "device capacity overflow (see rd_query_overflow)";
    case RD_ERR_CUDA: return "CUDA error (see rd_last_error)";
    case RD_ERR_STATE: return "call out of order";
  }
  return "unknown status";
}

const char* rd_last_error(void) { return g_err; }

rd_status rd_config_init(rd_config* c, int32_t width, int32_t height, int32_t pixel) {
  if (!c) return RD_ERR_PARAM;
  memset(c, 0, sizeof *c);
  c->width = width;
  c->height = height;
  c->pixel = pixel;
  c->max_value = pixel == RD_U8 ? 255 : 65535;
  c->smoothing_sigma = 1.5;
  c->curvature_threshold = -10.0;
  c->r_min = 8;
  c->r_max = 70;
  c->vote_threshold_raw = 3;
  c->vote_threshold_norm = 0.5;
  c->sig_a = 1;
  c->sig_b = 5;
  c->sig_den = 20;
  c->annulus_halfwidth = 0;
  c->max_rings_per_frame = 1024;
  c->max_ridges_per_tile = 512;
  c->max_entries_per_tile = 3072;
  c->max_hotspots_per_level = 0;   // automatic (rd_create)
  c->debug = 0;
  return RD_OK;
}

static rd_status validate(const rd_config* c) {
  if (c->width < 8 || c->height < 8 || c->width > 16384 || c->height > 16384) return RD_ERR_DIM;
  if (c->pixel != RD_U8 && c->pixel != RD_U16) return RD_ERR_PARAM;
  if (c->max_value < 1 || c->max_value > (c->pixel == RD_U8 ? 255 : 65535)) return RD_ERR_PARAM;
  // K_s = ceil(3 sigma_s) <= 13: the K1 strip's 16-column halo covers K_s + 3
  if (!(c->smoothing_sigma > 0.0) || !(std::ceil(3.0 * c->smoothing_sigma) <= (double)KS_MAX)) return RD_ERR_PARAM;
  if (c->feature != RD_FEATURE_RIDGE && c->feature != RD_FEATURE_EDGE) return RD_ERR_PARAM;
  if (c->feature == RD_FEATURE_RIDGE && (!(c->curvature_threshold <= 0.0) || !std::isfinite(c->curvature_threshold)))
    return RD_ERR_PARAM;
  if (c->feature == RD_FEATURE_EDGE && (!(c->edge_threshold > 0.0) || !std::isfinite(c->edge_threshold)))
    return RD_ERR_PARAM;
  if (c->r_min < 2 || c->r_max <= c->r_min || c->r_max > 1000) return RD_ERR_PARAM;
  if (c->vote_threshold_raw < 1 || c->vote_threshold_raw > 60000) return RD_ERR_PARAM;
  if (!(c->vote_threshold_norm > 0.0) || !std::isfinite(c->vote_threshold_norm)) return RD_ERR_PARAM;
  if (c->sig_a < 0 || c->sig_den < 1 || (int64_t)c->sig_a * (c->r_min - 1) + c->sig_b <= 0) return RD_ERR_PARAM;
  if (c->annulus_halfwidth < 0) return RD_ERR_PARAM;
  if (c->max_rings_per_frame < 0 || c->max_ridges_per_tile < 0 || c->max_entries_per_tile < 0 ||
      c->max_hotspots_per_level < 0)
    return RD_ERR_PARAM;
  return RD_OK;
}

rd_status rd_create(const rd_config* cin, int32_t max_batch, int32_t device, rd_detector** out) {
  if (!cin || !out || max_batch < 1) return RD_ERR_PARAM;
  *out = nullptr;
  rd_status st = validate(cin);
  if (st != RD_OK) return st;
  rd_config c = *cin;
  if (!c.max_rings_per_frame) c.max_rings_per_frame = 1024;
  if (!c.max_ridges_per_tile) c.max_ridges_per_tile = 512;
  if (!c.max_entries_per_tile) c.max_entries_per_tile = 3072;
  // automatic: cfg3 ridges need < 128 per level per Hough tile; directed edges vote about
  // twice as much (one frame of the 600-frame robustness corpus needs > 160)
  if (!c.max_hotspots_per_level) c.max_hotspots_per_level = c.feature == RD_FEATURE_EDGE ? 256 : 160;
  if (c.max_ridges_per_tile > T1 * T1) c.max_ridges_per_tile = T1 * T1;
  if (c.max_hotspots_per_level > 4095) return RD_ERR_PARAM;   // 12-bit hotspot index in K2 task lists
  if (c.max_entries_per_tile > ENTRY_MAX) c.max_entries_per_tile = ENTRY_MAX;

  // ---- host tables (DESIGN.md §2 A1, A5, A7, A8, A9)
  Params P;
  memset(&P, 0, sizeof P);
  P.W = c.width;
  P.H = c.height;
  P.pixel_bytes = c.pixel == RD_U8 ? 1 : 2;
  const double s = c.smoothing_sigma;
  P.Ks = (int)std::ceil(3.0 * s);
  if (P.Ks > KS_MAX) return RD_ERR_PARAM;
  int64_t sq = 0;
  for (int i = -P.Ks; i <= P.Ks; ++i) {
    P.q[i + P.Ks] = (int)llround(1024.0 * std::exp(-(double)(i * i) / (2.0 * s * s)));
    sq += P.q[i + P.Ks];
  }
  // exactness bounds: int32 row pass, fp64-exact smoothing and Hessian
  if ((int64_t)c.max_value * sq >= (int64_t(1) << 31)) return RD_ERR_CONFIG;
  if ((double)c.max_value * (double)sq * (double)sq * 64.0 >= 9007199254740992.0) return RD_ERR_CONFIG;
  P.t_int = c.curvature_threshold * (64.0 * (double)sq * (double)sq);
  P.feature = c.feature;
  if (c.feature == RD_FEATURE_EDGE && P.Ks > 13) return RD_ERR_CONFIG;   // the streaming K1's 16-column halo
  if (c.feature == RD_FEATURE_EDGE) {   // R19: |grad| of the 5x5 Sobel of G, compared squared in fp64
    if ((double)c.max_value * (double)sq * (double)sq * 96.0 >= 9007199254740992.0) return RD_ERR_CONFIG;
    const double te = c.edge_threshold * (128.0 * (double)sq * (double)sq);
    P.t_edge2 = te * te;
  }
  P.r_min = c.r_min;
  P.r_max = c.r_max;
  P.r_lo = c.r_min - 1;
  P.r_hi = c.r_max + 1;
  P.n_levels = P.r_hi - P.r_lo + 1;
  P.T_raw = c.vote_threshold_raw;
  std::vector<int> lvlK(P.n_levels), lvlAnn(P.n_levels);
  std::vector<double> lvlTn(P.n_levels);
  int Kmax = 0;
  for (int li = 0; li < P.n_levels; ++li) {
    int r = P.r_lo + li;
    int64_t sr = (int64_t)c.sig_a * r + c.sig_b;
    lvlK[li] = (int)((3 * sr + c.sig_den - 1) / c.sig_den);
    Kmax = std::max(Kmax, lvlK[li]);
    lvlTn[li] = ((c.vote_threshold_norm * (2.0 * M_PI)) * 16777216.0) * (double)r;
    if (c.annulus_halfwidth > 0) lvlAnn[li] = c.annulus_halfwidth;
    else lvlAnn[li] = std::max<int>(2, (int)((2 * sr + c.sig_den - 1) / c.sig_den));
  }
  if (Kmax > 48) return RD_ERR_CONFIG;  // raw tile halo bound (shared memory)
  P.K_max = Kmax;
  // K_r = ceil(3 (a r + b) / den) <= (3a/den) r + 3b/den + 1 (+ margin): ray-interval bound in K2
  P.k_slope = (float)(3.0 * c.sig_a / c.sig_den) * 1.0001f + 1e-6f;
  P.k_icpt = (float)(3.0 * c.sig_b / c.sig_den + 1.0) + 0.01f;
  P.hal = Kmax + 1;
  P.wstride = Kmax + 1;
  // K2 dp4a weight words per window row (table below), rounded up to odd: the kernel reads 3, 5, 7
  // or 9 words of a row, the least that holds the step's widest window, and relies on zero words
  // up to that count
  P.wp_nw = ((2 * Kmax + 1 + 3 + 3) / 4) | 1;
  std::vector<int> lvlW((size_t)P.n_levels * P.wstride, 0);
  double max_wsum = 0;
  for (int li = 0; li < P.n_levels; ++li) {
    int r = P.r_lo + li;
    int64_t sr = (int64_t)c.sig_a * r + c.sig_b;
    double den = 2.0 * (double)(sr * sr);
    double wsum = 0;
    for (int d = 0; d <= lvlK[li]; ++d) {
      double num = (double)((int64_t)d * d * c.sig_den * c.sig_den);
      int w = (int)llround(4096.0 * std::exp(-num / den));
      lvlW[(size_t)li * P.wstride + d] = w;
      wsum += (d ? 2.0 : 1.0) * w;
    }
    max_wsum = std::max(max_wsum, wsum);
  }
  bool wide = 65535.0 * max_wsum >= 4294967296.0;

  rd_detector* det = new rd_detector();
  det->cfg = c;
  det->device = device;
  det->max_batch = max_batch;
  det->wide = wide;
  cudaError_t e = cudaSetDevice(device);
  if (e != cudaSuccess) { delete det; return cuda_fail(e, "cudaSetDevice"); }

  P.nbx = (c.width + T1 - 1) / T1;
  P.nby = (c.height + T1 - 1) / T1;
  P.ridge_cap = c.max_ridges_per_tile;
  P.entry_cap = c.max_entries_per_tile;
  P.hot_cap = c.max_hotspots_per_level;
  P.ring_cap = c.max_rings_per_frame;
  P.debug = c.debug;
  P.dbg_cap = c.debug ? (1 << 20) : 0;

  cudaDeviceProp prop;
  e = cudaGetDeviceProperties(&prop, device);
  if (e != cudaSuccess) { delete det; return cuda_fail(e, "cudaGetDeviceProperties"); }
  const size_t smax = prop.sharedMemPerBlockOptin, sm_sm = prop.sharedMemPerMultiprocessor;
  struct Shape { int T, G, nt, minb; };
  det->G = 0;
  det->n_sm = prop.multiProcessorCount;
  {
    // persistent K2: the first (T, G, threads, CTAs/SM) candidate whose layout fits with at
    // least 256 resident rays per tile, then as many resident rays as fit (up to entry_cap).
    // The 16-bit redo pass must use the main pass's tile side (K1.5 routes rays per tile).
    // RD_K2_SHAPE2="G,threads,ctas" or "T,G,threads,ctas" puts a shape first;
    // RD_K2_CB=2 forces 16-bit counters.
    // Tiles: for a shape's side T, the rectangular tiling of the frame (nx x ny tiles of
    // ceil(W/nx) x ceil(H/ny)) whose raw buffers are no larger than T's square one and that
    // minimises buffer cells (votes, clears) plus a per-tile cost: cfg3 gets 8 x 8 tiles of
    // 128 x 86 instead of 10 x 7 of 104 x 104 (the last row and column only partly used).
    auto tilings = [&](int T) {
      const long long hh = 2LL * P.hal;
      double slack = 1.3;   // raw buffers up to 30 % larger than T's square (fewer resident rays)
      if (const char* env = getenv("RD_K2_TSLACK")) slack = atof(env);
      const double budget = slack * (double)((T + hh) * (T + hh));
      std::vector<std::tuple<double, int, int>> cand;
      for (int nx = 1; nx <= c.width; ++nx) {
        const int TX = (c.width + nx - 1) / nx;
        if (TX > 254) continue;
        if (TX < std::max(16, T / 2)) break;   // no slivers (K1.5 windows grow as 1 / side)
        for (int ny = 1; ny <= c.height; ++ny) {
          const int TY = (c.height + ny - 1) / ny;
          if (TY > 254) continue;
          if (TY < std::max(16, T / 2)) break;
          if ((double)((TX + hh) * (TY + hh)) > budget) continue;
          // buffer cells (votes, clears) plus a per-tile cost of 8000 cells (17 barrier-separated
          // steps, the ray load): fitted to cfg3's measured 64, 63, 60, 56, 54-tile tilings
          cand.emplace_back((double)nx * ny * ((double)(TX + hh) * (TY + hh) + 8000.0), TX, TY);
          break;   // larger ny only adds tiles
        }
      }
      std::sort(cand.begin(), cand.end());
      return cand;
    };
    // 2-byte level intervals, all resident (Params::k2_rr16) when the levels fit a byte
    P.k2_rr16 = P.n_levels <= 255 && P.entry_cap % 8 == 0 ? 1 : 0;
    if (const char* env = getenv("RD_K2_RR16")) P.k2_rr16 = P.k2_rr16 && atoi(env) != 0;
    int rmin = 256;   // resident rays a shape must hold (RD_K2_RMIN for A/B)
    if (const char* env = getenv("RD_K2_RMIN")) rmin = std::max(32, atoi(env));
    auto pick = [&](Params& Q, int cb, int& G, int& nt, int& minb, int forceT, int forceTY) {
      std::vector<Shape> sh = cb == 1 ? std::vector<Shape>{{104, 4, 512, 2}, {96, 4, 512, 2}, {64, 4, 256, 3}, {64, 4, 384, 2},
                                                           {64, 8, 512, 1}}
                                      : std::vector<Shape>{{64, 4, 384, 2}, {64, 4, 512, 2}, {64, 8, 512, 1},
                                                           {64, 4, 512, 1}};
      if (const char* env = getenv("RD_K2_SHAPE2")) {   // "G,threads,ctas" or "T,G,threads,ctas"
        Shape s{64, 0, 0, 0};
        const int n = sscanf(env, "%d,%d,%d,%d", &s.T, &s.G, &s.nt, &s.minb);
        if (n == 3) s = Shape{64, s.T, s.G, s.nt};
        if ((n == 3 || n == 4) && s.T >= 32 && s.T <= 128 && k_hough2_has_shape(cb, s.G, s.nt, s.minb))
          sh.insert(sh.begin(), s);
      }
      G = 0;
      for (const Shape& s : sh) {
        if (!k_hough2_has_shape(cb, s.G, s.nt, s.minb)) continue;
        if (cb == 1 && Q.wstride - 1 > 15) break;   // byte-counter windows: 2K + 1 <= 31 rows per half-warp
        if (forceT) {
          Q.k2t = forceT;
          Q.k2ty = forceTY;
        } else if (getenv("RD_K2_SQUARE")) {   // square tiles of side T (A/B)
          Q.k2t = Q.k2ty = s.T;
        } else if (getenv("RD_K2_TILE") &&   // "TX,TY" (A/B)
                   sscanf(getenv("RD_K2_TILE"), "%d,%d", &Q.k2t, &Q.k2ty) == 2 && Q.k2t >= 16 &&
                   Q.k2t <= 254 && Q.k2ty >= 16 && Q.k2ty <= 254) {
        } else {   // the cheapest tiling whose layout fits this shape with 256 resident rays
          Q.k2t = Q.k2ty = s.T;
          Q.k2_rcap = Q.k2_rr16 ? 0 : rmin;
          const size_t lim = s.minb == 1 ? smax : std::min(smax, sm_sm / s.minb - 1024);
          for (const auto& t : tilings(s.T)) {
            Q.k2t = std::get<1>(t);
            Q.k2ty = std::get<2>(t);
            Params Q16 = Q;   // the 16-bit redo pass must fit the same tiles (one CTA per SM)
            const bool redo_fits = cb == 2 || k_hough2_layout(Q16, 4, 512, 2) <= smax;
            if (redo_fits && k_hough2_layout(Q, s.G, s.nt, cb) <= lim) break;
            Q.k2t = Q.k2ty = s.T;
          }
        }
        const size_t limit = s.minb == 1 ? smax : std::min(smax, sm_sm / s.minb - 1024);
        Q.k2_rcap = Q.k2_rr16 ? 0 : rmin;
        if (k_hough2_layout(Q, s.G, s.nt, cb) > limit) continue;
        while (!Q.k2_rr16 && Q.k2_rcap < Q.entry_cap) {   // as many resident rays as fit
          Q.k2_rcap += 64;
          if (k_hough2_layout(Q, s.G, s.nt, cb) > limit) {
            Q.k2_rcap -= 64;
            break;
          }
        }
        Q.k2_rcap = std::min(Q.k2_rcap, Q.entry_cap);
        if (Q.k2_rcap >= 4) Q.k2_rcap &= ~3;   // whole 16-byte lines of 4-byte ray fields (K2 bulk copies)
        k_hough2_layout(Q, s.G, s.nt, cb);
        G = s.G;
        nt = s.nt;
        minb = s.minb;
        return;
      }
    };
    det->k2_cb = 1;
    if (const char* env = getenv("RD_K2_CB")) det->k2_cb = atoi(env) == 2 ? 2 : 1;
    if (det->k2_cb == 1) pick(P, 1, det->G, det->k2_threads, det->k2_minb, 0, 0);
    det->P16 = P;
    pick(det->P16, 2, det->G16, det->k2_threads16, det->k2_minb16, det->G ? P.k2t : 0, det->G ? P.k2ty : 0);
    if (det->G == 0 && det->G16 != 0) {   // 16-bit counters as the only pass
      det->k2_cb = 2;
      P.k2t = det->P16.k2t;
      P.k2ty = det->P16.k2ty;
      P.k2_rcap = det->P16.k2_rcap;
      P.k2o = det->P16.k2o;
      det->G = det->G16;
      det->k2_threads = det->k2_threads16;
      det->k2_minb = det->k2_minb16;
    }
    if (det->k2_cb == 1 && det->G16 == 0) det->G = 0;   // no 16-bit redo shape: not exact, do not use
  }
  if (getenv("RD_K2_VERBOSE"))
    fprintf(stderr, "rd: K2 tiles %dx%d cb %d G %d threads %d ctas/SM %d smem %d rcap %d | redo G %d threads %d "
            "ctas/SM %d smem %d rcap %d\n", P.k2t, P.k2ty, det->k2_cb, det->G, det->k2_threads, det->k2_minb,
            P.k2o.total, P.k2_rcap, det->G16,
            det->k2_threads16, det->k2_minb16, det->P16.k2o.total, det->P16.k2_rcap);
  P.ntx = (c.width + P.k2t - 1) / P.k2t;
  P.nty = (c.height + P.k2ty - 1) / P.k2ty;
  {   // K1.5 tests a bin's rays against a window of at most 64 Hough tiles
    const int reach = P.r_hi + P.hal + 1, wspan = (2 * reach + T1) / std::min(P.k2t, P.k2ty) + 2;
    if (wspan * wspan > 64) {
      delete det;
      snprintf(g_err, sizeof g_err, "search radius %d too large for the %d-px Hough tiles", c.r_max, P.k2t);
      return RD_ERR_CONFIG;
    }
  }
  if (k_ridges_smem(P.Ks) > smax || det->G == 0 || k_fit_smem(P) > smax) {
    snprintf(g_err, sizeof g_err, "shared memory: K1 %zu K3 %zu (limit %zu); K2 %s", k_ridges_smem(P.Ks),
             k_fit_smem(P), smax, det->G ? "fits" : "no persistent shape fits (halo K_max + 1 or capacities too large)");
    delete det;
    return RD_ERR_CONFIG;
  }

  const int64_t B = max_batch, nbins = (int64_t)P.nbx * P.nby;
  // byte-plane weight words for K2's dp4a window rows (byte counters): for level li, row start
  // alignment a = (segment start) mod 4 and word k, byte b is the weight of segment cell
  // o = 4k + b - a (0 outside [0, 2K]); w = 64 wh + wl with wl < 64, wh <= 64 (both bytes)
  std::vector<uint32_t> lvlWP((size_t)P.n_levels * 4 * P.wp_nw * 2, 0);
  for (int li = 0; li < P.n_levels; ++li)
    for (int a = 0; a < 4; ++a)
      for (int k = 0; k < P.wp_nw; ++k) {
        uint32_t lo = 0, hi = 0;
        for (int b = 0; b < 4; ++b) {
          const int o = 4 * k + b - a, K = lvlK[li];
          if (o < 0 || o > 2 * K) continue;
          const int w = lvlW[(size_t)li * P.wstride + std::abs(o - K)];
          lo |= (uint32_t)(w & 63) << (8 * b);
          hi |= (uint32_t)(w >> 6) << (8 * b);
        }
        const size_t base = (((size_t)li * 4 + a) * P.wp_nw + k) * 2;
        lvlWP[base] = lo;
        lvlWP[base + 1] = hi;
      }
  size_t tb = sizeof(int) * P.n_levels * 2 + sizeof(double) * P.n_levels + sizeof(int) * lvlW.size() +
              sizeof(uint32_t) * lvlWP.size() + 64;
#define ALLOC(ptr, bytes)                                          \
  do {                                                             \
    e = cudaMalloc(&(ptr), (bytes));                               \
    if (e != cudaSuccess) { rd_destroy(det); return cuda_fail(e, "cudaMalloc " #ptr); } \
  } while (0)
  ALLOC(det->d_tables, tb);
  ALLOC(det->d_bins_count, sizeof(int) * B * nbins);
  ALLOC(det->d_bins_xy, sizeof(uint32_t) * B * nbins * P.ridge_cap);
  ALLOC(det->d_bins_d, sizeof(double2) * B * nbins * P.ridge_cap);
  ALLOC(det->d_peaks, sizeof(Peak) * B * P.ring_cap);
  const int64_t ntl = (int64_t)P.ntx * P.nty;
  ALLOC(det->d_ray_d, sizeof(double2) * B * ntl * P.entry_cap);
  ALLOC(det->d_ray_xy, sizeof(uint32_t) * B * ntl * P.entry_cap);
  ALLOC(det->d_ray_r, sizeof(uint32_t) * B * ntl * P.entry_cap);
  det->counters_bytes = sizeof(Stats) * B + sizeof(int) * 3 * B + sizeof(int) * B * ntl + 8 * rd_detector::NPART +
                        sizeof(int) * B + sizeof(int) * B;
  ALLOC(det->d_counters, det->counters_bytes);
  ALLOC(det->d_rings_int, sizeof(Ring) * B * P.ring_cap);
  ALLOC(det->d_need, sizeof(int) * (1 + RD_HOST_DEPTH) * (NEED_N + 1));
  ALLOC(det->d_mem_off, sizeof(int) * (P.ring_cap + 1));
  {   // zeros the Hough kernel's level buffers are cleared from (bulk copies, K2 phase 3)
    const size_t zb = (size_t)std::max(P.k2o.total, det->P16.k2o.total);
    ALLOC(det->d_zeros, zb);
    e = cudaMemset(det->d_zeros, 0, zb);
    if (e != cudaSuccess) { rd_destroy(det); return cuda_fail(e, "cudaMemset zeros"); }
    P.zeros = det->d_zeros;
  }
  if (c.debug) {
    ALLOC(det->d_dbg, sizeof(HotRec) * B * P.dbg_cap);
    ALLOC(det->d_fpr, sizeof(unsigned long long) * 3 * B * P.n_levels);
  }
  // tables
  {
    std::vector<unsigned char> h(tb, 0);
    size_t o = 0;
    memcpy(h.data() + o, lvlTn.data(), sizeof(double) * P.n_levels);
    P.lvlTn = reinterpret_cast<const double*>((char*)det->d_tables + o);
    o += sizeof(double) * P.n_levels;
    memcpy(h.data() + o, lvlK.data(), sizeof(int) * P.n_levels);
    P.lvlK = reinterpret_cast<const int*>((char*)det->d_tables + o);
    o += sizeof(int) * P.n_levels;
    memcpy(h.data() + o, lvlAnn.data(), sizeof(int) * P.n_levels);
    P.lvlAnn = reinterpret_cast<const int*>((char*)det->d_tables + o);
    o += sizeof(int) * P.n_levels;
    memcpy(h.data() + o, lvlW.data(), sizeof(int) * lvlW.size());
    P.lvlW = reinterpret_cast<const int*>((char*)det->d_tables + o);
    o += sizeof(int) * lvlW.size();
    o = (o + 15) & ~size_t(15);
    memcpy(h.data() + o, lvlWP.data(), sizeof(uint32_t) * lvlWP.size());
    P.lvlWP = reinterpret_cast<const uint32_t*>((char*)det->d_tables + o);
    e = cudaMemcpy(det->d_tables, h.data(), tb, cudaMemcpyHostToDevice);
    if (e != cudaSuccess) { rd_destroy(det); return cuda_fail(e, "cudaMemcpy tables"); }
  }
  P.bin_count = (int*)det->d_bins_count;
  P.bin_xy = (uint32_t*)det->d_bins_xy;
  P.bin_d = (double2*)det->d_bins_d;
  P.peaks = (Peak*)det->d_peaks;
  P.stats = (Stats*)det->d_counters;
  P.peak_count = (int*)((char*)det->d_counters + sizeof(Stats) * B);
  P.flags = P.peak_count + B;
  P.dbg_count = P.flags + B;
  P.ray_count = P.dbg_count + B;
  P.k2_work = P.ray_count + B * ntl;
  P.redo = P.k2_work + 2 * rd_detector::NPART;
  P.need_ridges = P.redo + B;
  P.redo_list = nullptr;
  P.rings = (Ring*)det->d_rings_int;
  P.need = det->d_need;
  P.check = det->d_need + NEED_N;   // zeroed with the needs at every call
#ifdef RD_CHECKED
  P.jitter = getenv("RD_JITTER") ? 1 : 0;
#endif
  P.dbg_fpr = (unsigned long long*)det->d_fpr;
  P.n_sm = det->n_sm;
  P.k1_slots = k_ridges_slots(det->n_sm);
  P.force_redo = getenv("RD_K2_FORCE_REDO") ? 1 : 0;
  P.k2_ctas_per_sm = getenv("RD_K2_CTAS") ? atoi(getenv("RD_K2_CTAS")) : 0;
  P.u8_limit = 255;
  P.ablate = getenv("RD_K2_ABLATE") ? atoi(getenv("RD_K2_ABLATE")) : 0;
  if (const char* env = getenv("RD_K2_U8_LIMIT")) P.u8_limit = std::max(1, std::min(255, atoi(env)));
  P.ray_d = (double2*)det->d_ray_d;
  P.ray_xy = (uint32_t*)det->d_ray_xy;
  P.ray_r = (uint32_t*)det->d_ray_r;
  P.dbg_hot = (HotRec*)det->d_dbg;
  det->P = P;
  {   // the redo pass: same buffers, its own layout, shape and the redo list
    Params Q = P;
    Q.k2t = det->P16.k2t;
    Q.k2ty = det->P16.k2ty;
    Q.k2_rcap = det->P16.k2_rcap;
    Q.k2o = det->P16.k2o;
    e = cudaMalloc(&det->d_redo_list, sizeof(int) * rd_detector::NPART * (B + 1));   // one list per slot
    if (e != cudaSuccess) { rd_destroy(det); return cuda_fail(e, "cudaMalloc redo_list"); }
    Q.redo_list = (int*)det->d_redo_list;
    det->P16 = Q;
  }
  e = cudaEventCreateWithFlags(&det->ev_last, cudaEventDisableTiming);
  if (e != cudaSuccess) { rd_destroy(det); return cuda_fail(e, "cudaEventCreate"); }
  e = cudaStreamCreateWithFlags(&det->s_aux, cudaStreamNonBlocking);
  if (e != cudaSuccess) { rd_destroy(det); return cuda_fail(e, "cudaStreamCreate"); }
  *out = det;
  return RD_OK;
}

rd_status rd_destroy(rd_detector* det) {
  if (!det) return RD_OK;
  cudaSetDevice(det->device);
  cudaFree(det->d_tables);
  cudaFree(det->d_bins_count);
  cudaFree(det->d_bins_xy);
  cudaFree(det->d_bins_d);
  cudaFree(det->d_peaks);
  cudaFree(det->d_ray_d);
  cudaFree(det->d_ray_xy);
  cudaFree(det->d_ray_r);
  if (det->ev_last) cudaEventSynchronize(det->ev_last);
  if (det->s_aux) cudaStreamSynchronize(det->s_aux);
  cudaFree(det->d_counters);
  cudaFree(det->d_rings_int);
  cudaFree(det->d_need);
  cudaFree(det->d_mem_off);
  cudaFree(det->d_members);
  cudaFree(det->d_fpr);
  for (auto& c : det->hcall) {
    cudaFreeHost(c.h_stage);
    cudaFreeHost(c.h_co);
    cudaFree(c.d_cursor);
    if (c.ev_end) cudaEventDestroy(c.ev_end);
  }
  if (det->s_aux) cudaStreamDestroy(det->s_aux);
  cudaFree(det->d_dbg);
  cudaFree(det->d_redo_list);
  cudaFree(det->d_zeros);
  cudaFree(det->d_prof);
  for (int i = 0; i < rd_detector::NSTAGE; ++i) {
    cudaFree(det->d_stage[i]);
  }
  if (det->s_comp) {
    cudaStreamDestroy(det->s_comp);
    for (int i = 1; i < 4; ++i)
      if (det->s_hc[i]) cudaStreamDestroy(det->s_hc[i]);
    cudaStreamDestroy(det->s_h2d);
    cudaStreamDestroy(det->s_d2h);
    cudaStreamDestroy(det->s_join);
    cudaEventDestroy(det->ev_start);
    for (cudaEvent_t e : det->ev_tail) cudaEventDestroy(e);
    for (int i = 0; i < rd_detector::NSTAGE; ++i) {
      cudaEventDestroy(det->ev_h2d[i]);
      cudaEventDestroy(det->ev_done[i]);
      cudaEventDestroy(det->ev_d2h[i]);
    }
  }
  if (det->ev_last) cudaEventDestroy(det->ev_last);
  for (int i = 0; i < rd_detector::NPART; ++i) {
    if (det->s_half[i]) cudaStreamDestroy(det->s_half[i]);
    if (det->ev_join[i]) cudaEventDestroy(det->ev_join[i]);
  }
  if (det->ev_fork) cudaEventDestroy(det->ev_fork);
  for (cudaEvent_t e : det->tev) cudaEventDestroy(e);
  delete det;
  return RD_OK;
}

// The parameters of a call working on frames [f0, f0 + n) of the internal buffers, with the
// K2 work counters and redo list of slot `slot` (0 or 1): two such views are disjoint, so the
// host path can run consecutive chunks on two streams and let their kernels overlap.
static void frame_view(const rd_detector* det, int f0, int slot, Params& V, Params& V16, int* need = nullptr) {
  const Params& P = det->P;
  const int64_t nb = (int64_t)P.nbx * P.nby, ntl = (int64_t)P.ntx * P.nty;
  V = P;
  if (need) {   // the d_need slot of a host-path call
    V.need = need;
    V.check = need + NEED_N;
  }
  V.bin_count += f0 * nb;
  V.bin_xy += f0 * nb * P.ridge_cap;
  V.bin_d += f0 * nb * P.ridge_cap;
  V.peaks += (int64_t)f0 * P.ring_cap;
  V.rings += (int64_t)f0 * P.ring_cap;
  V.stats += f0;
  V.peak_count += f0;
  V.flags += f0;
  V.dbg_count += f0;
  V.ray_count += f0 * ntl;
  V.ray_d += f0 * ntl * P.entry_cap;
  V.ray_xy += f0 * ntl * P.entry_cap;
  V.ray_r += f0 * ntl * P.entry_cap;
  if (V.dbg_hot) V.dbg_hot += (int64_t)f0 * P.dbg_cap;
  if (V.dbg_fpr) V.dbg_fpr += (int64_t)f0 * 3 * P.n_levels;
  V.redo += f0;
  V.need_ridges += f0;
  V.k2_work = P.k2_work + 2 * slot;   // [main, redo] work counters of the slot
  V16 = V;
  V16.k2t = det->P16.k2t;
  V16.k2ty = det->P16.k2ty;
  V16.k2_rcap = det->P16.k2_rcap;
  V16.k2o = det->P16.k2o;
  V16.redo_list = det->P16.redo_list + (int64_t)slot * (det->max_batch + 1);   // slot < NPART
}

// K1 -> K1.5 -> K2 (+ 16-bit redo) -> K3 on frames [f0, f0 + n) of the internal buffers (frame
// view of slot `slot`); K3's rings stay in the per-frame scratch until k_emit.
static rd_status detect_impl(rd_detector* det, const void* d_frames, int64_t pitch, int64_t fstride, int n,
                             cudaStream_t st, int f0 = 0, int slot = 0, int parts = 1, int* need = nullptr) {
  Params P, P16;
  frame_view(det, f0, slot, P, P16, need);
  P.parts = P16.parts = parts;
  cudaEvent_t* ev = nullptr;
  if (det->timing) {
    size_t need = RD_NEV * (size_t)(det->n_timed + 1);
    while (det->tev.size() < need) {
      cudaEvent_t e;
      CK(cudaEventCreate(&e));
      det->tev.push_back(e);
    }
    ev = &det->tev[RD_NEV * (size_t)det->n_timed];
    det->n_timed++;
  }
  // per-frame counters of the view and the slot's work counters
  const int64_t ntl = (int64_t)P.ntx * P.nty;
  if (f0 == 0 && slot == 0 && n == det->max_batch) {
    CK(cudaMemsetAsync(det->d_counters, 0, det->counters_bytes, st));
  } else {
    CK(cudaMemsetAsync(P.stats, 0, sizeof(Stats) * n, st));
    CK(cudaMemsetAsync(P.peak_count, 0, sizeof(int) * n, st));
    CK(cudaMemsetAsync(P.flags, 0, sizeof(int) * n, st));
    CK(cudaMemsetAsync(P.dbg_count, 0, sizeof(int) * n, st));
    CK(cudaMemsetAsync(P.ray_count, 0, sizeof(int) * n * ntl, st));
    CK(cudaMemsetAsync(P.k2_work, 0, sizeof(int) * 2, st));
    CK(cudaMemsetAsync(P.redo, 0, sizeof(int) * n, st));
    CK(cudaMemsetAsync(P.need_ridges, 0, sizeof(int) * n, st));
  }
  if (P.dbg_fpr) CK(cudaMemsetAsync(P.dbg_fpr, 0, sizeof(unsigned long long) * 3 * P.n_levels * n, st));
  if (ev) CK(cudaEventRecord(ev[0], st));
  CK(launch_ridges(d_frames, pitch, fstride, n, P, st));
  if (ev) CK(cudaEventRecord(ev[1], st));
  CK(launch_rays(n, P, st));
  if (ev) CK(cudaEventRecord(ev[2], st));
  CK(launch_hough2(n, P, det->wide, det->G, det->k2_threads, det->k2_minb, det->k2_cb, det->n_sm, st));
  if (det->k2_cb == 1) {   // frames whose byte counters overflowed: recomputed with 16-bit counters
    CK(launch_redo_reset(n, P16, st));
    CK(launch_hough2(n, P16, det->wide, det->G16, det->k2_threads16, det->k2_minb16, 2, det->n_sm, st));
  }
  if (ev) CK(cudaEventRecord(ev[3], st));
  CK(launch_fit(n, P, st));
  return RD_OK;
}

static rd_status check_frames(rd_detector* det, const void* frames, int64_t pitch, int64_t fstride, int n) {
  if (!det || !frames) return RD_ERR_PARAM;
  const int pb = det->P.pixel_bytes;
  if (pitch < (int64_t)det->cfg.width * pb || (pitch % pb)) return RD_ERR_PARAM;
  if (n > 1 && fstride < pitch * det->cfg.height) return RD_ERR_PARAM;
  if (((uintptr_t)frames % pb) || (fstride % pb)) return RD_ERR_PARAM;
  return RD_OK;
}

rd_status rd_detect(rd_detector* det, const void* d_frames, int64_t pitch, int64_t fstride, int32_t n,
                    rd_ring* d_rings, int32_t ring_cap_total, int32_t* d_counts, int32_t* d_offsets, void* stream) {
  if (!det || n < 1 || n > det->max_batch || !d_counts || !d_offsets || ring_cap_total < 0 ||
      (ring_cap_total > 0 && !d_rings) || ((uintptr_t)d_rings % 16))
    return RD_ERR_PARAM;
  rd_status s = check_frames(det, d_frames, pitch, fstride, n);
  if (s != RD_OK) return s;
  CK(cudaSetDevice(det->device));
  if (det->n_pend) return RD_ERR_STATE;   // host-path calls in flight
  cudaStream_t st = (cudaStream_t)stream;
  if (det->have_last) CK(cudaStreamWaitEvent(st, det->ev_last, 0));   // the previous call's scratch
  det->have_last = false;
  det->need_cur = det->d_need;
  CK(cudaMemsetAsync(det->d_need, 0, sizeof(int) * (NEED_N + 1), st));
  // A large batch runs as two or three parts on internal streams (disjoint frame views of the
  // internal buffers), joined back into the caller's stream: each kernel's last partial
  // wave overlaps the other parts' kernels.  Per-kernel timing keeps one stream.
  int parts = n >= 192 ? 3 : n >= 128 ? 2 : 1;   // cfg3, 256 frames: 39.2 k frames/s at 3 parts, 38.7 k at 2, 38.1 k at 1
  if (const char* env = getenv("RD_SPLIT")) parts = std::max(1, std::min(rd_detector::NPART, atoi(env)));
  if (det->timing || n < 2 * parts) parts = 1;
  if (parts > 1) {
    if (!det->s_half[0]) {
      for (int i = 0; i < rd_detector::NPART; ++i) {
        CK(cudaStreamCreateWithFlags(&det->s_half[i], cudaStreamNonBlocking));
        CK(cudaEventCreateWithFlags(&det->ev_join[i], cudaEventDisableTiming));
      }
      CK(cudaEventCreateWithFlags(&det->ev_fork, cudaEventDisableTiming));
    }
    CK(cudaEventRecord(det->ev_fork, st));
    for (int i = 0; i < parts; ++i) {
      const int f0 = (int)((int64_t)n * i / parts), f1 = (int)((int64_t)n * (i + 1) / parts);
      CK(cudaStreamWaitEvent(det->s_half[i], det->ev_fork, 0));
      s = detect_impl(det, (const char*)d_frames + (size_t)f0 * fstride, pitch, fstride, f1 - f0, det->s_half[i],
                      f0, i, parts);
      if (s != RD_OK) return s;
      CK(cudaEventRecord(det->ev_join[i], det->s_half[i]));
      CK(cudaStreamWaitEvent(st, det->ev_join[i], 0));
    }
  } else {
    s = detect_impl(det, d_frames, pitch, fstride, n, st);
    if (s != RD_OK) return s;
  }
  // A11: counts, offsets and the compacted rings of all n frames
  CK(launch_emit(n, det->P, d_rings, ring_cap_total, d_counts, d_offsets, nullptr, nullptr, nullptr, st));
  if (det->timing) CK(cudaEventRecord(det->tev[RD_NEV * (size_t)(det->n_timed - 1) + RD_NEV - 1], st));
  CK(cudaEventRecord(det->ev_last, st));
  det->have_last = true;
  det->last_host = false;
  det->last_n = n;
  return RD_OK;
}

static rd_status ensure_host_path(rd_detector* det) {
  if (det->s_comp) return RD_OK;
  // two chunks in flight use disjoint halves of the internal buffers (frame_view)
  int slots = 2;
  if (const char* env = getenv("RD_HOST_SLOTS")) slots = std::max(1, std::min(4, atoi(env)));
  det->n_slots = std::max(1, std::min(slots, det->max_batch));
  const int room = det->max_batch / det->n_slots;
  det->room = room;
  const size_t fbytes = (size_t)det->cfg.width * det->cfg.height * det->P.pixel_bytes;
  // a call behind one in flight overlaps its copies with that call's detection, so its chunks
  // can be large (96 frames or 256 MB: cfg3 e2e 33.5 k frames/s against 31.8 k at 48, 32.7 k at
  // 64, 33.2 k at 128); a call into an empty pipeline ramps its chunks up to 48 frames (its fill
  // and drain are not overlapped)
  det->chunk_pipe = std::max(1, std::min({room, 96, (int)std::max<size_t>(1, (256u << 20) / fbytes)}));
  det->chunk = std::min(det->chunk_pipe, 48);
  if (const char* env = getenv("RD_HOST_CHUNK")) det->chunk = std::max(1, std::min(room, atoi(env)));
  if (const char* env = getenv("RD_HOST_CHUNK_PIPE")) det->chunk_pipe = std::max(1, std::min(room, atoi(env)));
  const int cmax = std::max(det->chunk, det->chunk_pipe);
  for (int i = 0; i < rd_detector::NSTAGE; ++i) {
    CK(cudaMalloc(&det->d_stage[i], fbytes * cmax));
    CK(cudaEventCreateWithFlags(&det->ev_h2d[i], cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&det->ev_done[i], cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&det->ev_d2h[i], cudaEventDisableTiming));
  }
  for (auto& c : det->hcall) CK(cudaEventCreateWithFlags(&c.ev_end, cudaEventDisableTiming));
  CK(cudaEventCreateWithFlags(&det->ev_start, cudaEventDisableTiming));
  for (cudaEvent_t& e : det->ev_tail) CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  CK(cudaStreamCreateWithFlags(&det->s_comp, cudaStreamNonBlocking));
  det->s_hc[0] = det->s_comp;
  for (int i = 1; i < det->n_slots; ++i) CK(cudaStreamCreateWithFlags(&det->s_hc[i], cudaStreamNonBlocking));
  CK(cudaStreamCreateWithFlags(&det->s_h2d, cudaStreamNonBlocking));
  CK(cudaStreamCreateWithFlags(&det->s_d2h, cudaStreamNonBlocking));
  CK(cudaStreamCreateWithFlags(&det->s_join, cudaStreamNonBlocking));
  return RD_OK;
}

// checked builds: the first failed kernel assertion of the last call (RD_ERR_CUDA with a message)
static rd_status check_flag(rd_detector* det) {
  int v = 0;
  CK(cudaMemcpy(&v, (det->need_cur ? det->need_cur : det->d_need) + NEED_N, sizeof(int), cudaMemcpyDeviceToHost));
  if (v) {
    snprintf(g_err, sizeof g_err, "checked build: kernel assertion %d failed at source line %d", v >> 16, v & 0xFFFF);
    return RD_ERR_CUDA;
  }
  return RD_OK;
}

// Mapped pinned host memory of at least `want` elements of `esize` bytes (grown, contents not kept).
static rd_status grow_mapped(void** p, int64_t* cap, int64_t want, size_t esize) {
  want = std::max<int64_t>(want, 1);
  if (*cap >= want) return RD_OK;
  cudaFreeHost(*p);
  *p = nullptr;
  *cap = 0;
  CK(cudaHostAlloc(p, esize * want, cudaHostAllocMapped));
  *cap = want;
  return RD_OK;
}

rd_status rd_submit_host(rd_detector* det, const void* h_frames, int64_t pitch, int64_t fstride, int32_t n,
                         rd_ring* h_rings, int32_t ring_cap_total, int32_t* h_counts, int32_t* h_offsets) {
  if (!det || n < 1 || !h_counts || !h_offsets || ring_cap_total < 0 || (ring_cap_total > 0 && !h_rings))
    return RD_ERR_PARAM;
  rd_status s = check_frames(det, h_frames, pitch, fstride, n);
  if (s != RD_OK) return s;
  if (det->n_pend >= RD_HOST_DEPTH) return RD_ERR_STATE;
  CK(cudaSetDevice(det->device));
  s = ensure_host_path(det);
  if (s != RD_OK) return s;
  const int j = (det->pend_head + det->n_pend) % RD_HOST_DEPTH;   // the call's slot (its last user was waited for)
  rd_detector::HostCall& c = det->hcall[j];
  if ((s = grow_mapped((void**)&c.h_stage, &c.stage_cap, ring_cap_total, sizeof(rd_ring))) != RD_OK) return s;
  if ((s = grow_mapped((void**)&c.h_co, &c.co_cap, 3LL * n + 1, sizeof(int))) != RD_OK) return s;
  int* need = det->d_need + (1 + j) * (NEED_N + 1);
  const int W = det->cfg.width, H = det->cfg.height, pb = det->P.pixel_bytes;
  const size_t row = (size_t)W * pb, fbytes = row * H;
  // chunk sizes: with the pipeline empty they ramp up from a quarter chunk by 3/2 per chunk
  // (the first copy is the only one nothing overlaps, and each copy ends before the previous,
  // smaller chunk's compute does); behind a call in flight every chunk is full
  const int C = det->n_pend ? det->chunk_pipe : det->chunk, R = det->room;
  std::vector<int> cstart;
  for (int f = 0, m = det->n_pend ? C : std::max(1, C / 4); f < n; f += m, m = std::min(C, std::max(m + 1, m * 3 / 2)))
    cstart.push_back(f);
  cstart.push_back(n);
  const int nchunks = (int)cstart.size() - 1;
  if (c.cursor_cap < nchunks + 1) {
    cudaFree(c.d_cursor);
    c.d_cursor = nullptr;
    c.cursor_cap = 0;
    CK(cudaMalloc(&c.d_cursor, sizeof(int) * (nchunks + 1)));
    c.cursor_cap = nchunks + 1;
  }
  rd_ring* d_out_rings = nullptr;
  int* d_out_co = nullptr;
  CK(cudaHostGetDevicePointer((void**)&d_out_rings, c.h_stage, 0));
  CK(cudaHostGetDevicePointer((void**)&d_out_co, c.h_co, 0));
  int* d_counts_all = d_out_co;            // [n]
  int* d_offsets_all = d_out_co + n;       // [n + 1]
  int* d_flags_all = d_out_co + 2 * n + 1; // [n]
  // a previous rd_detect (on a caller stream) must finish first; earlier host calls are
  // ordered chunk by chunk below (stage reuse, slot streams)
  if (det->have_last && !det->last_host) {
    CK(cudaStreamWaitEvent(det->s_h2d, det->ev_last, 0));
    for (int i = 0; i < det->n_slots; ++i) CK(cudaStreamWaitEvent(det->s_hc[i], det->ev_last, 0));
  }
  CK(cudaMemsetAsync(need, 0, sizeof(int) * (NEED_N + 1), det->s_h2d));
  CK(cudaMemsetAsync(c.d_cursor, 0, sizeof(int), det->s_h2d));
  CK(cudaEventRecord(det->ev_start, det->s_h2d));   // the memsets before any chunk's kernels
  for (int i = 0; i < det->n_slots; ++i) CK(cudaStreamWaitEvent(det->s_hc[i], det->ev_start, 0));
  // RD_HOST_TRACE: per-chunk copy / compute times on stderr (diagnostics only; synchronous)
  const bool trace = getenv("RD_HOST_TRACE") != nullptr;
  std::vector<cudaEvent_t> tev;
  auto mark = [&](cudaStream_t st) {
    if (!trace) return;
    cudaEvent_t e;
    cudaEventCreate(&e);
    cudaEventRecord(e, st);
    tev.push_back(e);
  };
  for (int k = 0; k < nchunks; ++k) {
    const int f0 = cstart[k], m = cstart[k + 1] - f0;
    // buffer slot and stream b: a chunk overlaps the previous one (other slot) and follows the
    // one before it on the same stream; stage q holds its frames (rotation across calls)
    const uint64_t seq = det->chunk_seq++;
    const int b = (int)(seq % det->n_slots), q = (int)(seq % rd_detector::NSTAGE);
    cudaStream_t sc = det->s_hc[b];
    // the H2D into stage q only after the stage's previous chunk finished computing
    if (seq >= (uint64_t)rd_detector::NSTAGE) CK(cudaStreamWaitEvent(det->s_h2d, det->ev_done[q], 0));
    mark(det->s_h2d);
    const char* src = (const char*)h_frames + (size_t)f0 * fstride;
    if (pitch == (int64_t)row && fstride == (int64_t)fbytes) {
      CK(cudaMemcpyAsync(det->d_stage[q], src, fbytes * m, cudaMemcpyHostToDevice, det->s_h2d));
    } else {
      for (int i = 0; i < m; ++i)
        CK(cudaMemcpy2DAsync((char*)det->d_stage[q] + fbytes * i, row, src + (size_t)i * fstride, pitch, row, H,
                             cudaMemcpyHostToDevice, det->s_h2d));
    }
    CK(cudaEventRecord(det->ev_h2d[q], det->s_h2d));
    mark(det->s_h2d);
    CK(cudaStreamWaitEvent(sc, det->ev_h2d[q], 0));
    mark(sc);
    s = detect_impl(det, det->d_stage[q], row, fbytes, m, sc, b * R, b, 1, need);
    if (s != RD_OK) return s;
    CK(cudaEventRecord(det->ev_done[q], sc));
    // A11 for the chunk: its first offset is the previous chunk's end (chained through d_cursor)
    if (k > 0) CK(cudaStreamWaitEvent(sc, det->ev_d2h[(seq - 1) % rd_detector::NSTAGE], 0));
    Params V, V16;
    frame_view(det, b * R, b, V, V16, need);
    CK(launch_emit(m, V, d_out_rings, ring_cap_total, d_counts_all + f0, d_offsets_all + f0, c.d_cursor + k,
                   c.d_cursor + k + 1, d_flags_all + f0, sc));
    if (det->timing) CK(cudaEventRecord(det->tev[RD_NEV * (size_t)(det->n_timed - 1) + RD_NEV - 1], sc));
    CK(cudaEventRecord(det->ev_d2h[q], sc));
    mark(sc);
  }
  // the call's end: every stream's tail, joined on s_join (no working stream waits for it)
  CK(cudaEventRecord(det->ev_tail[0], det->s_h2d));
  CK(cudaStreamWaitEvent(det->s_join, det->ev_tail[0], 0));
  for (int i = 0; i < det->n_slots; ++i) {
    CK(cudaEventRecord(det->ev_tail[1 + i], det->s_hc[i]));
    CK(cudaStreamWaitEvent(det->s_join, det->ev_tail[1 + i], 0));
  }
  CK(cudaEventRecord(c.ev_end, det->s_join));
  CK(cudaEventRecord(det->ev_last, det->s_join));
  if (trace) {   // per chunk: h2d start/end, compute start, emit end (ms from the first copy)
    CK(cudaEventSynchronize(c.ev_end));
    for (size_t i = 0; i + 4 <= tev.size(); i += 4) {
      float t[4];
      for (int jj = 0; jj < 4; ++jj) cudaEventElapsedTime(&t[jj], tev[0], tev[i + jj]);
      fprintf(stderr, "rd: chunk %zu h2d %.3f-%.3f comp %.3f-%.3f\n", i / 4, t[0], t[1], t[2], t[3]);
    }
    for (cudaEvent_t e : tev) cudaEventDestroy(e);
  }
  c.h_rings = h_rings;
  c.cap = ring_cap_total;
  c.h_counts = h_counts;
  c.h_offsets = h_offsets;
  c.n = n;
  det->n_pend++;
  det->have_last = true;
  det->last_host = true;
  return RD_OK;
}

rd_status rd_wait_host(rd_detector* det) {
  if (!det) return RD_ERR_PARAM;
  if (!det->n_pend) return RD_ERR_STATE;
  CK(cudaSetDevice(det->device));
  const int j = det->pend_head;
  rd_detector::HostCall& c = det->hcall[j];
  CK(cudaEventSynchronize(c.ev_end));
  det->pend_head = (j + 1) % RD_HOST_DEPTH;
  det->n_pend--;
  const int n = c.n;
  det->need_cur = det->d_need + (1 + j) * (NEED_N + 1);
  det->last_co = c.h_co;
  det->last_n = n;
  if (rd_status cs = check_flag(det)) return cs;
  memcpy(c.h_counts, c.h_co, sizeof(int) * n);
  memcpy(c.h_offsets, c.h_co + n, sizeof(int) * (n + 1));
  int64_t total = 0;   // rings written: the valid frames' ranges (all inside the capacity)
  rd_status result = RD_OK;
  for (int i = 0; i < n; ++i) {
    if (c.h_counts[i] < 0) result = RD_ERR_CAPACITY;
    else total = std::max<int64_t>(total, (int64_t)c.h_offsets[i] + c.h_counts[i]);
  }
  if (total > 0) memcpy(c.h_rings, c.h_stage, sizeof(rd_ring) * total);
  return result;
}

rd_status rd_detect_host(rd_detector* det, const void* h_frames, int64_t pitch, int64_t fstride, int32_t n,
                         rd_ring* h_rings, int32_t ring_cap_total, int32_t* h_counts, int32_t* h_offsets) {
  if (det && det->n_pend) return RD_ERR_STATE;
  rd_status s = rd_submit_host(det, h_frames, pitch, fstride, n, h_rings, ring_cap_total, h_counts, h_offsets);
  if (s != RD_OK) return s;
  return rd_wait_host(det);
}

rd_status rd_sync(rd_detector* det) {
  if (!det) return RD_ERR_PARAM;
  if (!det->have_last || det->last_host || det->n_pend) return RD_ERR_STATE;
  CK(cudaSetDevice(det->device));
  CK(cudaEventSynchronize(det->ev_last));
  if (rd_status cs = check_flag(det)) return cs;
  std::vector<int> fl(det->last_n);
  CK(cudaMemcpy(fl.data(), det->P.flags, sizeof(int) * det->last_n, cudaMemcpyDeviceToHost));
  for (int v : fl)
    if (v) return RD_ERR_CAPACITY;
  return RD_OK;
}

rd_status rd_query_overflow(rd_detector* det, rd_overflow* out) {
  if (!det || !out) return RD_ERR_PARAM;
  if (!det->have_last || det->n_pend) return RD_ERR_STATE;
  CK(cudaSetDevice(det->device));
  CK(cudaEventSynchronize(det->ev_last));
  int need[NEED_N];
  CK(cudaMemcpy(need, det->need_cur, sizeof need, cudaMemcpyDeviceToHost));
  memset(out, 0, sizeof *out);
  out->needed_ridges_per_tile = need[NEED_RIDGES];
  out->needed_entries_per_tile = need[NEED_ENTRIES];
  out->needed_hotspots_per_level = need[NEED_HOTSPOTS];
  out->needed_rings_per_frame = need[NEED_RINGS];
  const int n = det->last_n;
  std::vector<int> counts(n), offsets(n + 1), flags(n, 0);
  if (det->last_host) {   // the host path leaves counts, offsets and flags in its mapped staging
    memcpy(counts.data(), det->last_co, sizeof(int) * n);
    memcpy(offsets.data(), det->last_co + n, sizeof(int) * (n + 1));
    memcpy(flags.data(), det->last_co + 2 * n + 1, sizeof(int) * n);
  } else {
    CK(cudaMemcpy(flags.data(), det->P.flags, sizeof(int) * n, cudaMemcpyDeviceToHost));
    std::vector<int> pk(n);
    CK(cudaMemcpy(pk.data(), det->P.peak_count, sizeof(int) * n, cudaMemcpyDeviceToHost));
    offsets[0] = 0;
    for (int i = 0; i < n; ++i) {
      const bool valid = (flags[i] & ~OVF_OUTPUT) == 0 && pk[i] <= det->P.ring_cap;
      offsets[i + 1] = offsets[i] + (valid ? pk[i] : 0);
    }
  }
  for (int i = 0; i < n; ++i) {
    if (flags[i]) ++out->frames_overflowed;
    out->flags |= flags[i];
  }
  out->needed_rings_total = offsets[n];
  return RD_OK;
}

rd_status rd_query_flags(rd_detector* det, int32_t n, int32_t* h_flags) {
  if (!det || !h_flags || n < 1) return RD_ERR_PARAM;
  if (!det->have_last || det->last_host || det->n_pend) return RD_ERR_STATE;
  if (n > det->last_n) return RD_ERR_PARAM;
  CK(cudaSetDevice(det->device));
  CK(cudaEventSynchronize(det->ev_last));
  CK(cudaMemcpy(h_flags, det->P.flags, sizeof(int) * n, cudaMemcpyDeviceToHost));
  return RD_OK;
}

rd_status rd_get_stats(rd_detector* det, int32_t n, rd_frame_stats* h) {
  if (!det || !h || n < 1 || n > det->max_batch) return RD_ERR_PARAM;
  if (!det->have_last || det->last_host || det->n_pend) return RD_ERR_STATE;
  if (n > det->last_n) return RD_ERR_PARAM;
  static_assert(sizeof(rd_frame_stats) == sizeof(Stats), "stats layout");
  CK(cudaSetDevice(det->device));
  CK(cudaEventSynchronize(det->ev_last));
  CK(cudaMemcpy(h, det->P.stats, sizeof(Stats) * n, cudaMemcpyDeviceToHost));
  return RD_OK;
}

// members of frame `frame` into det->d_members (grown as needed); *npk, *total on return
static rd_status members_impl(rd_detector* det, int frame, int* npk_out, int* total_out) {
  const Params& P = det->P;
  int flags = 0, npk = 0;
  CK(cudaStreamWaitEvent(det->s_aux, det->ev_last, 0));
  CK(cudaMemcpyAsync(&flags, P.flags + frame, sizeof(int), cudaMemcpyDeviceToHost, det->s_aux));
  CK(cudaMemcpyAsync(&npk, P.peak_count + frame, sizeof(int), cudaMemcpyDeviceToHost, det->s_aux));
  CK(cudaStreamSynchronize(det->s_aux));
  if ((flags & ~OVF_OUTPUT) != 0 || npk > P.ring_cap) return RD_ERR_CAPACITY;   // no valid ring list
  CK(launch_members(P, frame, 0, det->d_mem_off, nullptr, det->s_aux));
  int total = 0;
  CK(cudaMemcpyAsync(&total, det->d_mem_off + npk, sizeof(int), cudaMemcpyDeviceToHost, det->s_aux));
  CK(cudaStreamSynchronize(det->s_aux));
  if (total > det->members_cap) {
    CK(cudaFree(det->d_members));
    det->d_members = nullptr;
    det->members_cap = 0;
    CK(cudaMalloc(&det->d_members, sizeof(uint32_t) * total));
    det->members_cap = total;
  }
  if (total > 0) CK(launch_members(P, frame, 1, det->d_mem_off, det->d_members, det->s_aux));
  *npk_out = npk;
  *total_out = total;
  return RD_OK;
}

rd_status rd_ring_members(rd_detector* det, int32_t frame, int32_t* h_offsets, int32_t offsets_cap,
                          uint32_t* h_members, int64_t cap, int64_t* n_total) {
  if (!det || !n_total || frame < 0 || frame >= det->max_batch || offsets_cap < 0 || cap < 0 ||
      (offsets_cap > 0 && !h_offsets) || (cap > 0 && !h_members))
    return RD_ERR_PARAM;
  if (!det->have_last || det->last_host || det->n_pend || frame >= det->last_n) return RD_ERR_STATE;
  CK(cudaSetDevice(det->device));
  int npk = 0, total = 0;
  rd_status s = members_impl(det, frame, &npk, &total);
  if (s != RD_OK) return s;
  const int no = std::min(offsets_cap, npk + 1);
  if (no > 0) CK(cudaMemcpyAsync(h_offsets, det->d_mem_off, sizeof(int) * no, cudaMemcpyDeviceToHost, det->s_aux));
  const int64_t nm = std::min<int64_t>(cap, total);
  if (nm > 0)
    CK(cudaMemcpyAsync(h_members, det->d_members, sizeof(uint32_t) * nm, cudaMemcpyDeviceToHost, det->s_aux));
  CK(cudaStreamSynchronize(det->s_aux));
  *n_total = total;
  return RD_OK;
}

rd_status rd_debug_dump(rd_detector* det, int32_t frame, int32_t what, void* h_buf, int64_t cap_bytes,
                        int64_t* n_out) {
  if (!det || !n_out || frame < 0 || frame >= det->max_batch || cap_bytes < 0 || (cap_bytes > 0 && !h_buf))
    return RD_ERR_PARAM;
  if (what < RD_DUMP_RIDGES || what > RD_DUMP_MEMBERS) return RD_ERR_PARAM;
  if (!det->have_last || det->last_host || det->n_pend || frame >= det->last_n) return RD_ERR_STATE;
  if ((what == RD_DUMP_LEVEL_FPR || what == RD_DUMP_HOTSPOTS) && !det->cfg.debug) return RD_ERR_STATE;
  CK(cudaSetDevice(det->device));
  CK(cudaEventSynchronize(det->ev_last));
  const Params& P = det->P;
  if (what == RD_DUMP_RIDGES) {
    const int64_t nb = (int64_t)P.nbx * P.nby;
    std::vector<int> cnt(nb);
    std::vector<uint32_t> xy((size_t)nb * P.ridge_cap);
    std::vector<double2> d((size_t)nb * P.ridge_cap);
    CK(cudaMemcpy(cnt.data(), P.bin_count + frame * nb, sizeof(int) * nb, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(xy.data(), P.bin_xy + frame * nb * P.ridge_cap, sizeof(uint32_t) * xy.size(),
                  cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(d.data(), P.bin_d + frame * nb * P.ridge_cap, sizeof(double2) * d.size(), cudaMemcpyDeviceToHost));
    rd_ridge* out = (rd_ridge*)h_buf;
    const int64_t cap = cap_bytes / (int64_t)sizeof(rd_ridge);
    int64_t k = 0;
    for (int64_t b = 0; b < nb; ++b)
      for (int i = 0; i < std::min(cnt[b], P.ridge_cap); ++i, ++k)
        if (k < cap) {
          const uint32_t v = xy[b * P.ridge_cap + i];
          out[k].x = (int32_t)(v & 0xFFFFu);
          out[k].y = (int32_t)(v >> 16);
          out[k].dx = d[b * P.ridge_cap + i].x;
          out[k].dy = d[b * P.ridge_cap + i].y;
        }
    *n_out = k;
    return RD_OK;
  }
  if (what == RD_DUMP_LEVEL_FPR) {
    static_assert(sizeof(rd_level_fpr) == 32, "fingerprint layout");
    std::vector<unsigned long long> f(3 * (size_t)P.n_levels);
    CK(cudaMemcpy(f.data(), P.dbg_fpr + (int64_t)frame * 3 * P.n_levels, sizeof(unsigned long long) * f.size(),
                  cudaMemcpyDeviceToHost));
    rd_level_fpr* out = (rd_level_fpr*)h_buf;
    const int64_t cap = cap_bytes / (int64_t)sizeof(rd_level_fpr);
    for (int li = 0; li < P.n_levels && li < cap; ++li) {
      out[li].r = P.r_lo + li;
      out[li].pad = 0;
      out[li].votes = (int64_t)f[3 * li];
      out[li].sq = (int64_t)f[3 * li + 1];
      out[li].pos = (int64_t)f[3 * li + 2];
    }
    *n_out = P.n_levels;
    return RD_OK;
  }
  if (what == RD_DUMP_HOTSPOTS) {
    static_assert(sizeof(rd_hotspot) == sizeof(HotRec), "hotspot layout");
    int n = 0;
    CK(cudaMemcpy(&n, P.dbg_count + frame, sizeof(int), cudaMemcpyDeviceToHost));
    const int64_t m = std::min<int64_t>(std::min<int64_t>(n, P.dbg_cap), cap_bytes / (int64_t)sizeof(HotRec));
    if (m > 0)
      CK(cudaMemcpy(h_buf, P.dbg_hot + (int64_t)frame * P.dbg_cap, sizeof(HotRec) * m, cudaMemcpyDeviceToHost));
    *n_out = n;
    return RD_OK;
  }
  int npk = 0, total = 0;   // RD_DUMP_MEMBERS
  rd_status s = members_impl(det, frame, &npk, &total);
  if (s != RD_OK) return s;
  const int64_t nm = std::min<int64_t>(cap_bytes / (int64_t)sizeof(uint32_t), total);
  if (nm > 0)
    CK(cudaMemcpyAsync(h_buf, det->d_members, sizeof(uint32_t) * nm, cudaMemcpyDeviceToHost, det->s_aux));
  CK(cudaStreamSynchronize(det->s_aux));
  *n_out = total;
  return RD_OK;
}

rd_status rd_set_timing(rd_detector* det, int32_t on) {
  if (!det) return RD_ERR_PARAM;
  CK(cudaSetDevice(det->device));
  if (det->n_timed) CK(cudaDeviceSynchronize());
  det->timing = on != 0;
  det->n_timed = 0;
  return RD_OK;
}

rd_status rd_kernel_times(rd_detector* det, float* h_ms, int32_t* n_calls) {
  if (!det || !h_ms || !n_calls) return RD_ERR_PARAM;
  CK(cudaSetDevice(det->device));
  float acc[RD_NEV - 1] = {0, 0, 0, 0};
  for (int c = 0; c < det->n_timed; ++c) {
    cudaEvent_t* ev = &det->tev[RD_NEV * (size_t)c];
    CK(cudaEventSynchronize(ev[RD_NEV - 1]));
    for (int k = 0; k < RD_NEV - 1; ++k) {
      float ms = 0;
      CK(cudaEventElapsedTime(&ms, ev[k], ev[k + 1]));
      acc[k] += ms;
    }
  }
  for (int k = 0; k < RD_NEV - 1; ++k) h_ms[k] = acc[k];
  *n_calls = det->n_timed;
  return RD_OK;
}

rd_status rd_phase_cycles(rd_detector* det, int32_t on, uint64_t* h_cycles) {
  if (!det) return RD_ERR_PARAM;
  CK(cudaSetDevice(det->device));
  if (!det->d_prof) CK(cudaMalloc(&det->d_prof, 16 * sizeof(unsigned long long)));
  CK(cudaDeviceSynchronize());
  if (h_cycles) CK(cudaMemcpy(h_cycles, det->d_prof, 16 * sizeof(unsigned long long), cudaMemcpyDeviceToHost));
  CK(cudaMemset(det->d_prof, 0, 16 * sizeof(unsigned long long)));
  det->P.prof = on ? det->d_prof : nullptr;
  return RD_OK;
}

rd_status rd_eigen(const double* d_abc, int64_t n, double* d_out, int32_t* d_deg, void* stream) {
  if (n < 0 || (n > 0 && (!d_abc || !d_out || !d_deg))) return RD_ERR_PARAM;
  CK(launch_eigen(d_abc, n, d_out, d_deg, (cudaStream_t)stream));
  return RD_OK;
}

}  // extern "C"
