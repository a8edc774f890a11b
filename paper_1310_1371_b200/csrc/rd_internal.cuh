// rd_internal.cuh — shared definitions of the librd.so kernels (sm_100a).
// Product code: independent of oracle/ (no shared source, tables or constants).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace rd {

constexpr int T1 = 32;          // K1 (ridge) tile: 32x32 output pixels; also the ridge-bin size
constexpr int KS_MAX = 13;      // smoothing half-width limit: K_s = ceil(3 sigma_s) <= 13 (sigma_s <= 13/3)
constexpr int K3_THREADS = 256;
constexpr int ENTRY_MAX = 65535;   // voting rays per Hough tile (16-bit indices in K2's active list)

// Per-frame overflow flag bits (rd_query_overflow)
constexpr int OVF_RIDGES = 1, OVF_ENTRIES = 2, OVF_HOTSPOTS = 4, OVF_RINGS = 8, OVF_DEBUG = 16, OVF_OUTPUT = 32;
// needed capacities (rd_query_overflow): largest value met, kept with atomicMax
constexpr int NEED_RIDGES = 0, NEED_ENTRIES = 1, NEED_HOTSPOTS = 2, NEED_RINGS = 3, NEED_N = 4;

struct Peak {          // peak record produced by K2, consumed by K3 (24 B)
  int32_t x, y, r, raw;
  int64_t S;
};

struct HotRec {        // debug hotspot record (24 B), same layout as rd_hotspot
  int32_t r, y, x, raw;
  int64_t S;
};

struct Stats {         // per-frame counters (same layout as rd_frame_stats)
  unsigned long long ridges, votes, hotspots, peaks;
};

struct Ring {          // == rd_ring (64 B)
  int32_t cx, cy, r, raw_votes;
  int64_t score_fixed;
  int32_t inliers, fit_ok;
  double fx, fy, fr, rms;
};

// Shared-memory layout of the persistent Hough kernel (byte offsets; host-computed)
struct K2Layout {
  int cb, raws, rawp, lvlc;   // counter bytes, raw rows, row pitch (cells), cells per level
  int rawc;                   // raw columns (tile width + 2 halo); raws = tile height + 2 halo
  int raw, hS, sd, rr, xy, rr16, hcell, hraw, task, cand, cdef, act, hcnt, w, wst, k, tn, dummy, mbar, total;
  uint32_t rawp_magic;        // ceil(2^32 / rawp): cell / rawp = umulhi(cell, magic) for cells < 2^16
};

// Everything the kernels need, passed by value (< 4 KB).
struct Params {
  int W, H, pixel_bytes;
  int Ks;
  int q[2 * KS_MAX + 1];        // smoothing taps, 2^10 fixed point (A1)
  double t_int;                 // curvature threshold in integer-Hessian units
  int feature;                  // 0: directed ridges; 1: directed edges (NEXT-2, R19)
  double t_edge2;               // edges: (t_e * 128 (sum q)^2)^2, compared with |grad|^2 in fp64
  int r_lo, r_hi, r_min, r_max, n_levels;
  int T_raw;
  int K_max;                    // largest level half-width
  int hal;                      // K2 raw halo = K_max + 1
  float k_slope, k_icpt;        // K_r <= k_slope * r + k_icpt (conservative, for ray intervals)
  // level tables (device, n_levels entries, index r - r_lo)
  const int* lvlK;              // K_r
  const int* lvlW;              // [n_levels][WSTRIDE] w_r(0..K_r), 2^12 fixed point
  const double* lvlTn;          // T_norm(r) in S units
  const int* lvlAnn;            // annulus half-width w(r)
  int wstride;
  const uint32_t* lvlWP;        // [n_levels][4 alignments][wp_nw][2] byte-plane weight words (K2 dp4a rows)
  int wp_nw;                    // weight words per row and alignment
  // ridge bins (K1 output)
  int nbx, nby;                 // 32x32 bins per frame
  int ridge_cap;                // per bin
  int* bin_count;               // [F][nby*nbx]
  uint32_t* bin_xy;             // [F][bins][ridge_cap] x | y<<16
  double2* bin_d;               // [F][bins][ridge_cap] K1: unnormalised v; K1.5 overwrites it with rho = v / |v| (dx, dy)
  // Hough tiles (K2)
  int k2t;                      // Hough tile width (k2t x k2ty accumulator cells per CTA)
  int k2ty;                     // Hough tile height (the persistent K2 balances the tiling; else = k2t)
  int parts;                    // concurrent launches sharing the GPU (rd_detect's batch parts)
  int ntx, nty;                 // Hough tiles per frame
  int entry_cap, hot_cap;
  int* ray_count;               // [F][tiles] voting rays routed to each Hough tile (K1.5)
  double2* ray_d;               // [F][tiles][entry_cap] (s*dx, s*dy)
  uint32_t* ray_xy;             // [F][tiles][entry_cap] x | y<<16
  uint32_t* ray_r;              // [F][tiles][entry_cap] ra | rb<<16 (level indices)
  int* k2_work;                 // persistent K2: next work item [0] main pass, [1] redo pass (zeroed per call)
  int* redo;                    // [F] frames whose byte counters overflowed (zeroed per call)
  int* redo_list;               // redo pass only: [0] count, [1..] frames; null in the main pass
  int force_redo;               // test knob (RD_K2_FORCE_REDO): every frame takes the 16-bit redo pass
  int ablate;                   // timing experiments only (RD_K2_ABLATE bits: 1 no window sums, 2 no NMS, 4 no S tasks,
                                //   8 no vote atomics, 16 no votes, 32 integer fixed-point vote targets)
  int u8_limit;                 // byte-counter value that triggers the redo (255; RD_K2_U8_LIMIT in tests)
  int k2_rcap;                  // K2: rays of a tile resident in shared memory (the rest read from global)
  int k2_ctas_per_sm;           // K2: resident CTAs per SM of a launch (0: as many as fit)
  const void* zeros;            // K2: a zero block at least as large as its level buffers (bulk-copy clears)
  int k2_rr16;                  // 1: level intervals as 2 bytes (ra | rb << 8; levels < 255): K1.5 writes
                                //   ray_r as uint16_t, K2 keeps every entry's interval in shared memory
                                //   (no resident rays: direction and pixel from L2)
  K2Layout k2o;
  int ring_cap;
  Peak* peaks;                  // [F][ring_cap]
  int* peak_count;              // [F]
  int* flags;                   // [F] overflow bits
  Stats* stats;                 // [F]
  Ring* rings;                  // [F][ring_cap] K3 output in canonical order (compacted by k_emit)
  int* need;                    // [NEED_N] capacities needed by the call (atomicMax)
  int* need_ridges;             // [F] largest ridge bin of each frame (K1.5; folded into need by k_scan)
  int n_sm;                     // SMs of the device (grid sizing)
  int k1_slots;                 // resident K1 CTAs on the device (row-segment choice)
  int debug;
  unsigned long long* dbg_fpr;  // [F][n_levels][3] level fingerprints (debug): sum raw, sum raw^2, sum raw*(yW+x)
  int* check;                   // checked builds (RD_CHECKED): first failed assertion, code << 16 | line
  int jitter;                   // checked builds: perturb the warp schedule of K2 (RD_JITTER=1)
  unsigned long long* prof;     // optional per-phase cycle counters (rd_phase_cycles), may be null
  int dbg_cap;
  HotRec* dbg_hot;              // [F][dbg_cap]
  int* dbg_count;               // [F]
};

// ---------------------------------------------------------------- checked builds
// The sanitizer tier of SURVEY.md §4 (T5) by assertion: a build with -DRD_CHECKED (librd_checked.so,
// tests/test_checked.py) tests every shared-memory and global index the kernels form against the
// bounds of its array; the first failure is recorded in P.check (code << 16 | source line) and
// reported by rd_sync / rd_detect_host as RD_ERR_CUDA.  Product builds compile the checks away.
enum CheckCode { CK_K1_SMEM = 1, CK_K1_BIN, CK_K15_TILE, CK_K15_ENTRY, CK_K2_VOTE, CK_K2_LIST, CK_K2_WINDOW,
                 CK_K2_TASK, CK_K2_NMS, CK_K2_RAY, CK_K3_ORDER, CK_K3_BIN, CK_EMIT };
__device__ __noinline__ inline void rd_check_fail(int* check, int code, int line) {
  if (check) atomicCAS(check, 0, (code << 16) | (line & 0xFFFF));
}
#ifdef RD_CHECKED
#define RD_CHECK(cond, code)                                                   \
  do {                                                                         \
    if (!(cond)) ::rd::rd_check_fail(P.check, (code), __LINE__);               \
  } while (0)
#else
#define RD_CHECK(cond, code) \
  do {                       \
  } while (0)
#endif

// ---------------------------------------------------------------- fp64 recipe (A3)
// kappa = 0.5*(T - sqrt(e*e + 4*(b*b))) and the unit eigenvector, each operation
// rounded separately (no FMA contraction): DESIGN.md A3 / PAPER.md:301-303.
__device__ __forceinline__ double kappa_of(double a, double b, double c, double* s_out, double* e_out) {
  double T = __dadd_rn(a, c);
  double e = __dsub_rn(a, c);
  double D = __dadd_rn(__dmul_rn(e, e), __dmul_rn(4.0, __dmul_rn(b, b)));
  double s = __dsqrt_rn(D);
  *s_out = s;
  *e_out = e;
  return __dmul_rn(0.5, __dsub_rn(T, s));
}
// returns false if degenerate (e == 0 and b == 0)
__device__ __forceinline__ bool direction_of(double b, double e, double s, double* dx, double* dy) {
  if (e == 0.0 && b == 0.0) { *dx = 0.0; *dy = 0.0; return false; }
  double vx, vy;
  if (e >= 0.0) { vx = -b; vy = __dmul_rn(0.5, __dadd_rn(e, s)); }
  else { vx = __dmul_rn(0.5, __dsub_rn(s, e)); vy = -b; }
  double n = __dsqrt_rn(__dadd_rn(__dmul_rn(vx, vx), __dmul_rn(vy, vy)));
  *dx = __ddiv_rn(vx, n);
  *dy = __ddiv_rn(vy, n);
  return true;
}

// The same direction before its normalisation: K1 keeps v = (vx, vy) and K1.5 divides by |v|
// where the ridges are dense in the lanes (the square root and the two divisions are ~95
// instructions, which K1 ran warp-wide wherever one lane held a candidate).  False if degenerate.
__device__ __forceinline__ bool direction_raw(double b, double e, double s, double* vx, double* vy) {
  if (e == 0.0 && b == 0.0) { *vx = 0.0; *vy = 0.0; return false; }
  if (e >= 0.0) { *vx = -b; *vy = __dmul_rn(0.5, __dadd_rn(e, s)); }
  else { *vx = __dmul_rn(0.5, __dsub_rn(s, e)); *vy = -b; }
  return true;
}
// rho = v / |v| with direction_of's roundings (v != 0)
__device__ __forceinline__ void normalise_dir(double vx, double vy, double* dx, double* dy) {
  const double n = __dsqrt_rn(__dadd_rn(__dmul_rn(vx, vx), __dmul_rn(vy, vy)));
  *dx = __ddiv_rn(vx, n);
  *dy = __ddiv_rn(vy, n);
}
// (llround(rho.x), llround(rho.y)) of rho = normalise_dir(v), each in {-1, 0, 1}, without the
// division where the squares decide: |rn(vx / n)| >= 1/2 iff vx^2 >= (vx^2 + vy^2)(1 + eta) / 4 with
// |eta| < 2^-49 (the roundings of the two squares, their sum, the root and the quotient), i.e.
// iff 3 vx^2 - vy^2 >= eta'(vx^2 + vy^2); outside a 2^-40 band around equality the sign of
// 3 vx^2 - vy^2 decides, inside it (never seen; v's components are dyadic rationals and sqrt(3)
// is not) the exact recipe runs.
__device__ __forceinline__ void dir_step(double vx, double vy, int* ox, int* oy) {
  const double A = vx * vx, B = vy * vy, band = (A + B) * 0x1p-40;
  const double tx = 3.0 * A - B, ty = 3.0 * B - A;
  if (fabs(tx) > band && fabs(ty) > band) {
    *ox = tx > 0.0 ? (vx > 0.0 ? 1 : -1) : 0;
    *oy = ty > 0.0 ? (vy > 0.0 ? 1 : -1) : 0;
  } else {
    double dx, dy;
    normalise_dir(vx, vy, &dx, &dy);
    *ox = (int)llround(dx);
    *oy = (int)llround(dy);
  }
}

// round half away from zero of an exactly computed double (llround semantics)
__device__ __forceinline__ int round_half_away(double v) { return (int)llround(v); }

// ---------------------------------------------------------------- TMA / mbarrier (sm_90+)
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_fence_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
// 1-D bulk copy (TMA engine) of `bytes` (a multiple of 16; 16-byte aligned ends) from global
// to shared memory; completes on `bar`
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
// 3-D tiled TMA load of box (x, y, z) of the tensor map into shared memory; completes on `bar`
__device__ __forceinline__ void tma_load_3d(void* dst, const void* tmap, uint64_t* bar, int x, int y, int z) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], [%2];"
      ::"r"(smem_u32(dst)), "l"(tmap), "r"(smem_u32(bar)), "r"(x), "r"(y), "r"(z)
      : "memory");
}

}  // namespace rd
