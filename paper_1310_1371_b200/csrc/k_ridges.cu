// k_ridges.cu — K1: scale-selection smoothing, 5x5 Sobel Hessian, least principal
// curvature and directed-ridge test, with deterministic compaction into 32x32 bins.
//
// Rows A1-A4 of DESIGN.md §2 ("Directed ridge detection"; SI steps 1-2,
// PAPER.md:919-931).  Per 32x32 output tile, everything stays on chip:
//   I (tile + 3 + K_s halo, replicate border) staged by TMA into shared memory
//   -> R = q (x) I along x                    (int32, exact)
//   -> G = q (x) R along y                    (fp64, exact integers < 2^53)
//   -> horizontal Sobel passes d2, s5, d1     (fp64, exact)
//   -> vertical passes s5, d2, d1 = Ixx, Iyy, Ixy on tile + 1   (fp64, exact)
//   -> kappa (fixed fp64 recipe, no FMA), ridge test on the tile, warp-ballot compaction.
// The integer stages are exact, so their evaluation order is free; only the kappa /
// direction recipe is order-sensitive and it is written with explicit _rn intrinsics.
// Every stencil pass is register-blocked: a thread produces a strip of 8 outputs from a
// sliding window held in registers (one shared-memory load per input, not per tap).
// The TMA kernel is persistent: while a tile is computed, the TMA engine already fetches
// the next tile's input into the other buffer (mbarrier double buffering).
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdlib>

#include "rd_internal.cuh"

namespace rd {

namespace {
constexpr int GRS = T1 + 6;     // G region side (tile + 3)
constexpr int KRS = T1 + 2;     // kappa region side (tile + 1)
constexpr int SB = 8;           // strip length of the register-blocked passes

struct K1Smem {
  int irs, ip, bh, co;          // region side, row pitch (elements), TMA box rows, region column offset
  size_t off_bar, off_in0, off_in1, off_x, off_g, off_k, off_d, off_s, off_list, off_cnt, total;
};

__host__ __device__ inline size_t al128(size_t v) { return (v + 127) & ~size_t(127); }

__host__ __device__ inline K1Smem k1_layout(int KS, int pb) {
  K1Smem L;
  L.irs = T1 + 6 + 2 * KS;
  const int vec = 16 / pb;                       // TMA box rows are multiples of 16 bytes
  // The TMA box must start on a 16-byte boundary in x (measured on B200: other starts trap
  // with an illegal instruction), so the box starts `co` elements left of the region; tile
  // origins are multiples of 32 >= 16/pb, hence co is the same for every tile.
  L.co = ((-(3 + KS)) % vec + vec) % vec;
  L.ip = (L.co + L.irs + vec - 1) / vec * vec;
  L.bh = (L.irs + 15) / 16 * 16;                 // TMA box rows (multiple of 16)
  const size_t in_bytes = (size_t)L.bh * L.ip * pb + SB * 4;    // + strip over-read pad
  const size_t x_dbl = (size_t)L.irs * GRS > (size_t)3 * GRS * KRS ? (size_t)L.irs * GRS : (size_t)3 * GRS * KRS;
  size_t o = 0;
  L.off_bar = o;  o = al128(o + 16);
  L.off_in0 = o;  o = al128(o + in_bytes);
  L.off_in1 = o;  o = al128(o + in_bytes);
  L.off_x = o;    o = al128(o + 8 * x_dbl);            // R, later HA|HB|HC
  L.off_g = o;    o = al128(o + 8 * (size_t)GRS * GRS);
  L.off_k = o;    o = al128(o + 8 * (size_t)KRS * KRS);
  L.off_d = o;    o = al128(o + 16 * (size_t)T1 * T1);
  L.off_s = o;    o = al128(o + 8 * (size_t)T1 * T1);   // s of candidates, -1 otherwise
  L.off_list = o; o = al128(o + 2 * (size_t)T1 * T1);   // candidate pixel list
  L.off_cnt = o;  o = al128(o + 4 * 33);
  L.total = o;
  return L;
}

// Steps 2-6 for one tile whose input region (origin x0-3-KS, y0-3-KS, replicate border
// already applied) is in sIn with row pitch L.ip.
template <typename PixT, int KS>
__device__ __forceinline__ void ridge_tile(const PixT* __restrict__ sIn, unsigned char* smem, const K1Smem& L,
                                           int x0, int y0, int f, int bx, int by, const Params& P) {
  constexpr int NTAP = 2 * KS + 1;
  constexpr int IRS = T1 + 6 + 2 * KS;
  constexpr int RSTR = (GRS + SB - 1) / SB;
  const int IP = L.ip;
  double* sR = reinterpret_cast<double*>(smem + L.off_x);   // [IRS][GRS]
  double* sHA = sR;                                         // [GRS][KRS] x3 (after R is consumed)
  double* sHB = sHA + GRS * KRS;
  double* sHC = sHB + GRS * KRS;
  double* sG = reinterpret_cast<double*>(smem + L.off_g);   // [GRS][GRS]
  double* sK = reinterpret_cast<double*>(smem + L.off_k);   // [KRS][KRS]
  double2* sD = reinterpret_cast<double2*>(smem + L.off_d); // [T1][T1] (e, Ixy), then rho
  double* sS = reinterpret_cast<double*>(smem + L.off_s);   // [T1][T1] s if candidate, else -1
  uint16_t* sList = reinterpret_cast<uint16_t*>(smem + L.off_list);
  int* sCnt = reinterpret_cast<int*>(smem + L.off_cnt);     // [33]
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int W = P.W, H = P.H;
  int q[NTAP];
#pragma unroll
  for (int j = 0; j < NTAP; ++j) q[j] = P.q[j];

  // 2. row pass (int32 exact: max_value * sum q < 2^31 checked at rd_create)
  for (int it = tid; it < IRS * RSTR; it += K1_THREADS) {
    const int r = it / RSTR, c0 = (it - r * RSTR) * SB;
    const PixT* src = sIn + r * IP + c0;
    int v[SB + NTAP - 1];
#pragma unroll
    for (int j = 0; j < SB + NTAP - 1; ++j) v[j] = (int)src[j];
#pragma unroll
    for (int o = 0; o < SB; ++o) {
      int acc = 0;
#pragma unroll
      for (int j = 0; j < NTAP; ++j) acc += q[j] * v[o + j];
      if (c0 + o < GRS) sR[r * GRS + c0 + o] = (double)acc;
    }
  }
  __syncthreads();
  // 3. column pass (fp64, exact): thread = (column, strip of SB rows)
  for (int it = tid; it < GRS * ((GRS + SB - 1) / SB); it += K1_THREADS) {
    const int c = it % GRS, r0 = (it / GRS) * SB;
    double v[SB + NTAP - 1];
#pragma unroll
    for (int j = 0; j < SB + NTAP - 1; ++j) v[j] = (r0 + j < IRS) ? sR[(r0 + j) * GRS + c] : 0.0;
#pragma unroll
    for (int o = 0; o < SB; ++o) {
      double acc = 0.0;
#pragma unroll
      for (int j = 0; j < NTAP; ++j) acc = fma((double)q[j], v[o + j], acc);
      if (r0 + o < GRS) sG[(r0 + o) * GRS + c] = acc;
    }
  }
  __syncthreads();
  // 4. horizontal Sobel passes on G (correlation; offsets -2..2): thread = (row, strip)
  for (int it = tid; it < GRS * ((KRS + SB - 1) / SB); it += K1_THREADS) {
    const int r = it / ((KRS + SB - 1) / SB), c0 = (it - r * ((KRS + SB - 1) / SB)) * SB;
    double g[SB + 4];
#pragma unroll
    for (int j = 0; j < SB + 4; ++j) g[j] = (c0 + j < GRS) ? sG[r * GRS + c0 + j] : 0.0;
#pragma unroll
    for (int o = 0; o < SB; ++o) {
      if (c0 + o >= KRS) break;
      const double g0 = g[o], g1 = g[o + 1], g2 = g[o + 2], g3 = g[o + 3], g4 = g[o + 4];
      sHA[r * KRS + c0 + o] = (g0 + g4) - 2.0 * g2;                       // d2 = [1,0,-2,0,1]
      sHB[r * KRS + c0 + o] = (g0 + g4) + 4.0 * (g1 + g3) + 6.0 * g2;     // s5 = [1,4,6,4,1]
      sHC[r * KRS + c0 + o] = (g4 - g0) + 2.0 * (g3 - g1);                // d1 = [-1,-2,0,2,1]
    }
  }
  __syncthreads();
  // 5. vertical passes -> Ixx = s5_y (x) d2_x, Iyy = d2_y (x) s5_x, Ixy = d1_y (x) d1_x; kappa.
  //    Tile pixels with kappa < t keep (e, b, s) for step 5b; the others get s = -1.
  constexpr int SB5 = 6;   // 34 columns x 6 strips = 204 work items <= 256 threads
  const double t_int = P.t_int;
  for (int it = tid; it < KRS * ((KRS + SB5 - 1) / SB5); it += K1_THREADS) {
    const int c = it % KRS, r0 = (it / KRS) * SB5;
    double a[SB5 + 4], b[SB5 + 4], d[SB5 + 4];
#pragma unroll
    for (int j = 0; j < SB5 + 4; ++j) {
      const bool ok = r0 + j < GRS;
      a[j] = ok ? sHA[(r0 + j) * KRS + c] : 0.0;
      b[j] = ok ? sHB[(r0 + j) * KRS + c] : 0.0;
      d[j] = ok ? sHC[(r0 + j) * KRS + c] : 0.0;
    }
    const int x = x0 - 1 + c;
#pragma unroll
    for (int o = 0; o < SB5; ++o) {
      const int r = r0 + o;
      if (r >= KRS) break;
      const int y = y0 - 1 + r;
      const bool in_tile = r >= 1 && r <= T1 && c >= 1 && c <= T1;
      double kap = HUGE_VAL, s = -1.0, e = 0.0, Ixy = 0.0;
      if (x >= 2 && x <= W - 3 && y >= 2 && y <= H - 3) {
        const double Ixx = (a[o] + a[o + 4]) + 4.0 * (a[o + 1] + a[o + 3]) + 6.0 * a[o + 2];
        const double Iyy = (b[o] + b[o + 4]) - 2.0 * b[o + 2];
        Ixy = (d[o + 4] - d[o]) + 2.0 * (d[o + 3] - d[o + 1]);
        kap = kappa_of(Ixx, Ixy, Iyy, &s, &e);
        if (!(kap < t_int)) s = -1.0;
      }
      sK[r * KRS + c] = kap;
      if (in_tile) {
        const int k = (r - 1) * T1 + (c - 1);
        sS[k] = s;
        sD[k] = make_double2(e, Ixy);
      }
    }
  }
  __syncthreads();
  // 5b. directions rho of the candidate pixels (kappa < t), dealt evenly to all threads
  {
    unsigned cb[T1 * T1 / K1_THREADS];
#pragma unroll
    for (int it = 0; it < T1 * T1 / K1_THREADS; ++it) {
      cb[it] = __ballot_sync(0xffffffffu, sS[tid + it * K1_THREADS] >= 0.0);
      if (lane == 0) sCnt[it * (K1_THREADS / 32) + warp] = __popc(cb[it]);
    }
    __syncthreads();
    if (warp == 0) {
      int v = sCnt[lane], incl = v;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int n = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += n;
      }
      sCnt[lane] = incl - v;
      if (lane == 31) sCnt[32] = incl;
    }
    __syncthreads();
    const unsigned lt = (1u << lane) - 1u;
#pragma unroll
    for (int it = 0; it < T1 * T1 / K1_THREADS; ++it)
      if ((cb[it] >> lane) & 1u)
        sList[sCnt[it * (K1_THREADS / 32) + warp] + __popc(cb[it] & lt)] = (uint16_t)(tid + it * K1_THREADS);
    const int ncand = sCnt[32];
    __syncthreads();
    for (int i = tid; i < ncand; i += K1_THREADS) {
      const int k = sList[i];
      const double2 eb = sD[k];
      double dx, dy;
      if (direction_of(eb.y, eb.x, sS[k], &dx, &dy)) sD[k] = make_double2(dx, dy);
      else sS[k] = -1.0;   // isotropic: never a ridge (R3)
    }
  }
  __syncthreads();
  // 6. ridge test (kappa_p <= kappa(after), kappa_p < kappa(before); R6) + compaction
  bool is_r[T1 * T1 / K1_THREADS];
  unsigned bal[T1 * T1 / K1_THREADS];
#pragma unroll
  for (int it = 0; it < T1 * T1 / K1_THREADS; ++it) {
    int k = tid + it * K1_THREADS;
    int ty = k / T1, tx = k - ty * T1;
    int x = x0 + tx, y = y0 + ty;
    bool ok = false;
    const bool cand = sS[k] >= 0.0;
    double2 dir = sD[k];
    if (x >= 3 && x <= W - 4 && y >= 3 && y <= H - 4 && cand) {
      double kp = sK[(ty + 1) * KRS + tx + 1];
      int ox = (int)llround(dir.x), oy = (int)llround(dir.y);
      bool after_plus = (oy > 0) || (oy == 0 && ox > 0);
      double kplus = sK[(ty + 1 + oy) * KRS + tx + 1 + ox];
      double kminus = sK[(ty + 1 - oy) * KRS + tx + 1 - ox];
      double kafter = after_plus ? kplus : kminus, kbefore = after_plus ? kminus : kplus;
      ok = (kp <= kafter) && (kp < kbefore);
    }
    is_r[it] = ok;
    bal[it] = __ballot_sync(0xffffffffu, ok);
    if (lane == 0) sCnt[it * (K1_THREADS / 32) + warp] = __popc(bal[it]);
  }
  __syncthreads();
  if (warp == 0) {  // exclusive scan of the 32 (iteration, warp) counts = row-major order
    int v = sCnt[lane];
    int incl = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      int n = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += n;
    }
    sCnt[lane] = incl - v;
    if (lane == 31) sCnt[32] = incl;
  }
  __syncthreads();
  const int total = sCnt[32];
  const int bin = by * P.nbx + bx;
  const int64_t base = ((int64_t)f * P.nbx * P.nby + bin) * P.ridge_cap;
  const unsigned lt = (1u << lane) - 1u;
#pragma unroll
  for (int it = 0; it < T1 * T1 / K1_THREADS; ++it) {
    if (!is_r[it]) continue;
    int slot = sCnt[it * (K1_THREADS / 32) + warp] + __popc(bal[it] & lt);
    if (slot < P.ridge_cap) {
      int k = tid + it * K1_THREADS;
      int ty = k / T1, tx = k - ty * T1;
      P.bin_xy[base + slot] = (uint32_t)(x0 + tx) | ((uint32_t)(y0 + ty) << 16);
      P.bin_d[base + slot] = sD[k];
    }
  }
  if (tid == 0) {
    P.bin_count[(int64_t)f * P.nbx * P.nby + bin] = min(total, P.ridge_cap);
    if (total > P.ridge_cap) atomicOr(&P.flags[f], OVF_RIDGES);
    if (total) atomicAdd(&P.stats[f].ridges, (unsigned long long)total);
  }
}
}  // namespace

// One CTA per tile; input staged with plain loads (any pitch / alignment).
template <typename PixT, int KS>
__global__ void __launch_bounds__(K1_THREADS, 2)
k_ridges(const uint8_t* __restrict__ frames, int64_t pitch, int64_t fstride, Params P) {
  extern __shared__ __align__(128) unsigned char smem[];
  const K1Smem L = k1_layout(KS, (int)sizeof(PixT));
  constexpr int IRS = T1 + 6 + 2 * KS;
  PixT* sIn = reinterpret_cast<PixT*>(smem + L.off_in0);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int f = blockIdx.z;
  const int x0 = blockIdx.x * T1, y0 = blockIdx.y * T1;
  const int W = P.W, H = P.H;
  const uint8_t* frame = frames + (int64_t)f * fstride;
  const int ox = x0 - 3 - KS, oy = y0 - 3 - KS;
  for (int r = warp; r < IRS; r += K1_THREADS / 32) {  // warp per row, replicate border
    const int gy = min(max(oy + r, 0), H - 1);
    const PixT* row = reinterpret_cast<const PixT*>(frame + (int64_t)gy * pitch);
    for (int c = lane; c < IRS; c += 32) sIn[r * L.ip + c] = __ldg(row + min(max(ox + c, 0), W - 1));
  }
  __syncthreads();
  ridge_tile<PixT, KS>(sIn, smem, L, x0, y0, f, blockIdx.x, blockIdx.y, P);
}

// Persistent CTAs; the input region of the next tile is fetched by TMA (zero fill out of
// the frame, then patched to replicate the border) while the current tile is computed.
template <typename PixT, int KS>
__global__ void __launch_bounds__(K1_THREADS, 2)
k_ridges_tma(const __grid_constant__ CUtensorMap tmap, int n_frames, Params P) {
  extern __shared__ __align__(128) unsigned char smem[];
  const K1Smem L = k1_layout(KS, (int)sizeof(PixT));
  constexpr int IRS = T1 + 6 + 2 * KS;
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + L.off_bar);
  PixT* buf[2] = {reinterpret_cast<PixT*>(smem + L.off_in0), reinterpret_cast<PixT*>(smem + L.off_in1)};
  const uint32_t box_bytes = (uint32_t)(L.bh * L.ip * sizeof(PixT));
  const int tid = threadIdx.x;
  const int W = P.W, H = P.H;
  const int tiles_per_frame = P.nbx * P.nby;
  const int ntiles = tiles_per_frame * n_frames;
  if (tid == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    mbar_fence_init();
  }
  __syncthreads();
  auto issue = [&](int t, int b) {
    const int f = t / tiles_per_frame, rem = t - f * tiles_per_frame;
    const int by = rem / P.nbx, bx = rem - by * P.nbx;
    fence_proxy_async_smem();
    mbar_expect_tx(&bar[b], box_bytes);
    tma_load_3d(buf[b], &tmap, &bar[b], bx * T1 - 3 - KS - L.co, by * T1 - 3 - KS, f);
  };
  int t = blockIdx.x;
  if (tid == 0 && t < ntiles) issue(t, 0);
  uint32_t phase[2] = {0u, 0u};
  for (int k = 0; t < ntiles; ++k, t += gridDim.x) {
    const int b = k & 1;
    if (tid == 0 && t + (int)gridDim.x < ntiles) issue(t + gridDim.x, b ^ 1);
    mbar_wait(&bar[b], phase[b]);
    phase[b] ^= 1u;
    const int f = t / tiles_per_frame, rem = t - f * tiles_per_frame;
    const int by = rem / P.nbx, bx = rem - by * P.nbx;
    const int x0 = bx * T1, y0 = by * T1;
    const int ox = x0 - 3 - KS, oy = y0 - 3 - KS;
    PixT* sIn = buf[b] + L.co;   // region origin inside the 16-byte aligned box
    if (ox < 0 || oy < 0 || ox + IRS > W || oy + IRS > H) {  // replicate-border patch
      for (int i = tid; i < IRS * IRS; i += K1_THREADS) {
        const int r = i / IRS, c = i - r * IRS;
        const int sy = min(max(oy + r, 0), H - 1) - oy, sx = min(max(ox + c, 0), W - 1) - ox;
        if (sy != r || sx != c) sIn[r * L.ip + c] = sIn[sy * L.ip + sx];
      }
      __syncthreads();
    }
    ridge_tile<PixT, KS>(sIn, smem, L, x0, y0, f, bx, by, P);
    __syncthreads();   // all reads of buf[b] done before it is refilled
  }
}

size_t k_ridges_smem(int Ks) { return k1_layout(Ks, 2).total; }

namespace {
PFN_cuTensorMapEncodeTiled_v12000 g_encode = nullptr;

bool make_tmap(CUtensorMap* map, const void* frames, int pb, int W, int H, int n, int64_t pitch, int64_t fstride,
               int box_w, int box_h) {
  if (!g_encode) {
    cudaDriverEntryPointQueryResult q;
    void* fn = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess || !fn)
      return false;
    g_encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  }
  if (((uintptr_t)frames & 15) || (pitch & 15) || (fstride & 15) || box_w > 256 || box_h > 256) return false;
  cuuint64_t dims[3] = {(cuuint64_t)W, (cuuint64_t)H, (cuuint64_t)n};
  cuuint64_t strides[2] = {(cuuint64_t)pitch, (cuuint64_t)(n > 1 ? fstride : pitch * H)};
  cuuint32_t box[3] = {(cuuint32_t)box_w, (cuuint32_t)box_h, 1};
  cuuint32_t es[3] = {1, 1, 1};
  CUresult r = g_encode(map, pb == 1 ? CU_TENSOR_MAP_DATA_TYPE_UINT8 : CU_TENSOR_MAP_DATA_TYPE_UINT16, 3,
                        const_cast<void*>(frames), dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                        CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

int g_num_sms = 0;
}  // namespace

template <typename PixT, int KS>
static cudaError_t launch_t(const void* frames, int64_t pitch, int64_t fstride, int n_frames, const Params& P,
                            cudaStream_t st) {
  const K1Smem L = k1_layout(KS, (int)sizeof(PixT));
  CUtensorMap map;
  static const bool no_tma = getenv("RD_NO_TMA") != nullptr;   // diagnostic switch
  if (!no_tma && make_tmap(&map, frames, (int)sizeof(PixT), P.W, P.H, n_frames, pitch, fstride, L.ip, L.bh)) {
    if (!g_num_sms) {
      int dev = 0;
      cudaGetDevice(&dev);
      cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev);
    }
    cudaFuncSetAttribute(k_ridges_tma<PixT, KS>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)L.total);
    int per_sm = 1;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_ridges_tma<PixT, KS>, K1_THREADS, L.total);
    const int ntiles = P.nbx * P.nby * n_frames;
    const int grid = std::min(ntiles, std::max(1, per_sm) * g_num_sms);
    k_ridges_tma<PixT, KS><<<grid, K1_THREADS, L.total, st>>>(map, n_frames, P);
    return cudaGetLastError();
  }
  dim3 grid(P.nbx, P.nby, n_frames);
  cudaFuncSetAttribute(k_ridges<PixT, KS>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)L.total);
  k_ridges<PixT, KS><<<grid, K1_THREADS, L.total, st>>>((const uint8_t*)frames, pitch, fstride, P);
  return cudaGetLastError();
}

template <typename PixT>
static cudaError_t launch_p(const void* frames, int64_t pitch, int64_t fstride, int n, const Params& P,
                            cudaStream_t st) {
  switch (P.Ks) {
    case 1: return launch_t<PixT, 1>(frames, pitch, fstride, n, P, st);
    case 2: return launch_t<PixT, 2>(frames, pitch, fstride, n, P, st);
    case 3: return launch_t<PixT, 3>(frames, pitch, fstride, n, P, st);
    case 4: return launch_t<PixT, 4>(frames, pitch, fstride, n, P, st);
    case 5: return launch_t<PixT, 5>(frames, pitch, fstride, n, P, st);
    case 6: return launch_t<PixT, 6>(frames, pitch, fstride, n, P, st);
    case 7: return launch_t<PixT, 7>(frames, pitch, fstride, n, P, st);
    case 8: return launch_t<PixT, 8>(frames, pitch, fstride, n, P, st);
    case 9: return launch_t<PixT, 9>(frames, pitch, fstride, n, P, st);
    case 10: return launch_t<PixT, 10>(frames, pitch, fstride, n, P, st);
    case 11: return launch_t<PixT, 11>(frames, pitch, fstride, n, P, st);
    case 12: return launch_t<PixT, 12>(frames, pitch, fstride, n, P, st);
    case 13: return launch_t<PixT, 13>(frames, pitch, fstride, n, P, st);
    case 14: return launch_t<PixT, 14>(frames, pitch, fstride, n, P, st);
    case 15: return launch_t<PixT, 15>(frames, pitch, fstride, n, P, st);
  }
  return cudaErrorInvalidValue;
}

bool ridges_stream_ok(const Params& P);
cudaError_t launch_ridges_stream(const void* frames, int64_t pitch, int64_t fstride, int n_frames, const Params& P,
                                 cudaStream_t st);

cudaError_t launch_ridges(const void* frames, int64_t pitch, int64_t fstride, int n_frames, const Params& P,
                          cudaStream_t st) {
  // column-streaming K1 (k_ridges2.cu) unless K_s exceeds its halo or RD_K1_IMPL=1 asks for the tiled one
  static const bool tiled = getenv("RD_K1_IMPL") && atoi(getenv("RD_K1_IMPL")) == 1;
  if ((!tiled || P.feature == 1) && ridges_stream_ok(P))   // edges exist in the streaming K1 only
    return launch_ridges_stream(frames, pitch, fstride, n_frames, P, st);
  if (P.feature == 1) return cudaErrorInvalidValue;
  if (P.pixel_bytes == 1) return launch_p<uint8_t>(frames, pitch, fstride, n_frames, P, st);
  return launch_p<uint16_t>(frames, pitch, fstride, n_frames, P, st);
}

// A3 in isolation (rd_eigen): the same recipe on caller-supplied Hessians.
__global__ void k_eigen(const double* __restrict__ abc, int64_t n, double* __restrict__ out, int* __restrict__ deg) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  double a = abc[3 * i], b = abc[3 * i + 1], c = abc[3 * i + 2];
  double s, e;
  double k = kappa_of(a, b, c, &s, &e);
  double dx, dy;
  bool ok = direction_of(b, e, s, &dx, &dy);
  out[3 * i] = k;
  out[3 * i + 1] = dx;
  out[3 * i + 2] = dy;
  deg[i] = ok ? 0 : 1;
}

cudaError_t launch_eigen(const double* abc, int64_t n, double* out, int* deg, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  k_eigen<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(abc, n, out, deg);
  return cudaGetLastError();
}

}  // namespace rd
