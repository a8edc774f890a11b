// k_ridges.cu — K1: scale-selection smoothing, 5x5 Sobel Hessian, least principal
// curvature and directed-ridge test, with deterministic compaction into 32x32 bins.
//
// Rows A1-A4 of DESIGN.md §2 ("Directed ridge detection"; SI steps 1-2,
// PAPER.md:919-931).  One CTA per 32x32 output tile; everything stays on chip:
//   I (tile + 3 + K_s halo, replicate border, int32)
//   -> R = q (x) I along x                    (int32, exact)
//   -> G = q (x) R along y                    (fp64, exact integers < 2^53)
//   -> horizontal Sobel passes d2, s5, d1     (fp64, exact)
//   -> vertical passes s5, d2, d1 = Ixx, Iyy, Ixy on tile + 1   (fp64, exact)
//   -> kappa (fixed fp64 recipe, no FMA), ridge test on the tile, warp-ballot compaction.
// The integer stages are exact, so their evaluation order is free; only the kappa /
// direction recipe is order-sensitive and it is written with explicit _rn intrinsics.
#include "rd_internal.cuh"

namespace rd {

template <typename PixT>
__global__ void __launch_bounds__(K1_THREADS, 2)
k_ridges(const uint8_t* __restrict__ frames, int64_t pitch, int64_t fstride, Params P) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int Ks = P.Ks;
  const int IRS = T1 + 6 + 2 * Ks;      // input region side
  constexpr int GRS = T1 + 6;           // G region side (tile + 3)
  constexpr int KRS = T1 + 2;           // kappa region side (tile + 1)
  double* sR = reinterpret_cast<double*>(smem);             // [IRS][GRS]
  double* sG = sR + IRS * GRS;                               // [GRS][GRS]
  double* sHA = sG + GRS * GRS;                              // [GRS][KRS]
  double* sHB = sHA + GRS * KRS;
  double* sHC = sHB + GRS * KRS;
  double* sK = sHC + GRS * KRS;                              // [KRS][KRS]
  double2* sD = reinterpret_cast<double2*>(sK + KRS * KRS);  // [T1][T1]
  int* sI = reinterpret_cast<int*>(sD + T1 * T1);            // [IRS][IRS]
  int* sCnt = sI + IRS * IRS;                                // [32]

  const int tid = threadIdx.x;
  const int f = blockIdx.z;
  const int x0 = blockIdx.x * T1, y0 = blockIdx.y * T1;
  const int W = P.W, H = P.H;
  const uint8_t* frame = frames + (int64_t)f * fstride;

  // 1. input region with replicate border
  {
    const int ox = x0 - 3 - Ks, oy = y0 - 3 - Ks;
    for (int i = tid; i < IRS * IRS; i += K1_THREADS) {
      int r = i / IRS, c = i - r * IRS;
      int gy = min(max(oy + r, 0), H - 1), gx = min(max(ox + c, 0), W - 1);
      sI[i] = (int)reinterpret_cast<const PixT*>(frame + (int64_t)gy * pitch)[gx];
    }
  }
  __syncthreads();
  // 2. row pass (int32 exact: max_value * sum q < 2^31 checked at rd_create)
  for (int i = tid; i < IRS * GRS; i += K1_THREADS) {
    int r = i / GRS, c = i - r * GRS;
    const int* row = sI + r * IRS + c;
    int acc = 0;
    for (int j = 0; j <= 2 * Ks; ++j) acc += P.q[j] * row[j];
    sR[i] = (double)acc;
  }
  __syncthreads();
  // 3. column pass (fp64, exact)
  for (int i = tid; i < GRS * GRS; i += K1_THREADS) {
    int r = i / GRS, c = i - r * GRS;
    const double* col = sR + r * GRS + c;
    double acc = 0.0;
    for (int k = 0; k <= 2 * Ks; ++k) acc = fma((double)P.q[k], col[k * GRS], acc);
    sG[i] = acc;
  }
  __syncthreads();
  // 4. horizontal Sobel passes on G (correlation; offsets -2..2)
  for (int i = tid; i < GRS * KRS; i += K1_THREADS) {
    int r = i / KRS, c = i - r * KRS;
    const double* g = sG + r * GRS + c;
    double g0 = g[0], g1 = g[1], g2 = g[2], g3 = g[3], g4 = g[4];
    sHA[i] = (g0 + g4) - 2.0 * g2;                                  // d2 = [1,0,-2,0,1]
    sHB[i] = (g0 + g4) + 4.0 * (g1 + g3) + 6.0 * g2;                // s5 = [1,4,6,4,1]
    sHC[i] = (g4 - g0) + 2.0 * (g3 - g1);                           // d1 = [-1,-2,0,2,1]
  }
  __syncthreads();
  // 5. vertical passes -> Ixx = s5_y (x) d2_x, Iyy = d2_y (x) s5_x, Ixy = d1_y (x) d1_x; kappa
  const double t_int = P.t_int;
  for (int i = tid; i < KRS * KRS; i += K1_THREADS) {
    int r = i / KRS, c = i - r * KRS;
    int y = y0 - 1 + r, x = x0 - 1 + c;
    double kap = HUGE_VAL;
    double2 dir = make_double2(2.0, 2.0);  // 2.0 = "not a candidate"
    if (x >= 2 && x <= W - 3 && y >= 2 && y <= H - 3) {
      const double* a = sHA + r * KRS + c;
      const double* b = sHB + r * KRS + c;
      const double* d = sHC + r * KRS + c;
      double Ixx = (a[0] + a[4 * KRS]) + 4.0 * (a[KRS] + a[3 * KRS]) + 6.0 * a[2 * KRS];
      double Iyy = (b[0] + b[4 * KRS]) - 2.0 * b[2 * KRS];
      double Ixy = (d[4 * KRS] - d[0]) + 2.0 * (d[3 * KRS] - d[KRS]);
      double s, e;
      kap = kappa_of(Ixx, Ixy, Iyy, &s, &e);
      bool in_tile = r >= 1 && r <= T1 && c >= 1 && c <= T1;
      if (in_tile && kap < t_int) {
        double dx, dy;
        if (direction_of(Ixy, e, s, &dx, &dy)) dir = make_double2(dx, dy);
      }
    }
    sK[i] = kap;
    if (r >= 1 && r <= T1 && c >= 1 && c <= T1) sD[(r - 1) * T1 + (c - 1)] = dir;
  }
  __syncthreads();
  // 6. ridge test (kappa_p <= kappa(after), kappa_p < kappa(before); R6) + compaction
  const int warp = tid >> 5, lane = tid & 31;
  bool is_r[T1 * T1 / K1_THREADS];
  unsigned bal[T1 * T1 / K1_THREADS];
#pragma unroll
  for (int it = 0; it < T1 * T1 / K1_THREADS; ++it) {
    int k = tid + it * K1_THREADS;
    int ty = k / T1, tx = k - ty * T1;
    int x = x0 + tx, y = y0 + ty;
    bool ok = false;
    double2 dir = sD[k];
    if (x >= 3 && x <= W - 4 && y >= 3 && y <= H - 4 && dir.x != 2.0) {
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
  const int bin = blockIdx.y * P.nbx + blockIdx.x;
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

size_t k_ridges_smem(int Ks) {
  const int IRS = T1 + 6 + 2 * Ks, GRS = T1 + 6, KRS = T1 + 2;
  size_t dbl = (size_t)IRS * GRS + GRS * GRS + 3 * GRS * KRS + KRS * KRS + 2 * T1 * T1;
  return dbl * 8 + (size_t)IRS * IRS * 4 + 33 * 4;
}

cudaError_t launch_ridges(const void* frames, int64_t pitch, int64_t fstride, int n_frames, const Params& P,
                          cudaStream_t st) {
  dim3 grid(P.nbx, P.nby, n_frames);
  size_t sm = k_ridges_smem(P.Ks);
  if (P.pixel_bytes == 1) {
    cudaFuncSetAttribute(k_ridges<uint8_t>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    k_ridges<uint8_t><<<grid, K1_THREADS, sm, st>>>((const uint8_t*)frames, pitch, fstride, P);
  } else {
    cudaFuncSetAttribute(k_ridges<uint16_t>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    k_ridges<uint16_t><<<grid, K1_THREADS, sm, st>>>((const uint8_t*)frames, pitch, fstride, P);
  }
  return cudaGetLastError();
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
