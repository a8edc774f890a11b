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
// Every stencil pass is register-blocked: a thread produces a strip of 8 outputs from a
// sliding window held in registers (one shared-memory load per input, not per tap).
#include "rd_internal.cuh"

namespace rd {

namespace {
constexpr int GRS = T1 + 6;     // G region side (tile + 3)
constexpr int KRS = T1 + 2;     // kappa region side (tile + 1)
constexpr int SB = 8;           // strip length of the register-blocked passes
}  // namespace

template <typename PixT, int KS>
__global__ void __launch_bounds__(K1_THREADS, 2)
k_ridges(const uint8_t* __restrict__ frames, int64_t pitch, int64_t fstride, Params P) {
  extern __shared__ __align__(16) unsigned char smem[];
  constexpr int IRS = T1 + 6 + 2 * KS;  // input region side
  constexpr int NTAP = 2 * KS + 1;
  constexpr int RSTR = (GRS + SB - 1) / SB;   // row-pass strips per row
  double* sR = reinterpret_cast<double*>(smem);              // [IRS][GRS]
  double* sG = sR + IRS * GRS;                                // [GRS][GRS]
  double* sHA = sG + GRS * GRS;                               // [GRS][KRS]
  double* sHB = sHA + GRS * KRS;
  double* sHC = sHB + GRS * KRS;
  double* sK = sHC + GRS * KRS;                               // [KRS][KRS]
  double2* sD = reinterpret_cast<double2*>(sK + KRS * KRS);   // [T1][T1]
  int* sI = reinterpret_cast<int*>(sD + T1 * T1);             // [IRS][IRS + SB] (padded for strips)
  int* sCnt = sI + IRS * (IRS + SB);                          // [33]
  constexpr int IP = IRS + SB;                                // sI row pitch

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int f = blockIdx.z;
  const int x0 = blockIdx.x * T1, y0 = blockIdx.y * T1;
  const int W = P.W, H = P.H;
  const uint8_t* frame = frames + (int64_t)f * fstride;
  int q[NTAP];
#pragma unroll
  for (int j = 0; j < NTAP; ++j) q[j] = P.q[j];

  // 1. input region with replicate border (warp per row, lanes along the row)
  {
    const int ox = x0 - 3 - KS, oy = y0 - 3 - KS;
    for (int r = warp; r < IRS; r += K1_THREADS / 32) {
      const int gy = min(max(oy + r, 0), H - 1);
      const PixT* row = reinterpret_cast<const PixT*>(frame + (int64_t)gy * pitch);
      for (int c = lane; c < IRS; c += 32) sI[r * IP + c] = (int)__ldg(row + min(max(ox + c, 0), W - 1));
    }
  }
  __syncthreads();
  // 2. row pass (int32 exact: max_value * sum q < 2^31 checked at rd_create)
  for (int it = tid; it < IRS * RSTR; it += K1_THREADS) {
    const int r = it / RSTR, c0 = (it - r * RSTR) * SB;
    const int* src = sI + r * IP + c0;
    int v[SB + NTAP - 1];
#pragma unroll
    for (int j = 0; j < SB + NTAP - 1; ++j) v[j] = src[j];
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
  // 5. vertical passes -> Ixx = s5_y (x) d2_x, Iyy = d2_y (x) s5_x, Ixy = d1_y (x) d1_x; kappa
  const double t_int = P.t_int;
  for (int it = tid; it < KRS * ((KRS + SB - 1) / SB); it += K1_THREADS) {
    const int c = it % KRS, r0 = (it / KRS) * SB;
    double a[SB + 4], b[SB + 4], d[SB + 4];
#pragma unroll
    for (int j = 0; j < SB + 4; ++j) {
      const bool ok = r0 + j < GRS;
      a[j] = ok ? sHA[(r0 + j) * KRS + c] : 0.0;
      b[j] = ok ? sHB[(r0 + j) * KRS + c] : 0.0;
      d[j] = ok ? sHC[(r0 + j) * KRS + c] : 0.0;
    }
    const int x = x0 - 1 + c;
#pragma unroll
    for (int o = 0; o < SB; ++o) {
      const int r = r0 + o;
      if (r >= KRS) break;
      const int y = y0 - 1 + r;
      double kap = HUGE_VAL;
      double2 dir = make_double2(2.0, 2.0);  // 2.0 = "not a candidate"
      if (x >= 2 && x <= W - 3 && y >= 2 && y <= H - 3) {
        const double Ixx = (a[o] + a[o + 4]) + 4.0 * (a[o + 1] + a[o + 3]) + 6.0 * a[o + 2];
        const double Iyy = (b[o] + b[o + 4]) - 2.0 * b[o + 2];
        const double Ixy = (d[o + 4] - d[o]) + 2.0 * (d[o + 3] - d[o + 1]);
        double s, e;
        kap = kappa_of(Ixx, Ixy, Iyy, &s, &e);
        if (r >= 1 && r <= T1 && c >= 1 && c <= T1 && kap < t_int) {
          double dx, dy;
          if (direction_of(Ixy, e, s, &dx, &dy)) dir = make_double2(dx, dy);
        }
      }
      sK[r * KRS + c] = kap;
      if (r >= 1 && r <= T1 && c >= 1 && c <= T1) sD[(r - 1) * T1 + (c - 1)] = dir;
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
  const int IRS = T1 + 6 + 2 * Ks;
  size_t dbl = (size_t)IRS * GRS + GRS * GRS + 3 * GRS * KRS + KRS * KRS + 2 * T1 * T1;
  return dbl * 8 + (size_t)IRS * (IRS + SB) * 4 + 33 * 4;
}

template <typename PixT, int KS>
static cudaError_t launch_t(const void* frames, int64_t pitch, int64_t fstride, int n_frames, const Params& P,
                            cudaStream_t st) {
  dim3 grid(P.nbx, P.nby, n_frames);
  size_t sm = k_ridges_smem(KS);
  cudaFuncSetAttribute(k_ridges<PixT, KS>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  k_ridges<PixT, KS><<<grid, K1_THREADS, sm, st>>>((const uint8_t*)frames, pitch, fstride, P);
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

cudaError_t launch_ridges(const void* frames, int64_t pitch, int64_t fstride, int n_frames, const Params& P,
                          cudaStream_t st) {
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
