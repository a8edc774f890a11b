// k_ridges2.cu — K1 (column-streaming form): scale-selection smoothing, 5x5 Sobel Hessian,
// least principal curvature and directed-ridge test, with ridges compacted straight into
// the 32x32 bins.
//
// Rows A1-A4 of DESIGN.md §1 ("Directed ridge detection"; SI steps 1-2,
// PAPER.md:919-931).  A CTA owns a vertical strip of KS_COLS = 384 frame columns (352
// output columns = 11 ridge bins, 16 halo columns on each side) and a segment of rows; thread
// t owns column X0 - 16 + t and the CTA walks down the rows, RB input rows per step:
//   R = q (x) I along x      from the input rows in shared memory         (int32, exact)
//   G = q (x) R along y      2K_s+1 R values in a register window          (fp64, exact)
//   HA|HB|HC = d2|s5|d1 (x) G along x   from the G rows in shared memory   (fp64, exact)
//   Ixx|Iyy|Ixy = s5|d2|d1 (x) H along y   5-row register windows          (fp64, exact)
//   kappa (fixed fp64 recipe, no FMA) and rho of the candidates kappa < t, into row rings
//   ridge test one row behind against the kappa ring (R6)
// Three phase boundaries per step of RB rows, each joining a warp only with its two neighbours
// (mbarriers; every exchange is between columns < 32 apart); the RB rows of a phase are
// independent chains.
// Every integer stage is exact, so evaluation order is free; kappa/rho use the shared
// explicit-rounding recipe (rd_internal.cuh).  Replicate border: input rows and columns are
// clamped at load time.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>

#include "rd_internal.cuh"

namespace rd {

namespace {
#ifndef RD_K1_COLS
#define RD_K1_COLS 384   // 352 output columns = 11 bins (cfg3: 3 strips); 256 and 320 measured slower
#endif
constexpr int KS_COLS = RD_K1_COLS; // strip columns = threads per CTA (32 + a multiple of 32)
constexpr int KS_HALO = 16;         // halo columns on each side (>= K_s + 3)
constexpr int KS_OUT = KS_COLS - 2 * KS_HALO;   // 224 output columns = 7 bins
constexpr int KS_NB = KS_OUT / 32;  // bins per strip
#ifndef RD_K1_MINB
#define RD_K1_MINB 2   // 2 CTAs of 384 threads at 80 registers
#endif
#ifndef RD_K1_RB
#define RD_K1_RB 4   // rows per step (TMA input: 9.8 us/frame vs 10.6 at 2, 10.9 at 3, 10.6 at 6 on cfg3)
#endif
#define NOT_CAND __longlong_as_double(0x7ff8000000000000LL)   // v.x of a pixel that is not a ridge candidate (NaN)
#ifndef RD_K1_NSTAGE
#define RD_K1_NSTAGE 2   // TMA input stages: rows are fetched NSTAGE - 1 steps ahead (3, 4, 6 measured slower)
#endif
constexpr int NSTAGE = RD_K1_NSTAGE;
#ifndef RD_K1_LOCALSYNC
#define RD_K1_LOCALSYNC 1   // phases joined by neighbour-warp mbarriers instead of CTA barriers
#endif
constexpr int KS_NW = KS_COLS / 32;  // warps per CTA
constexpr int TMA_BOX = 128;       // a strip row is KS_COLS / 128 TMA boxes (128-byte aligned destinations)
#ifndef RD_K1_TMA_TID
#define RD_K1_TMA_TID (KS_COLS - 1)   // the issuing thread: a right-halo column (no ridge output)
#endif
constexpr int TMA_TID = RD_K1_TMA_TID;
static_assert(KS_COLS % TMA_BOX == 0, "strip rows are whole TMA boxes");

template <int RB>
struct K1SSmem {                       // dynamic shared memory of k_ridges2 (128-byte aligned base)
  alignas(128) uint16_t sIn[NSTAGE][RB][KS_COLS];   // TMA: input rows of NSTAGE steps (uint8 frames: rows
                                                    // of KS_COLS bytes at the same row offsets)
  uint64_t bar[NSTAGE];                // TMA: one mbarrier per input stage (full)
  uint64_t empty[NSTAGE];              // TMA: every thread has copied the stage out (local sync)
  uint64_t nbar[3][KS_NW];             // local sync: phase boundary x of warp w, arrived on by
                                       // the threads of warps w - 1, w, w + 1
  double2 sD[RB + 2][KS_COLS];         // ring of unnormalised directions v (x = NaN: no candidate)
  double sK[RB + 2][KS_COLS];          // kappa ring
  double sG[RB][KS_COLS];              // G rows
  int sI[KS_COLS][RB];                 // input rows (as int), a column's RB rows adjacent
  unsigned sBal[2][RB][KS_COLS / 32];  // ridge ballots of a step's rows, by parity
  int sCur[KS_NB];                     // ridges so far in the current row of each bin
};
}  // namespace

// Input rows reach shared memory either by TMA (TMA = true: cp.async.bulk.tensor of each row's
// two 192-pixel boxes into a ring of NSTAGE stages, issued by one thread NSTAGE - 1 steps ahead
// and completed on the stage's mbarrier; rows outside the frame are fetched at the clamped row,
// columns outside it arrive as zeros and are read at the clamped column: replicate border) or
// by per-thread loads prefetched one step ahead in registers (frames whose address or pitch is
// not 16-byte aligned).
template <typename PixT, int KS, int RB, bool EDGE, bool TMA>
__global__ void __launch_bounds__(KS_COLS, RD_K1_MINB)
k_ridges2(const uint8_t* __restrict__ frames, int64_t pitch, int64_t fstride, int seg_rows, Params P,
          const __grid_constant__ CUtensorMap tmap) {
  constexpr int NTAP = 2 * KS + 1;
  constexpr int NR = RB + 2;        // kappa / rho ring rows
  extern __shared__ __align__(128) unsigned char smem_raw[];
  K1SSmem<RB>& S = *reinterpret_cast<K1SSmem<RB>*>(smem_raw);
  auto& sD = S.sD;
  auto& sK = S.sK;
  auto& sG = S.sG;
  auto& sI = S.sI;
  auto& sBal = S.sBal;
  auto& sCur = S.sCur;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int W = P.W, H = P.H;
  const int f = blockIdx.z;
  const int X0 = blockIdx.x * KS_OUT;                 // first output column of the strip
  const int Y0 = blockIdx.y * seg_rows;               // first output row of the segment
  const int Y1 = min(Y0 + seg_rows, H);               // one past the last output row
  const int x = X0 - KS_HALO + tid;                   // this thread's column
  const int xc = min(max(x, 0), W - 1);               // clamped (replicate border)
  const uint8_t* frame = frames + (int64_t)f * fstride;
  const int* q = P.q;   // taps stay in the constant bank
  const double t_int = P.t_int, t_edge2 = P.t_edge2;
  constexpr bool edge = EDGE;   // directed edges (NEXT-2) instead of ridges, a separate instance
  // which columns compute what: R on [KS, 256-KS), G..H on [13, 243), output on [16, 240)
  const bool doR = tid >= KS && tid < KS_COLS - KS;
  const bool doH = tid >= KS_HALO - 3 && tid < KS_COLS - KS_HALO + 3;
  const bool outc = tid >= KS_HALO && tid < KS_COLS - KS_HALO && x < W;
  const bool colH = doH && x >= 2 && x <= W - 3;      // Hessian valid in this column
  const bool colR = outc && x >= 3 && x <= W - 4;     // ridge candidates in this column

  // Rows, relative to the input row yi of a phase row: G row yi - KS, kappa row yi - KS - 2,
  // ridge row yi - KS - 3.  The first G needed is row Y0 - 3 (kappa row Y0 - 1 needs H rows
  // Y0 - 3 .. Y0 + 1), so input starts at Y0 - 3 - KS.  Ring slots are (row - ybase) mod NR.
  const int ys0 = Y0 - 3 - KS;
  const int ybase = ys0 - KS - 8 * NR;                // <= every ring row, keeps the mod positive
  const int n_rows = (Y1 - 1) + KS + 3 - ys0 + 1;     // input rows through ridge row Y1 - 1
  const int n_steps = (n_rows + RB - 1) / RB;

  uint32_t wR[NTAP];               // R rows yi - 2KS .. yi (this column; R < 2^31)
  double wA[5], wB[5], wC[5];      // HA, HB, HC rows yg - 4 .. yg
#pragma unroll
  for (int j = 0; j < NTAP; ++j) wR[j] = 0u;
#pragma unroll
  for (int j = 0; j < 5; ++j) wA[j] = wB[j] = wC[j] = 0.0;
  // input prefetch: the next step's RB rows (registers), or the first NSTAGE - 1 steps (TMA)
  PixT pf[RB];
  const int xs = xc - (X0 - KS_HALO);   // this thread's clamped column inside a TMA row
  auto tma_issue = [&](int stp) {       // one thread: the RB rows of step stp into stage stp % NSTAGE
    const int sg = stp % NSTAGE;
    // local sync: warps can be steps apart, so the stage's previous step must be copied out by all
    if (RD_K1_LOCALSYNC && stp >= NSTAGE) mbar_wait(&S.empty[sg], (uint32_t)((stp / NSTAGE - 1) & 1));
    fence_proxy_async_smem();           // generic reads of the stage (NSTAGE steps ago) before the async writes
    mbar_expect_tx(&S.bar[sg], (uint32_t)(RB * KS_COLS * sizeof(PixT)));
#pragma unroll
    for (int r = 0; r < RB; ++r) {
      const int yy = min(max(ys0 + stp * RB + r, 0), H - 1);
      PixT* dst = reinterpret_cast<PixT*>(&S.sIn[sg][0][0]) + r * KS_COLS;
#pragma unroll
      for (int b = 0; b < KS_COLS / TMA_BOX; ++b)
        tma_load_3d(dst + b * TMA_BOX, &tmap, &S.bar[sg], X0 - KS_HALO + b * TMA_BOX, yy, f);
    }
  };
  if (tid == 0) {
    for (int i = 0; i < NSTAGE; ++i) {
      mbar_init(&S.bar[i], 1);
      mbar_init(&S.empty[i], KS_COLS);
    }
    for (int x = 0; x < 3; ++x)
      for (int w = 0; w < KS_NW; ++w) mbar_init(&S.nbar[x][w], 32u * (1 + (w > 0) + (w < KS_NW - 1)));
    mbar_fence_init();
  }
  __syncthreads();
  // Phase boundaries (RD_K1_LOCALSYNC): every shared-memory exchange of this kernel is between
  // columns at most K_s + 3 <= 16 apart, i.e. between neighbouring warps (a bin spans two), so a
  // warp waits at a boundary only for warps w - 1 and w + 1 to reach it, not for the whole CTA;
  // a slow warp (many rho candidates) delays its neighbours instead of every warp.  Neighbours
  // stay within one boundary of each other, so one mbarrier per (boundary, warp) suffices.
  auto phase_sync = [&](int x, int st) {
    if (RD_K1_LOCALSYNC) {
      if (warp > 0) mbar_arrive(&S.nbar[x][warp - 1]);
      mbar_arrive(&S.nbar[x][warp]);
      if (warp < KS_NW - 1) mbar_arrive(&S.nbar[x][warp + 1]);
      mbar_wait(&S.nbar[x][warp], (uint32_t)(st & 1));
    } else {
      __syncthreads();
    }
  };
  if (TMA) {
    if (tid == TMA_TID)
      for (int i = 0; i < NSTAGE - 1 && i < n_steps; ++i) tma_issue(i);
  } else {
#pragma unroll
    for (int r = 0; r < RB; ++r) {
      const int yy = min(max(ys0 + r, 0), H - 1);
      pf[r] = reinterpret_cast<const PixT*>(frame + (int64_t)yy * pitch)[xc];
    }
  }
  // bin output: bin b of the strip covers threads 16 + 32b .. 47 + 32b (upper half of warp b,
  // lower half of warp b + 1).  A step's ridges are written in the next step, once both
  // halves' ballots are in shared memory, so every bin keeps row-major order.
  const int b_own = (tid - KS_HALO) >> 5, b_i = (tid - KS_HALO) & 31;   // bin and index in it
  const int64_t fbase = (int64_t)f * P.nbx * P.nby;
  if (b_own >= 0 && b_own < KS_NB && b_i == 0) sCur[b_own] = 0;   // (by its writer: local sync)
  unsigned rd_bits = 0;            // ridge flags of the previous step's RB test rows
  int rd_y0 = 0;                   // first test row of the previous step
  bool rd_any = false;             // the previous step tested rows of this segment
  int rd_cur = 0;                  // the bin cursor after the emitted rows

  for (int st = 0; st <= n_steps; ++st) {   // the extra step only emits the last rows
    const int yi0 = ys0 + st * RB;
    const bool compute = st < n_steps;
    // 1. input rows -> shared memory; prefetch the next step's rows
    if (compute && TMA) {
      // the stage of step st + NSTAGE - 1 was last read in step st - 1 (barriers since)
      if (tid == TMA_TID && st + NSTAGE - 1 < n_steps) tma_issue(st + NSTAGE - 1);
      const int sg = st % NSTAGE;
      mbar_wait(&S.bar[sg], (uint32_t)((st / NSTAGE) & 1));
      const PixT* in = reinterpret_cast<const PixT*>(&S.sIn[sg][0][0]);
#pragma unroll
      for (int r = 0; r < RB; ++r) sI[tid][r] = (int)in[r * KS_COLS + xs];
      if (RD_K1_LOCALSYNC) mbar_arrive(&S.empty[sg]);
    } else if (compute) {
#pragma unroll
      for (int r = 0; r < RB; ++r) {
        sI[tid][r] = (int)pf[r];
        const int yy = min(max(yi0 + RB + r, 0), H - 1);
        pf[r] = reinterpret_cast<const PixT*>(frame + (int64_t)yy * pitch)[xc];
      }
    }
    phase_sync(0, st);
    // ridges of the previous step's test rows (ballots of parity (st - 1) & 1): slots follow
    // from the bin cursor and the popcounts of earlier rows, so no shared state changes here
    const bool in_bin = b_own >= 0 && b_own < KS_NB;
    if (rd_any && in_bin) {
      const int p = (st - 1) & 1;
      int base = sCur[b_own];
#pragma unroll
      for (int r = 0; r < RB; ++r) {
        const int yr = rd_y0 + r;
        if (yr < Y0 || yr >= Y1) continue;   // uniform across the CTA
        const unsigned m = (sBal[p][r][b_own] >> 16) | (sBal[p][r][b_own + 1] << 16);
        if ((rd_bits >> r) & 1u) {
          const int slot = base + __popc(m & ((1u << b_i) - 1u));
          const int64_t bin = fbase + (int64_t)(yr / T1) * P.nbx + X0 / T1 + b_own;
          RD_CHECK(X0 / T1 + b_own < P.nbx && yr / T1 < P.nby && x < P.W, CK_K1_BIN);
          if (slot < P.ridge_cap) {
            const int64_t o = bin * P.ridge_cap + slot;
            P.bin_xy[o] = (uint32_t)x | ((uint32_t)yr << 16);
            P.bin_d[o] = sD[(yr - ybase) % NR][tid];
          }
        }
        base += __popc(m);
        if ((yr & (T1 - 1)) == T1 - 1 || yr == Y1 - 1) {   // the bin row is complete
          const int bx = X0 / T1 + b_own;
          if (b_i == 0 && bx < P.nbx) {
            const int64_t bin = fbase + (int64_t)(yr / T1) * P.nbx + bx;
            P.bin_count[bin] = base;   // the true count (readers clamp to ridge_cap; K1.5 reports the need)
            if (base > P.ridge_cap) atomicOr(&P.flags[f], OVF_RIDGES);
            if (base) atomicAdd(&P.stats[f].ridges, (unsigned long long)base);
          }
          base = 0;
        }
      }
      rd_cur = base;   // the bin owner stores it after the next barrier
    }
    if (!compute) break;
    // 2. row passes R(yi) (int32 exact) -> column window; G(yg) (fp64 exact), RB rows
    int accr[RB];   // R of the RB rows: one (vector) load per tap serves all of them
#pragma unroll
    for (int r = 0; r < RB; ++r) accr[r] = 0;
    if (doR) {
#pragma unroll
      for (int j = 0; j < NTAP; ++j) {
        const int* col = sI[tid - KS + j];
        if constexpr (RB == 2) {
          const int2 v = *reinterpret_cast<const int2*>(col);
          accr[0] += q[j] * v.x;
          accr[1] += q[j] * v.y;
        } else if constexpr (RB == 4) {
          const int4 v = *reinterpret_cast<const int4*>(col);
          accr[0] += q[j] * v.x;
          accr[1] += q[j] * v.y;
          accr[2] += q[j] * v.z;
          accr[3] += q[j] * v.w;
        } else {
#pragma unroll
          for (int r = 0; r < RB; ++r) accr[r] += q[j] * col[r];
        }
      }
    }
#pragma unroll
    for (int r = 0; r < RB; ++r) {
#pragma unroll
      for (int j = 0; j < NTAP - 1; ++j) wR[j] = wR[j + 1];
      wR[NTAP - 1] = (uint32_t)accr[r];
      // G = sum q_j R_j < 2^53 in 64-bit integers (symmetric taps), then exactly to fp64
      unsigned long long g = (unsigned long long)(uint32_t)q[KS] * wR[KS];
#pragma unroll
      for (int j = 0; j < KS; ++j) g += (unsigned long long)(uint32_t)q[j] * (unsigned long long)(wR[j] + wR[NTAP - 1 - j]);
      sG[r][tid] = (double)g;
    }
    phase_sync(1, st);
    if (rd_any && in_bin && b_i == 0) sCur[b_own] = rd_cur;
    // 3. horizontal Sobel passes, vertical windows, kappa and rho of the kappa rows, RB rows
#pragma unroll
    for (int r = 0; r < RB; ++r) {
      const int yk = yi0 + r - KS - 2;
      double ha = 0.0, hb = 0.0, hc = 0.0;
      if (doH) {
        const double g0 = sG[r][tid - 2], g1 = sG[r][tid - 1], g2 = sG[r][tid], g3 = sG[r][tid + 1],
                     g4 = sG[r][tid + 2];
        ha = (g0 + g4) - 2.0 * g2;                       // d2 = [1,0,-2,0,1]
        hb = (g0 + g4) + 4.0 * (g1 + g3) + 6.0 * g2;     // s5 = [1,4,6,4,1]
        hc = (g4 - g0) + 2.0 * (g3 - g1);                // d1 = [-1,-2,0,2,1]
      }
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        wA[j] = wA[j + 1];
        wB[j] = wB[j + 1];
        wC[j] = wC[j + 1];
      }
      wA[4] = ha;
      wB[4] = hb;
      wC[4] = hc;
      double kap = edge ? 0.0 : HUGE_VAL;
      double2 dir = make_double2(NOT_CAND, 0.0);
      if (colH && yk >= 2 && yk <= H - 3) {
        if (!edge) {
          const double Ixx = (wA[0] + wA[4]) + 4.0 * (wA[1] + wA[3]) + 6.0 * wA[2];
          const double Iyy = (wB[0] + wB[4]) - 2.0 * wB[2];
          const double Ixy = (wC[4] - wC[0]) + 2.0 * (wC[3] - wC[1]);
          double sq, e;
          kap = kappa_of(Ixx, Ixy, Iyy, &sq, &e);
          double dx, dy;
          // R3; the direction stays unnormalised here (K1.5 divides by its norm)
          if (kap < t_int && direction_raw(Ixy, e, sq, &dx, &dy)) dir = make_double2(dx, dy);
        } else {   // edge variant (NEXT-2, R19): Ix = s5_y (x) d1_x, Iy = d1_y (x) s5_x, m2 = |grad|^2
          const double Ix = (wC[0] + wC[4]) + 4.0 * (wC[1] + wC[3]) + 6.0 * wC[2];
          const double Iy = (wB[4] - wB[0]) + 2.0 * (wB[3] - wB[1]);
          kap = __dadd_rn(__dmul_rn(Ix, Ix), __dmul_rn(Iy, Iy));
          if (kap > t_edge2) dir = make_double2(Ix, Iy);   // n = sqrt(kap) divides in K1.5
        }
      }
      const int slot = (yk - ybase) % NR;
      sK[slot][tid] = kap;
      sD[slot][tid] = dir;
    }
    phase_sync(2, st);
    // 4. ridge tests of the rows one behind the kappa rows (R6)
    rd_bits = 0;
    rd_y0 = yi0 - KS - 3;
    rd_any = false;
#pragma unroll
    for (int r = 0; r < RB; ++r) {
      const int yr = rd_y0 + r;
      bool is_r = false;
      if (colR && yr >= Y0 && yr < Y1 && yr >= 3 && yr <= H - 4) {
        const int s0 = (yr - ybase) % NR, sm = (yr - 1 - ybase) % NR, sp = (yr + 1 - ybase) % NR;
        const double2 dir = sD[s0][tid];
        if (dir.x == dir.x) {   // a candidate (not NaN)
          const double kp = sK[s0][tid];
          int ox, oy;   // llround of rho's components
          dir_step(dir.x, dir.y, &ox, &oy);
          const bool after_plus = (oy > 0) || (oy == 0 && ox > 0);
          const double kplus = sK[oy > 0 ? sp : (oy < 0 ? sm : s0)][tid + ox];
          const double kminus = sK[oy > 0 ? sm : (oy < 0 ? sp : s0)][tid - ox];
          RD_CHECK(tid - ox >= 0 && tid + ox < KS_COLS && ox >= -1 && ox <= 1 && oy >= -1 && oy <= 1, CK_K1_SMEM);
          const double kafter = after_plus ? kplus : kminus, kbefore = after_plus ? kminus : kplus;
          // ridges: kappa a local minimum along rho (R6); edges: |grad|^2 a local maximum (R19)
          is_r = edge ? (kp >= kafter) && (kp > kbefore) : (kp <= kafter) && (kp < kbefore);
        }
      }
      const unsigned bal = __ballot_sync(0xffffffffu, is_r);
      if (lane == 0) sBal[st & 1][r][warp] = bal;
      rd_bits |= (unsigned)is_r << r;
      rd_any |= yr >= Y0 && yr < Y1;
    }
  }
}

namespace {
PFN_cuTensorMapEncodeTiled_v12000 g_encode = nullptr;

// 3-D tensor map (x, y, frame) of the caller's frames with boxes of TMA_BOX x 1 x 1 pixels;
// false if TMA cannot address them (16-byte alignment of base, pitch and frame stride)
bool make_tmap(CUtensorMap* map, const void* frames, int pb, int W, int H, int n, int64_t pitch, int64_t fstride) {
  if (!g_encode) {
    cudaDriverEntryPointQueryResult q;
    void* fn = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess || !fn)
      return false;
    g_encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  }
  if (((uintptr_t)frames & 15) || (pitch & 15) || (n > 1 && (fstride & 15))) return false;
  cuuint64_t dims[3] = {(cuuint64_t)W, (cuuint64_t)H, (cuuint64_t)n};
  cuuint64_t strides[2] = {(cuuint64_t)pitch, (cuuint64_t)(n > 1 ? fstride : pitch * H)};
  cuuint32_t box[3] = {(cuuint32_t)TMA_BOX, 1, 1};
  cuuint32_t es[3] = {1, 1, 1};
  return g_encode(map, pb == 1 ? CU_TENSOR_MAP_DATA_TYPE_UINT8 : CU_TENSOR_MAP_DATA_TYPE_UINT16, 3,
                  const_cast<void*>(frames), dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                  CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}
}  // namespace

template <typename PixT, int KS, bool EDGE>
static cudaError_t launch_s(const void* frames, int64_t pitch, int64_t fstride, int n_frames, const Params& P,
                            cudaStream_t st) {
  constexpr int RB = RD_K1_RB;
  // dynamic shared memory: rings + rows (NR = RB + 2 rows of rho and kappa) + TMA stages
  const size_t sm = sizeof(K1SSmem<RB>);
  CUtensorMap tmap;
  static const bool no_tma = getenv("RD_K1_NO_TMA") != nullptr;   // A/B: per-thread loads
  const bool tma = !no_tma && make_tmap(&tmap, frames, (int)sizeof(PixT), P.W, P.H, n_frames, pitch, fstride);
  if (!tma) memset(&tmap, 0, sizeof tmap);
  cudaFuncSetAttribute(k_ridges2<PixT, KS, RB, EDGE, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  cudaFuncSetAttribute(k_ridges2<PixT, KS, RB, EDGE, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  // segments of whole bin rows: the count that best fills the resident CTA slots (P.k1_slots,
  // from rd_create), each segment paying 3K_s + 6 rows of pipeline warm-up
  const int slots = std::max(1, P.k1_slots);
  const int strips = (P.W + KS_OUT - 1) / KS_OUT, bin_rows = (P.H + T1 - 1) / T1;
  int seg = bin_rows * T1;
  double best = -1.0;
  for (int nseg = 1; nseg <= std::min(bin_rows, 8); ++nseg) {
    const int sr = (bin_rows + nseg - 1) / nseg * T1;            // rows per segment
    const int ns = (P.H + sr - 1) / sr;
    // concurrent parts of a batch share the SMs: each sees its share of the CTA slots
    const double ctas = (double)strips * ns * n_frames, waves = ctas / (slots / (double)std::max(1, P.parts));
    const double eff = waves / std::ceil(waves) * (double)P.H / (P.H + ns * (3.0 * KS + 6.0));
    if (eff > best + 1e-9) {
      best = eff;
      seg = sr;
    }
  }
  if (const char* env = getenv("RD_K1_NSEG")) {   // A/B: a fixed number of row segments
    const int ns = std::max(1, std::min(bin_rows, atoi(env)));
    seg = (bin_rows + ns - 1) / ns * T1;
  }
  dim3 grid(strips, (P.H + seg - 1) / seg, n_frames);
  if (tma)
    k_ridges2<PixT, KS, RB, EDGE, true><<<grid, KS_COLS, sm, st>>>((const uint8_t*)frames, pitch, fstride, seg, P, tmap);
  else
    k_ridges2<PixT, KS, RB, EDGE, false><<<grid, KS_COLS, sm, st>>>((const uint8_t*)frames, pitch, fstride, seg, P, tmap);
  return cudaGetLastError();
}

template <typename PixT, bool EDGE>
static cudaError_t launch_sp(const void* frames, int64_t pitch, int64_t fstride, int n, const Params& P,
                             cudaStream_t st) {
  switch (P.Ks) {
    case 1: return launch_s<PixT, 1, EDGE>(frames, pitch, fstride, n, P, st);
    case 2: return launch_s<PixT, 2, EDGE>(frames, pitch, fstride, n, P, st);
    case 3: return launch_s<PixT, 3, EDGE>(frames, pitch, fstride, n, P, st);
    case 4: return launch_s<PixT, 4, EDGE>(frames, pitch, fstride, n, P, st);
    case 5: return launch_s<PixT, 5, EDGE>(frames, pitch, fstride, n, P, st);
    case 6: return launch_s<PixT, 6, EDGE>(frames, pitch, fstride, n, P, st);
    case 7: return launch_s<PixT, 7, EDGE>(frames, pitch, fstride, n, P, st);
    case 8: return launch_s<PixT, 8, EDGE>(frames, pitch, fstride, n, P, st);
    case 9: return launch_s<PixT, 9, EDGE>(frames, pitch, fstride, n, P, st);
    case 10: return launch_s<PixT, 10, EDGE>(frames, pitch, fstride, n, P, st);
    case 11: return launch_s<PixT, 11, EDGE>(frames, pitch, fstride, n, P, st);
    case 12: return launch_s<PixT, 12, EDGE>(frames, pitch, fstride, n, P, st);
    case 13: return launch_s<PixT, 13, EDGE>(frames, pitch, fstride, n, P, st);
  }
  return cudaErrorInvalidValue;
}

static_assert(KS_MAX <= KS_HALO - 3, "the 16-column halo covers K_s + 3");

size_t k_ridges_smem(int) { return sizeof(K1SSmem<RD_K1_RB>); }

// resident K1 CTAs per device (all K1 instances share the launch bounds and shared memory)
int k_ridges_slots(int n_sm) {
  int per = 0;
  const size_t sm = sizeof(K1SSmem<RD_K1_RB>);
  cudaFuncSetAttribute(k_ridges2<uint16_t, 5, RD_K1_RB, false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       (int)sm);
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_ridges2<uint16_t, 5, RD_K1_RB, false, true>, KS_COLS, sm) !=
      cudaSuccess)
    per = 1;
  return std::max(1, n_sm * std::max(per, 1));
}

cudaError_t launch_ridges(const void* frames, int64_t pitch, int64_t fstride, int n_frames, const Params& P,
                          cudaStream_t st) {
  if (P.Ks < 1 || P.Ks > KS_MAX) return cudaErrorInvalidValue;
  if (P.feature == 1)
    return P.pixel_bytes == 1 ? launch_sp<uint8_t, true>(frames, pitch, fstride, n_frames, P, st)
                              : launch_sp<uint16_t, true>(frames, pitch, fstride, n_frames, P, st);
  return P.pixel_bytes == 1 ? launch_sp<uint8_t, false>(frames, pitch, fstride, n_frames, P, st)
                            : launch_sp<uint16_t, false>(frames, pitch, fstride, n_frames, P, st);
}

// A3 in isolation (rd_eigen): the same recipe on caller-supplied Hessians.
__global__ void k_eigen(const double* __restrict__ abc, int64_t n, double* __restrict__ out, int* __restrict__ deg) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double a = abc[3 * i], b = abc[3 * i + 1], c = abc[3 * i + 2];
  double s, e;
  const double k = kappa_of(a, b, c, &s, &e);
  // the product's split of the recipe: K1 keeps v unnormalised and takes the ridge test's
  // neighbour step from dir_step; K1.5 normalises
  double vx, vy, dx = 0.0, dy = 0.0;
  int ox = 0, oy = 0;
  const bool ok = direction_raw(b, e, s, &vx, &vy);
  if (ok) {
    normalise_dir(vx, vy, &dx, &dy);
    dir_step(vx, vy, &ox, &oy);
  }
  out[3 * i] = k;
  out[3 * i + 1] = dx;
  out[3 * i + 2] = dy;
  deg[i] = (ok ? 0 : 1) | ((ox + 1) << 1) | ((oy + 1) << 3);
}

cudaError_t launch_eigen(const double* abc, int64_t n, double* out, int* deg, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  k_eigen<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(abc, n, out, deg);
  return cudaGetLastError();
}

}  // namespace rd
