// k_hough.cu — K2: directed voting, hotspot registration, radius-dependent smoothing
// with 1/r normalisation and 3x3x3 peak extraction, one CTA per (frame, T x T tile).
//
// Rows A5-A8 of DESIGN.md §2 (SI steps 2-4, PAPER.md:931-978;
// range extension PAPER.md:998-1001).  The CTA owns the accumulator cells of its tile and
// sweeps r upward through the Hough range G levels at a time, keeping on chip:
//   raw(r..r+G-1) — G levels of packed uint16 counters over tile + (K_r + 1) halo, filled
//                  with shared-memory atomics;
//   hotspot lists (cell, raw, S) and candidate lists of the last G + 2 levels — the
//                  paper's rolling level window, 3 levels -> G + 2.
// Voting rays (a ridge pixel, a sense of rho and the level interval in which its votes can
// land in the tile's level boxes) are gathered once per CTA.  Each G-level step compacts
// the rays active in it; the (ray, level) pairs of the step are dealt evenly to the threads
// and processed four at a time (independent targets, then independent atomics).
// A hotspot is registered by the one atomic that lifts its counter past T_raw (the paper's
// "surpassed" test at increment time).  S is computed for hotspots only,
// a sub-warp per hotspot with lanes over window rows.  NMS of a level runs once the level
// above is complete, one warp per candidate scanning three neighbouring
// lists.  Counters are cleared by undoing exactly the cells this CTA incremented (the
// paper's register-and-undo).  Only peak records (and optional debug
// hotspots) leave the SM.
#include "rd_internal.cuh"

namespace rd {

namespace {
#ifndef RD_K2_BATCH
#define RD_K2_BATCH 4
#endif
constexpr int BATCH = RD_K2_BATCH;   // (ray, level) pairs in flight per thread

struct K2Smem {
  int raws, rawp, lvlc;           // raw side, row pitch, cells per level (multiple of 8; uint16 units)
  size_t off_hS, off_ed, off_raw, off_exy, off_err, off_act, off_hcell, off_hraw, off_task, off_ccur, off_cdef,
      off_hcnt, off_w, off_k, off_tn, off_box, total;
};

__host__ __device__ inline size_t align16(size_t v) { return (v + 15) & ~size_t(15); }

__host__ __device__ inline K2Smem k2_layout(int G, int T, int hal, int entry_cap, int hot_cap, int n_levels,
                                            int wstride) {
  const int NSLOT = G + 2;
  K2Smem L;
  L.raws = T + 2 * hal;
  // row pitch with an odd number of 32-bit words: the rows of a window fall in distinct banks
  L.rawp = ((L.raws / 2) & 1) ? L.raws : L.raws + 2;
  size_t o = 0;
  L.off_hS = o;    o = align16(o + sizeof(unsigned long long) * NSLOT * hot_cap);
  L.off_ed = o;    o = align16(o + sizeof(double2) * entry_cap);
  L.lvlc = (L.raws * L.rawp + 7) & ~7;   // 16-byte aligned level buffers (bulk clears)
  L.off_raw = o;   o = align16(o + 2 * (size_t)G * L.lvlc);
  L.off_exy = o;   o = align16(o + 4 * (size_t)entry_cap);
  L.off_err = o;   o = align16(o + 4 * (size_t)entry_cap);
  L.off_act = o;   o = align16(o + 2 * (size_t)entry_cap);
  L.off_hcell = o; o = align16(o + 2 * (size_t)NSLOT * hot_cap);
  L.off_hraw = o;  o = align16(o + 2 * (size_t)NSLOT * hot_cap);
  L.off_task = o;  o = align16(o + 2 * (size_t)G * hot_cap);         // step's hotspots (g << 12 | h)
  L.off_ccur = o;  o = align16(o + 2 * (size_t)G * hot_cap);         // step's candidates below Lhi
  L.off_cdef = o;  o = align16(o + 2 * (size_t)2 * hot_cap);         // candidates of Lhi, by parity
  L.off_hcnt = o;  o = align16(o + 4 * (size_t)(n_levels + G + 16));
  L.off_w = o;     o = align16(o + 4 * (size_t)n_levels * wstride);   // level tables, resident
  L.off_k = o;     o = align16(o + 4 * (size_t)n_levels);
  L.off_tn = o;    o = align16(o + 8 * (size_t)n_levels);
  L.off_box = o;   o = align16(o + 16 * (size_t)G);
  L.total = o;
  return L;
}

}  // namespace

template <bool kWide, int G, int MINB>
__global__ void __launch_bounds__(512, MINB) k_hough(Params P) {
  constexpr int NSLOT = G + 2;
  constexpr int LG = G == 8 ? 3 : G == 4 ? 2 : 1;
  static_assert((1 << LG) == G, "G must be a power of two");
  extern __shared__ __align__(16) unsigned char smem[];
  const int T = P.k2t;
  const int RING = T + 2;          // tile + 1 ring side (hotspot registration region)
  const K2Smem L = k2_layout(G, T, P.hal, P.entry_cap, P.hot_cap, P.n_levels, P.wstride);
  unsigned long long* hS = reinterpret_cast<unsigned long long*>(smem + L.off_hS);  // [NSLOT][hot_cap]
  double2* eD = reinterpret_cast<double2*>(smem + L.off_ed);             // [entry_cap] (s*dx, s*dy)
  uint32_t* raw32 = reinterpret_cast<uint32_t*>(smem + L.off_raw);       // [G] packed uint16 levels
  uint16_t* raw16 = reinterpret_cast<uint16_t*>(smem + L.off_raw);
  uint32_t* eXY = reinterpret_cast<uint32_t*>(smem + L.off_exy);         // [entry_cap] x | y<<16
  uint32_t* eR = reinterpret_cast<uint32_t*>(smem + L.off_err);          // [entry_cap] ra | rb<<16 (level idx)
  uint16_t* act = reinterpret_cast<uint16_t*>(smem + L.off_act);         // active entries of the step
  uint16_t* hcell = reinterpret_cast<uint16_t*>(smem + L.off_hcell);     // [NSLOT][hot_cap] ring-local cell
  uint16_t* hraw = reinterpret_cast<uint16_t*>(smem + L.off_hraw);       // [NSLOT][hot_cap]
  uint16_t* tasks = reinterpret_cast<uint16_t*>(smem + L.off_task);     // [G*hot_cap] step hotspots
  uint16_t* ccur = reinterpret_cast<uint16_t*>(smem + L.off_ccur);       // [G*hot_cap] step candidates
  uint16_t* cdef = reinterpret_cast<uint16_t*>(smem + L.off_cdef);       // [2][hot_cap] deferred candidates
  int* hcnt = reinterpret_cast<int*>(smem + L.off_hcnt);                 // [n_levels + G] + misc
  int* tW = reinterpret_cast<int*>(smem + L.off_w);                      // [n_levels][wstride] w_r(d)
  int* tK = reinterpret_cast<int*>(smem + L.off_k);                      // [n_levels] K_r
  double* tTn = reinterpret_cast<double*>(smem + L.off_tn);              // [n_levels] T_norm(r)
  int4* box = reinterpret_cast<int4*>(smem + L.off_box);                 // [G] vote box per level
  int* s_ecnt = hcnt + P.n_levels + G;
  int* s_flags = s_ecnt + 1;
  int* s_nact = s_ecnt + 2;                                              // [2], by step parity
  int* s_ntask = s_ecnt + 4;                                             // [2], by step parity
  int* s_ndef = s_ecnt + 6;                                              // [2], by step parity
  int* s_ncur = s_ecnt + 8;                                              // [1]

  const int NT = blockDim.x, NW = NT >> 5;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int f = blockIdx.y;
  const int tile = blockIdx.x;
  const int tyi = tile / P.ntx, txi = tile - tyi * P.ntx;
  const int X0 = txi * T, Y0 = tyi * T;
  const int W = P.W, H = P.H, hal = P.hal;
  const int RX0 = X0 - hal, RY0 = Y0 - hal;   // raw buffer origin
  const int rawp = L.rawp;
  const int lvl_cells = L.lvlc;              // uint16 cells per raw level (16-byte multiple)
  const int hot_cap = P.hot_cap, nlev = P.n_levels;
  const int rlo = P.r_lo;

  // optional per-phase cycle accounting (thread 0, after each barrier; rd_phase_cycles)
  unsigned long long t_acc[6] = {0, 0, 0, 0, 0, 0};
  long long t_last = clock64();
#define PMARK(i)                                      \
  if (P.prof && tid == 0) {                           \
    const long long t_ = clock64();                   \
    t_acc[i] += (unsigned long long)(t_ - t_last);    \
    t_last = t_;                                      \
  }
  for (int i = tid; i < nlev + G + 16; i += NT) hcnt[i] = 0;
  for (int i = tid; i < nlev * P.wstride; i += NT) tW[i] = P.lvlW[i];
  for (int i = tid; i < nlev; i += NT) {
    tK[i] = P.lvlK[i];
    tTn[i] = P.lvlTn[i];
  }
  {  // zero all raw levels once; afterwards cells are restored to zero by undo
    uint4* r4 = reinterpret_cast<uint4*>(raw32);
    const int n4 = (G * lvl_cells) / 8;
    for (int i = tid; i < n4; i += NT) r4[i] = make_uint4(0, 0, 0, 0);
    for (int i = n4 * 8 + tid; i < G * lvl_cells; i += NT) raw16[i] = 0;
  }
  __syncthreads();

  // ---------------- phase 0: this tile's voting rays, routed by K1.5 (k_rays.cu)
  const int64_t tl = (int64_t)f * P.ntx * P.nty + tile;
  const int ne = min(P.ray_count[tl], P.entry_cap);
  {
    const double2* gd = P.ray_d + tl * P.entry_cap;
    const uint32_t* gxy = P.ray_xy + tl * P.entry_cap;
    const uint32_t* gr = P.ray_r + tl * P.entry_cap;
    for (int e = tid; e < ne; e += NT) {
      eD[e] = gd[e];
      eXY[e] = gxy[e];
      eR[e] = gr[e];
    }
  }
  __syncthreads();
  PMARK(0);
  int my_votes = 0, my_hot = 0;
  const uint32_t T_raw = (uint32_t)P.T_raw;

  // per-step setup: level boxes and the compacted active rays (into the parity counter)
  auto setup = [&](int L0s) {
    const int Lhs = min(L0s + G - 1, nlev - 1);
    if (tid < G) {
      const int K = (L0s + tid < nlev) ? tK[L0s + tid] : 0;
      box[tid] = make_int4(max(X0 - K - 1, 0), min(X0 + T + K, W - 1), max(Y0 - K - 1, 0), min(Y0 + T + K, H - 1));
    }
    int* cnt = s_nact + ((L0s >> LG) & 1);
    for (int e0 = 0; e0 < ne; e0 += NT) {
      const int e = e0 + tid;
      bool a = false;
      if (e < ne) {
        const uint32_t rr = eR[e];
        a = (int)(rr & 0xFFFFu) <= Lhs && (int)(rr >> 16) >= L0s;
      }
      const unsigned bal = __ballot_sync(0xffffffffu, a);
      int base = 0;
      if (lane == 0 && bal) base = atomicAdd(cnt, __popc(bal));
      base = __shfl_sync(0xffffffffu, base, 0);
      if (a) act[base + __popc(bal & ((1u << lane) - 1u))] = (uint16_t)e;
    }
  };
  setup(0);
  __syncthreads();
  PMARK(1);

  // target cell of pair (ray e, level L0+g) in the raw buffers, or -1 (not in the level box)
  auto target = [&](int e, int g, int L0s, int& tx, int& ty) -> int {
    const uint32_t rr = eR[e];
    const int li = L0s + g;
    if (li < (int)(rr & 0xFFFFu) || li > (int)(rr >> 16)) return -1;
    const double2 d = eD[e];
    const uint32_t xy = eXY[e];
    const double rd = (double)(rlo + li);
    tx = (int)(xy & 0xFFFFu) + (int)llround(__dmul_rn(rd, d.x));
    ty = (int)(xy >> 16) + (int)llround(__dmul_rn(rd, d.y));
    const int4 bb = box[g];
    if (tx < bb.x || tx > bb.y || ty < bb.z || ty > bb.w) return -1;
    return g * lvl_cells + (ty - RY0) * rawp + (tx - RX0);
  };

  // ---------------- level sweep, G levels per step
  for (int L0 = 0; L0 < nlev; L0 += G) {
    const int Lhi = min(L0 + G - 1, nlev - 1);
    const int par = (L0 >> LG) & 1;
    const int npair = s_nact[par] << LG;   // (active ray, level) pairs, ray-major
    if (tid == 0) {   // counters first written in (c0) of this step (last read a barrier ago)
      s_ncur[0] = 0;
      s_ndef[par] = 0;
    }
    // (a) votes of levels L0..Lhi
    for (int p0 = tid; p0 < npair; p0 += BATCH * NT) {
      int cell[BATCH], txs[BATCH], tys[BATCH];
      uint32_t old[BATCH];
#pragma unroll
      for (int k = 0; k < BATCH; ++k) {
        const int p = p0 + k * NT;
        cell[k] = p < npair ? target(act[p >> LG], p & (G - 1), L0, txs[k], tys[k]) : -1;
      }
#pragma unroll
      for (int k = 0; k < BATCH; ++k)
#ifdef RD_K2_EXPERIMENT_NORET   // timing experiment only: wrong hotspot registration
        if (cell[k] >= 0) { atomicAdd(&raw32[cell[k] >> 1], 1u << ((cell[k] & 1) << 4)); old[k] = 0; }
#else
        if (cell[k] >= 0) old[k] = atomicAdd(&raw32[cell[k] >> 1], 1u << ((cell[k] & 1) << 4));
#endif
#pragma unroll
      for (int k = 0; k < BATCH; ++k) {
        if (cell[k] < 0) continue;
        const int tx = txs[k], ty = tys[k];
        const uint32_t oc = (old[k] >> ((cell[k] & 1) << 4)) & 0xFFFFu;
        if (oc == T_raw) {
          const int ix = tx - (X0 - 1), iy = ty - (Y0 - 1);
          if ((unsigned)ix < (unsigned)RING && (unsigned)iy < (unsigned)RING) {
            const int g = (p0 + k * NT) & (G - 1), li = L0 + g;
            const int h = atomicAdd(&hcnt[li], 1);
            if (h < hot_cap) {
              hcell[(li % NSLOT) * hot_cap + h] = (uint16_t)(iy * RING + ix);
              tasks[atomicAdd(&s_ntask[par], 1)] = (uint16_t)((g << 12) | h);
            } else {
              atomicOr(s_flags, OVF_HOTSPOTS);
            }
          }
        }
        my_votes += ((unsigned)(tx - X0) < (unsigned)T) & ((unsigned)(ty - Y0) < (unsigned)T);
      }
    }
    if (tid == 0) s_nact[par ^ 1] = 0;   // counter of the next step (last read a barrier ago)
    __syncthreads();
    PMARK(2);
    const int ntask = s_ntask[par];
    // (b) S = sum_i w(i) sum_j w(j) raw(y+i, x+j) at each hotspot:
    //     one warp per hotspot, lanes over window rows; integer sums, reduced in-warp
    for (int t = warp; t < ntask; t += NW) {
      const int tk = tasks[t], g = tk >> 12, h = tk & 0xFFF;
      const int li = L0 + g, sl = li % NSLOT;
      const int K = tK[li], R = 2 * K + 1;
      const int* w = tW + li * P.wstride;
      const uint16_t* lvl = raw16 + g * lvl_cells;
      const int c16 = hcell[sl * hot_cap + h];
      const int iy = c16 / RING, ix = c16 - iy * RING;
      const int ly = iy - 1 + hal, lx = ix - 1 + hal;   // raw-local coordinates of the hotspot
      unsigned long long acc = 0;
      for (int row = lane; row < R; row += 32) {
        const uint16_t* rowp = lvl + (ly + row - K) * rawp + lx;
        if (kWide) {
          unsigned long long rs = (unsigned long long)w[0] * rowp[0];
          for (int j = 1; j <= K; ++j) rs += (unsigned long long)w[j] * (uint32_t)(rowp[-j] + rowp[j]);
          acc += rs * (unsigned long long)w[abs(row - K)];
        } else {
          uint32_t rs = (uint32_t)w[0] * rowp[0];
#pragma unroll 4
          for (int j = 1; j <= K; ++j) rs += (uint32_t)w[j] * (uint32_t)(rowp[-j] + rowp[j]);
          acc += (unsigned long long)rs * (unsigned long long)w[abs(row - K)];
        }
      }
      unsigned long long S;
      if (kWide) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
        S = acc;
      } else {   // every lane term < 2^45: split in 24-bit halves, two single-instruction reductions
        const unsigned lo = __reduce_add_sync(0xffffffffu, (unsigned)(acc & 0xFFFFFFull));
        const unsigned hi = __reduce_add_sync(0xffffffffu, (unsigned)(acc >> 24));
        S = ((unsigned long long)hi << 24) + lo;
      }
      if (lane == 0) {
        hS[sl * hot_cap + h] = S;
        hraw[sl * hot_cap + h] = lvl[ly * rawp + lx];
      }
    }
    __syncthreads();
    PMARK(3);
    // (c0) hotspot bookkeeping: interior count, debug records, candidates S > T_norm(r)
    //       for r in [r_min, r_max]; candidates of the top level
    //      of the step wait for the next step (its upper neighbour level is not done yet)
    for (int t = tid; t < ntask; t += NT) {
      const int tk = tasks[t], g = tk >> 12, h = tk & 0xFFF;
      const int li = L0 + g, sl = li % NSLOT;
      const int c16 = hcell[sl * hot_cap + h];
      const int iy = c16 / RING, ix = c16 - iy * RING;
      if (ix < 1 || ix > T || iy < 1 || iy > T) continue;     // interior cells only
      ++my_hot;
      const unsigned long long S = hS[sl * hot_cap + h];
      if (P.debug) {
        int kd = atomicAdd(&P.dbg_count[f], 1);
        if (kd < P.dbg_cap) {
          HotRec rec;
          rec.r = rlo + li; rec.y = Y0 - 1 + iy; rec.x = X0 - 1 + ix; rec.raw = hraw[sl * hot_cap + h];
          rec.S = (long long)S;
          P.dbg_hot[(int64_t)f * P.dbg_cap + kd] = rec;
        } else {
          atomicOr(&P.flags[f], OVF_DEBUG);
        }
      }
      if (li >= 1 && li <= nlev - 2 && (double)(long long)S > tTn[li]) {
        if (li == Lhi) cdef[par * hot_cap + atomicAdd(&s_ndef[par], 1)] = (uint16_t)h;
        else ccur[atomicAdd(&s_ncur[0], 1)] = (uint16_t)tk;
      }
    }
    // (c1) restore the step's counters to zero.  The paper undoes the registered cells
    //     (PAPER.md:426-434); here the rows of each level box are cleared with 16-byte
    //     stores, which costs far fewer instructions than re-walking the votes.
#pragma unroll 1
    for (int g = 0; g < G; ++g) {
      if (L0 + g >= nlev) break;
      const int4 bb = box[g];
      const int s8 = (g * lvl_cells + (bb.z - RY0) * rawp) >> 3;               // align down
      const int e8 = (g * lvl_cells + (bb.w - RY0 + 1) * rawp + 7) >> 3;       // align up
      uint4* r4 = reinterpret_cast<uint4*>(raw16);
      for (int i = s8 + tid; i < e8; i += NT) r4[i] = make_uint4(0u, 0u, 0u, 0u);
    }
    __syncthreads();
    PMARK(4);
    // (d) peaks among the candidates of levels L0-1 (deferred) .. Lhi-1: 3x3x3 maxima of
    //     N = S/r (R14), one warp per candidate; meanwhile the next step's setup
    {
      const int nd = L0 > 0 ? s_ndef[par ^ 1] : 0, nc = s_ncur[0];
      for (int p = warp; p < nd + nc; p += NW) {
        int lc, h;
        if (p < nd) {
          lc = L0 - 1;
          h = cdef[(par ^ 1) * hot_cap + p];
        } else {
          const int tk = ccur[p - nd];
          lc = L0 + (tk >> 12);
          h = tk & 0xFFF;
        }
        const int sc = lc % NSLOT;
        const int c16 = hcell[sc * hot_cap + h];
        const int iy = c16 / RING, ix = c16 - iy * RING;
        const long long S = (long long)hS[sc * hot_cap + h];
        const long long rc = rlo + lc;
        bool beaten = false;
#pragma unroll
        for (int dl = -1; dl <= 1; ++dl) {
          const int l = lc + dl, sl = l % NSLOT;
          const int n = min(hcnt[l], hot_cap);
          const long long ru = rlo + l;
          for (int j = lane; j < n; j += 32) {
            const int u16 = hcell[sl * hot_cap + j];
            const int uy = u16 / RING, ux = u16 - uy * RING;
            const int dy = uy - iy, dx = ux - ix;
            if (dy < -1 || dy > 1 || dx < -1 || dx > 1 || (dl == 0 && dy == 0 && dx == 0)) continue;
            const long long Su = (long long)hS[sl * hot_cap + j];
            const long long lhs = S * ru, rhs = Su * rc;
            const bool v_first = dl > 0 || (dl == 0 && (dy > 0 || (dy == 0 && dx > 0)));
            if (!(lhs > rhs || (lhs == rhs && v_first))) beaten = true;
          }
        }
        if (__any_sync(0xffffffffu, beaten)) continue;
        if (lane == 0) {
          const int kk = atomicAdd(&P.peak_count[f], 1);
          if (kk < P.ring_cap) {
            Peak pk;
            pk.x = X0 - 1 + ix; pk.y = Y0 - 1 + iy; pk.r = (int)rc; pk.raw = hraw[sc * hot_cap + h]; pk.S = S;
            P.peaks[(int64_t)f * P.ring_cap + kk] = pk;
          } else {
            atomicOr(&P.flags[f], OVF_RINGS);
          }
        }
      }
    }
    if (L0 + G < nlev) setup(L0 + G);
    if (tid == 0) s_ntask[par ^ 1] = 0;   // hotspot-task counter of the next step
    __syncthreads();
    PMARK(5);
  }
  if (P.prof && tid == 0) {
#pragma unroll
    for (int i = 0; i < 6; ++i) atomicAdd(&P.prof[i], t_acc[i]);
    atomicAdd(&P.prof[15], 1ull);
  }
#undef PMARK
  // ---------------- counters
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    my_votes += __shfl_xor_sync(0xffffffffu, my_votes, o);
    my_hot += __shfl_xor_sync(0xffffffffu, my_hot, o);
  }
  if (lane == 0) {
    (void)my_votes;   // the per-frame vote count comes from K1.5 (k_rays.cu)
    if (my_hot) atomicAdd(&P.stats[f].hotspots, (unsigned long long)my_hot);
  }
  if (tid == 0 && *s_flags) atomicOr(&P.flags[f], *s_flags);
}

size_t k_hough_smem(const Params& P, int G) {
  return k2_layout(G, P.k2t, P.hal, P.entry_cap, P.hot_cap, P.n_levels, P.wstride).total;
}

int k_hough_max_entries() { return 65535; }

template <bool Wd, int Gv, int MB>
static void launch_one(int n_frames, const Params& P, int nt, cudaStream_t st) {
  const size_t sm = k_hough_smem(P, Gv);
  cudaFuncSetAttribute(k_hough<Wd, Gv, MB>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  k_hough<Wd, Gv, MB><<<dim3(P.ntx * P.nty, n_frames), nt, sm, st>>>(P);
}

cudaError_t launch_hough(int n_frames, const Params& P, bool wide, int G, int nt, int minb, cudaStream_t st) {
  const int key = (G << 2) | (wide ? 2 : 0) | (minb > 1 ? 1 : 0);
  switch (key) {
    case (8 << 2) | 0: launch_one<false, 8, 1>(n_frames, P, nt, st); break;
    case (8 << 2) | 2: launch_one<true, 8, 1>(n_frames, P, nt, st); break;
    case (8 << 2) | 1: launch_one<false, 8, 2>(n_frames, P, nt, st); break;
    case (8 << 2) | 3: launch_one<true, 8, 2>(n_frames, P, nt, st); break;
    case (4 << 2) | 0: launch_one<false, 4, 1>(n_frames, P, nt, st); break;
    case (4 << 2) | 2: launch_one<true, 4, 1>(n_frames, P, nt, st); break;
    case (4 << 2) | 1: launch_one<false, 4, 2>(n_frames, P, nt, st); break;
    case (4 << 2) | 3: launch_one<true, 4, 2>(n_frames, P, nt, st); break;
    case (2 << 2) | 0: launch_one<false, 2, 1>(n_frames, P, nt, st); break;
    case (2 << 2) | 2: launch_one<true, 2, 1>(n_frames, P, nt, st); break;
    case (2 << 2) | 1: launch_one<false, 2, 2>(n_frames, P, nt, st); break;
    case (2 << 2) | 3: launch_one<true, 2, 2>(n_frames, P, nt, st); break;
    default: return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

}  // namespace rd
