// k_hough.cu — K2: directed voting, hotspot registration, radius-dependent smoothing
// with 1/r normalisation and 3x3x3 peak extraction, one CTA per (frame, 64x64 tile).
//
// Rows A5-A8 of DESIGN.md §2 (SI steps 2-4, PAPER.md:931-978;
// range extension PAPER.md:998-1001).  The CTA owns the accumulator cells of its tile and
// sweeps r upward through the Hough range, keeping on chip:
//   raw(r)  — one level of packed uint16 counters over tile + (K_r + 1) halo,
//             filled with warp-issued shared-memory atomics;
//   three rolling levels (r-2, r-1, r) of hotspot lists + a cell->hotspot index map over
//             tile + 1 (the paper's r mod 3 recycling, re-expressed
//             for shared memory), holding the exact fixed-point window sums S.
// A hotspot is registered by the one atomic that lifts its counter past T_raw (the
// paper's "surpassed" test at increment time).  S is computed for
// hotspots only; NMS of level r-1 runs once level r is complete.
// Nothing but the peak records (and optional debug hotspots) leaves the SM.
#include "rd_internal.cuh"

namespace rd {

namespace {
constexpr int IDXS = T2 + 2;      // index-map side: tile + 1 ring

struct K2Smem {
  // computed on host and device identically
  int raws, rawp;                 // raw side and row pitch (uint16 units, even)
  size_t off_hS, off_ed, off_raw, off_idx, off_hcell, off_hraw, off_exy, off_err, off_hcnt, off_w, off_bins, total;
};

__host__ __device__ inline size_t align16(size_t v) { return (v + 15) & ~size_t(15); }

__host__ __device__ inline K2Smem k2_layout(int hal, int entry_cap, int hot_cap, int n_levels, int wstride,
                                            int max_bins) {
  K2Smem L;
  L.raws = T2 + 2 * hal;
  L.rawp = (L.raws + 7) & ~7;
  size_t o = 0;
  L.off_hS = o;    o = align16(o + sizeof(long long) * 3 * hot_cap);
  L.off_ed = o;    o = align16(o + sizeof(double2) * entry_cap);
  L.off_raw = o;   o = align16(o + 2 * (size_t)L.raws * L.rawp);
  L.off_idx = o;   o = align16(o + 2 * 3 * IDXS * IDXS);
  L.off_hcell = o; o = align16(o + 2 * 3 * hot_cap);
  L.off_hraw = o;  o = align16(o + 2 * 3 * hot_cap);
  L.off_exy = o;   o = align16(o + 4 * entry_cap);
  L.off_err = o;   o = align16(o + 4 * entry_cap);
  L.off_hcnt = o;  o = align16(o + 4 * (n_levels + 8));
  L.off_w = o;     o = align16(o + 4 * wstride);
  L.off_bins = o;  o = align16(o + 4 * (max_bins + 1));
  L.total = o;
  return L;
}
}  // namespace

template <bool kWide>
__global__ void __launch_bounds__(K2_THREADS, 2) k_hough(Params P, int max_bins) {
  extern __shared__ __align__(16) unsigned char smem[];
  const K2Smem L = k2_layout(P.hal, P.entry_cap, P.hot_cap, P.n_levels, P.wstride, max_bins);
  long long* hS = reinterpret_cast<long long*>(smem + L.off_hS);        // [3][hot_cap]
  double2* eD = reinterpret_cast<double2*>(smem + L.off_ed);             // [entry_cap] (s*dx, s*dy)
  uint32_t* raw32 = reinterpret_cast<uint32_t*>(smem + L.off_raw);       // packed uint16 counters
  uint16_t* raw16 = reinterpret_cast<uint16_t*>(smem + L.off_raw);
  uint16_t* idx = reinterpret_cast<uint16_t*>(smem + L.off_idx);         // [3][IDXS*IDXS]
  uint16_t* hcell = reinterpret_cast<uint16_t*>(smem + L.off_hcell);     // [3][hot_cap]
  uint16_t* hraw = reinterpret_cast<uint16_t*>(smem + L.off_hraw);       // [3][hot_cap]
  uint32_t* eXY = reinterpret_cast<uint32_t*>(smem + L.off_exy);         // [entry_cap] x | y<<16
  uint32_t* eR = reinterpret_cast<uint32_t*>(smem + L.off_err);          // [entry_cap] ra | rb<<16
  int* hcnt = reinterpret_cast<int*>(smem + L.off_hcnt);                 // [n_levels] + misc
  int* wl = reinterpret_cast<int*>(smem + L.off_w);                      // current level weights
  int* binpre = reinterpret_cast<int*>(smem + L.off_bins);               // bin prefix sums
  int* s_ecnt = hcnt + P.n_levels;
  int* s_flags = s_ecnt + 1;
  unsigned long long* s_votes = reinterpret_cast<unsigned long long*>(hcnt + P.n_levels + 2);
  int* s_nhot = hcnt + P.n_levels + 4;

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int f = blockIdx.y;
  const int tile = blockIdx.x;
  const int tyi = tile / P.ntx, txi = tile - tyi * P.ntx;
  const int X0 = txi * T2, Y0 = tyi * T2;
  const int W = P.W, H = P.H, hal = P.hal;
  const int RX0 = X0 - hal, RY0 = Y0 - hal;   // raw buffer origin
  const int rawp = L.rawp, raws = L.raws;

  for (int i = tid; i < 3 * IDXS * IDXS; i += K2_THREADS) idx[i] = 0;
  for (int i = tid; i < P.n_levels + 8; i += K2_THREADS) hcnt[i] = 0;

  // ---------------- phase 0: voting rays that can reach tile + max halo
  // box E = (tile + hal) intersected with the frame
  const int bx0 = max(X0 - hal, 0), bx1 = min(X0 + T2 - 1 + hal, W - 1);
  const int by0 = max(Y0 - hal, 0), by1 = min(Y0 + T2 - 1 + hal, H - 1);
  const int rhi = P.r_hi, rlo = P.r_lo;
  const int nbx = P.nbx;
  const int cbx0 = max((bx0 - rhi) / T1, 0), cbx1 = min((bx1 + rhi) / T1, P.nbx - 1);
  const int cby0 = max((by0 - rhi) / T1, 0), cby1 = min((by1 + rhi) / T1, P.nby - 1);
  const int nbw = cbx1 - cbx0 + 1, nbins = nbw * (cby1 - cby0 + 1);
  const int64_t fbins = (int64_t)f * P.nbx * P.nby;
  for (int i = tid; i < nbins; i += K2_THREADS) {
    int by = cby0 + i / nbw, bx = cbx0 + i % nbw;
    binpre[i + 1] = P.bin_count[fbins + by * nbx + bx];
  }
  __syncthreads();
  if (tid == 0) {
    binpre[0] = 0;
    for (int i = 1; i <= nbins; ++i) binpre[i] += binpre[i - 1];
  }
  __syncthreads();
  const int nrid = binpre[nbins];
  for (int k = tid; k < 2 * nrid; k += K2_THREADS) {
    int rk = k >> 1;
    double sgn = (k & 1) ? -1.0 : 1.0;
    int lo = 0, hi = nbins - 1;  // bin containing ridge rk
    while (lo < hi) {
      int mid = (lo + hi + 1) >> 1;
      if (binpre[mid] <= rk) lo = mid; else hi = mid - 1;
    }
    int by = cby0 + lo / nbw, bx = cbx0 + lo % nbw;
    int64_t g = (fbins + by * nbx + bx) * P.ridge_cap + (rk - binpre[lo]);
    uint32_t xy = P.bin_xy[g];
    double2 d = P.bin_d[g];
    int x = (int)(xy & 0xFFFFu), y = (int)(xy >> 16);
    double u = sgn * d.x, v = sgn * d.y;
    // conservative interval of r with target inside E (exactness restored per vote)
    float rl = (float)rlo, rh = (float)rhi;
    float fu = (float)u, fv = (float)v;
    if (fu > 0.f) { rl = fmaxf(rl, (bx0 - x - 0.5f) / fu); rh = fminf(rh, (bx1 - x + 0.5f) / fu); }
    else if (fu < 0.f) { rl = fmaxf(rl, (bx1 - x + 0.5f) / fu); rh = fminf(rh, (bx0 - x - 0.5f) / fu); }
    else if (x < bx0 || x > bx1) continue;
    if (fv > 0.f) { rl = fmaxf(rl, (by0 - y - 0.5f) / fv); rh = fminf(rh, (by1 - y + 0.5f) / fv); }
    else if (fv < 0.f) { rl = fmaxf(rl, (by1 - y + 0.5f) / fv); rh = fminf(rh, (by0 - y - 0.5f) / fv); }
    else if (y < by0 || y > by1) continue;
    int ra = max((int)floorf(rl) - 1, rlo), rb = min((int)ceilf(rh) + 1, rhi);
    if (ra > rb) continue;
    int e = atomicAdd(s_ecnt, 1);
    if (e < P.entry_cap) {
      eD[e] = make_double2(u, v);
      eXY[e] = xy;
      eR[e] = (uint32_t)(ra - rlo) | ((uint32_t)(rb - rlo) << 16);
    } else {
      atomicOr(s_flags, OVF_ENTRIES);
    }
  }
  __syncthreads();
  const int ne = min(*s_ecnt, P.entry_cap);
  unsigned long long my_votes = 0;
  int my_hot = 0;
  const uint32_t raw_words = (uint32_t)(raws * rawp) >> 1;

  // ---------------- level sweep
  for (int li = 0; li < P.n_levels; ++li) {
    const int r = rlo + li;
    const int slot = li % 3;
    const int K = P.lvlK[li];
    // (a) clear raw, clear the index-map entries of level li-3 (same slot), load weights
    {
      uint4* r4 = reinterpret_cast<uint4*>(raw32);
      for (uint32_t i = tid; i < raw_words / 4; i += K2_THREADS) r4[i] = make_uint4(0, 0, 0, 0);
      for (uint32_t i = (raw_words / 4) * 4 + tid; i < raw_words; i += K2_THREADS) raw32[i] = 0;
      if (li >= 3) {
        int nold = min(hcnt[li - 3], P.hot_cap);
        uint16_t* im = idx + slot * IDXS * IDXS;
        const uint16_t* hc = hcell + slot * P.hot_cap;
        for (int k = tid; k < nold; k += K2_THREADS) im[hc[k]] = 0;
      }
      for (int i = tid; i <= K; i += K2_THREADS) wl[i] = P.lvlW[li * P.wstride + i];
    }
    __syncthreads();
    // (b) votes of level r into raw(r) over tile + (K_r + 1)
    {
      const int vx0 = max(X0 - K - 1, 0), vx1 = min(X0 + T2 + K, W - 1);
      const int vy0 = max(Y0 - K - 1, 0), vy1 = min(Y0 + T2 + K, H - 1);
      const double rd = (double)r;
      uint16_t* im = idx + slot * IDXS * IDXS;
      uint16_t* hc = hcell + slot * P.hot_cap;
      const uint32_t T_raw = (uint32_t)P.T_raw;
      for (int e = tid; e < ne; e += K2_THREADS) {
        uint32_t rr = eR[e];
        if (li < (int)(rr & 0xFFFFu) || li > (int)(rr >> 16)) continue;
        double2 d = eD[e];
        uint32_t xy = eXY[e];
        int tx = (int)(xy & 0xFFFFu) + (int)llround(__dmul_rn(rd, d.x));
        int ty = (int)(xy >> 16) + (int)llround(__dmul_rn(rd, d.y));
        if (tx < vx0 || tx > vx1 || ty < vy0 || ty > vy1) continue;
        int cell = (ty - RY0) * rawp + (tx - RX0);
        uint32_t sh = (cell & 1) << 4;
        uint32_t old = atomicAdd(&raw32[cell >> 1], 1u << sh);
        uint32_t oc = (old >> sh) & 0xFFFFu;
        int ix = tx - (X0 - 1), iy = ty - (Y0 - 1);
        bool in_ring = (unsigned)ix < (unsigned)IDXS && (unsigned)iy < (unsigned)IDXS;
        if (oc == T_raw && in_ring) {
          int k = atomicAdd(&hcnt[li], 1);
          if (k < P.hot_cap) {
            uint16_t c16 = (uint16_t)(iy * IDXS + ix);
            hc[k] = c16;
            im[c16] = (uint16_t)(k + 1);
          } else {
            atomicOr(s_flags, OVF_HOTSPOTS);
          }
        }
        my_votes += (ix >= 1 && ix <= T2 && iy >= 1 && iy <= T2);
      }
    }
    __syncthreads();
    // (c) S = sum_{|i|,|j|<=K} w(i) w(j) raw(y+i, x+j) at each hotspot
    {
      const int nh = min(hcnt[li], P.hot_cap);
      const uint16_t* hc = hcell + slot * P.hot_cap;
      long long* hs = hS + slot * P.hot_cap;
      uint16_t* hr = hraw + slot * P.hot_cap;
      for (int h = warp; h < nh; h += K2_THREADS / 32) {
        int c16 = hc[h];
        int iy = c16 / IDXS, ix = c16 - iy * IDXS;
        int ly = iy - 1 + hal, lx = ix - 1 + hal;   // raw-local coordinates
        unsigned long long acc = 0;
        for (int i = lane - K; i <= K; i += 32) {
          const uint16_t* row = raw16 + (ly + i) * rawp + lx;
          if (kWide) {
            unsigned long long rs = 0;
            for (int j = -K; j <= K; ++j) rs += (unsigned long long)wl[j < 0 ? -j : j] * row[j];
            acc += rs * (unsigned long long)wl[i < 0 ? -i : i];
          } else {
            uint32_t rs = 0;
            for (int j = -K; j <= K; ++j) rs += (uint32_t)wl[j < 0 ? -j : j] * row[j];
            acc += (unsigned long long)rs * (unsigned long long)wl[i < 0 ? -i : i];
          }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
        if (lane == 0) {
          hs[h] = (long long)acc;
          uint16_t c = raw16[ly * rawp + lx];
          hr[h] = c;
          bool interior = ix >= 1 && ix <= T2 && iy >= 1 && iy <= T2;
          if (interior) {
            ++my_hot;
            if (P.debug) {
              int k = atomicAdd(&P.dbg_count[f], 1);
              if (k < P.dbg_cap) {
                HotRec rec;
                rec.r = r; rec.y = Y0 - 1 + iy; rec.x = X0 - 1 + ix; rec.raw = c; rec.S = (long long)acc;
                P.dbg_hot[(int64_t)f * P.dbg_cap + k] = rec;
              } else {
                atomicOr(&P.flags[f], OVF_DEBUG);
              }
            }
          }
        }
      }
    }
    __syncthreads();
    // (d) peaks of level rc = r - 1: candidates S > T_norm(rc), 3x3x3 maxima of S/r (R14)
    if (li >= 2 && r - 1 >= P.r_min && r - 1 <= P.r_max) {
      const int lc = li - 1, sc = lc % 3, rc = r - 1;
      const int nh = min(hcnt[lc], P.hot_cap);
      const double Tn = P.lvlTn[lc];
      const uint16_t* hc = hcell + sc * P.hot_cap;
      for (int h = tid; h < nh; h += K2_THREADS) {
        int c16 = hc[h];
        int iy = c16 / IDXS, ix = c16 - iy * IDXS;
        if (ix < 1 || ix > T2 || iy < 1 || iy > T2) continue;    // interior cells only
        long long S = hS[sc * P.hot_cap + h];
        if (!((double)S > Tn)) continue;
        int gy = Y0 - 1 + iy, gx = X0 - 1 + ix;
        bool peak = true;
        for (int dl = -1; dl <= 1 && peak; ++dl) {
          const int l = lc + dl, sl = l % 3;
          const long long ru = rlo + l;
          const uint16_t* im = idx + sl * IDXS * IDXS;
          const long long* hs = hS + sl * P.hot_cap;
          for (int dy = -1; dy <= 1 && peak; ++dy) {
            if (gy + dy < 0 || gy + dy >= H) continue;
            for (int dx = -1; dx <= 1; ++dx) {
              if (!dl && !dy && !dx) continue;
              if (gx + dx < 0 || gx + dx >= W) continue;
              int k = im[(iy + dy) * IDXS + ix + dx];
              long long Su = k ? hs[k - 1] : 0;
              long long lhs = S * ru, rhs = Su * (long long)rc;
              bool v_first = dl > 0 || (dl == 0 && (dy > 0 || (dy == 0 && dx > 0)));
              if (!(lhs > rhs || (lhs == rhs && v_first))) { peak = false; break; }
            }
          }
        }
        if (peak) {
          int k = atomicAdd(&P.peak_count[f], 1);
          if (k < P.ring_cap) {
            Peak pk;
            pk.x = gx; pk.y = gy; pk.r = rc; pk.raw = hraw[sc * P.hot_cap + h]; pk.S = S;
            P.peaks[(int64_t)f * P.ring_cap + k] = pk;
          } else {
            atomicOr(&P.flags[f], OVF_RINGS);
          }
        }
      }
    }
    __syncthreads();
  }
  // ---------------- counters
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    my_votes += __shfl_xor_sync(0xffffffffu, my_votes, o);
    my_hot += __shfl_xor_sync(0xffffffffu, my_hot, o);
  }
  if (lane == 0) {
    if (my_votes) atomicAdd(&P.stats[f].votes, my_votes);
    if (my_hot) atomicAdd(&P.stats[f].hotspots, (unsigned long long)my_hot);
  }
  if (tid == 0 && *s_flags) atomicOr(&P.flags[f], *s_flags);
  (void)s_votes;
  (void)s_nhot;
}

size_t k_hough_smem(const Params& P, int max_bins) {
  return k2_layout(P.hal, P.entry_cap, P.hot_cap, P.n_levels, P.wstride, max_bins).total;
}

int k_hough_max_bins(const Params& P) {
  int span = T2 + 2 * P.hal + 2 * P.r_hi;
  int n = span / T1 + 2;
  return n * n;
}

cudaError_t launch_hough(int n_frames, const Params& P, bool wide, cudaStream_t st) {
  int mb = k_hough_max_bins(P);
  size_t sm = k_hough_smem(P, mb);
  dim3 grid(P.ntx * P.nty, n_frames);
  if (wide) {
    cudaFuncSetAttribute(k_hough<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    k_hough<true><<<grid, K2_THREADS, sm, st>>>(P, mb);
  } else {
    cudaFuncSetAttribute(k_hough<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    k_hough<false><<<grid, K2_THREADS, sm, st>>>(P, mb);
  }
  return cudaGetLastError();
}

}  // namespace rd
