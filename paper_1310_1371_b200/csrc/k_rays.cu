// k_rays.cu — K1.5: route every voting ray to the Hough tiles its votes can reach.
//
// A voting ray is a ridge pixel p with one sense s of its direction rho (reading R8): its
// votes land at p + s*llround(r*rho), r in [r_min-1, r_max+1] (PAPER.md:308-313, 931-933,
// 998-1001).  For each ray and each T x T Hough tile whose level boxes (tile + K_r + 1) the
// ray's target segment can touch, the ray is appended to the tile's list together with a
// conservative level interval [ra, rb] (necessary conditions, linear in r because
// K_r <= m r + c; exactness is restored per vote in K2).
// A bin's rays can only reach the tiles of a small window around the 32x32 ridge bin, which
// a warp walks uniformly; the rays that hit a tile are appended with one global atomic per
// warp and tile (ballot + popc), so list appends do not contend per ray.
#include "rd_internal.cuh"

namespace rd {

namespace {
// llround of an exactly computed product (|v| < 2^31), as in K2 (reading R9)
__device__ __forceinline__ int rnd_half_away(double v) { return __double2int_rz(__dadd_rz(v, copysign(0.5, v))); }

// Largest r in [rlo - 1, rhi] such that c + llround(r' d) lies in [0, n - 1] for every r' in
// [rlo, r]: the target coordinate is monotone in r and starts inside the frame (r = 0), so
// the in-frame levels of a ray are a prefix of the level range.  A float estimate of the
// crossing, then exact steps to the boundary.
__device__ __forceinline__ bool inframe_at(int c, double d, int n, int r) {
  const int t = c + rnd_half_away(__dmul_rn((double)r, d));
  return t >= 0 && t <= n - 1;
}
__device__ int inframe_prefix(int c, double d, float inv_d, int n, int rlo, int rhi) {
  const float fd = (float)d;   // (inv_d = 1 / fd, 0 if fd = 0)
  const float lim = fd > 0.f ? ((float)n - 0.5f - (float)c) * inv_d : fd < 0.f ? (-0.5f - (float)c) * inv_d : 1e9f;
  int r = (int)fminf(fmaxf(floorf(lim), (float)(rlo - 1)), (float)rhi);
  while (r < rhi && inframe_at(c, d, n, r + 1)) ++r;
  while (r >= rlo && !inframe_at(c, d, n, r)) --r;
  return r;
}

__device__ __forceinline__ void half_ge(float a, float b, float& lo, float& hi) {
  if (a > 0.f) lo = fmaxf(lo, __fdividef(b, a));
  else if (a < 0.f) hi = fminf(hi, __fdividef(b, a));
  else if (b > 0.f) hi = -1e30f;
}
// the same half-plane a r >= b, branch-free, with ia = 1 / a (0 if a = 0)
__device__ __forceinline__ void clip(float a, float ia, float b, float& lo, float& hi) {
  const float t = b * ia;
  lo = a > 0.f ? fmaxf(lo, t) : lo;
  hi = a < 0.f ? fminf(hi, t) : ((a == 0.f && b > 0.f) ? -1e30f : hi);
}
__device__ __forceinline__ float rcp0(float a) { return a != 0.f ? __frcp_rn(a) : 0.f; }
}  // namespace

// One warp per (ridge bin, frame) (32 rays per pass), K15_WPB warps per CTA: small CTAs, so a
// CTA's slot is not held by warps that finished while another one still walks a busy bin.
// The clip of a ray's level interval splits into frame constraints (per ray), row
// constraints (per tile row ty) and column constraints (per tile column tx), so the inner
// tile loop evaluates two half-planes with precomputed reciprocals.
#ifndef RD_K15_WPB
#define RD_K15_WPB 1
#endif
constexpr int K15_WPB = RD_K15_WPB;
#ifndef RD_K15_MINB
#define RD_K15_MINB (32 / RD_K15_WPB)   // 64 registers: occupancy decides this latency-bound kernel
#endif
__global__ void __launch_bounds__(32 * K15_WPB, RD_K15_MINB) k_rays(Params P) {
  const int f = blockIdx.y;
  const int TX = P.k2t, TY = P.k2ty, hal = P.hal, W = P.W, H = P.H;
  const int rlo = P.r_lo, rhi = P.r_hi;
  const float m = P.k_slope, c = P.k_icpt;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t tile0 = (int64_t)f * P.ntx * P.nty;
  // tiles any ray of a bin can reach: |offset| <= r_hi, halo <= hal
  const int reach = rhi + hal + 1;
  int my_votes = 0, need_r = 0;
  const int bin = blockIdx.x * K15_WPB + warp;
  if (bin < P.nbx * P.nby) {
    const int by = bin / P.nbx, bx = bin - by * P.nbx;
    const int wy0 = max((by * T1 - reach) / TY, 0), wy1 = min((by * T1 + T1 - 1 + reach) / TY, P.nty - 1);
    const int64_t fb = (int64_t)f * P.nbx * P.nby + by * P.nbx + bx;
    const int cnt_all = P.bin_count[fb];   // the true count: ridges beyond ridge_cap were not stored
    need_r = max(need_r, cnt_all);
    const int cnt = min(cnt_all, P.ridge_cap);
    const int wx0 = max((bx * T1 - reach) / TX, 0), wx1 = min((bx * T1 + T1 - 1 + reach) / TX, P.ntx - 1);
    for (int j0 = 0; j0 < 2 * cnt; j0 += 32) {
      const int j = j0 + lane;
      const bool valid = j < 2 * cnt;
      uint32_t xy = 0;
      double2 d = make_double2(0.0, 0.0);
      if (valid) {
        const int64_t gi = fb * P.ridge_cap + (j >> 1);
        xy = P.bin_xy[gi];
        const double2 vraw = P.bin_d[gi];
        // K1 leaves the direction unnormalised: rho = v / |v| here, where ridges are dense in the
        // lanes (both senses compute it; sense 0 stores it for the dumps)
        normalise_dir(vraw.x, vraw.y, &d.x, &d.y);
        if (!(j & 1)) P.bin_d[gi] = d;
      }
      const double sgn = (j & 1) ? -1.0 : 1.0;
      const int x = (int)(xy & 0xFFFFu), y = (int)(xy >> 16);
      const double u = sgn * d.x, v = sgn * d.y;
      const float fu = (float)u, fv = (float)v, fx = (float)x, fy = (float)y;
      const float iu = rcp0(fu), iv = rcp0(fv);
      if (valid) {   // the ray's in-frame votes (per-frame vote count)
        const int px = inframe_prefix(x, u, iu, W, rlo, rhi), py = inframe_prefix(y, v, iv, H, rlo, rhi);
        my_votes += max(0, min(px, py) - rlo + 1);
      }
      // frame constraints (tile independent)
      float flo = (float)rlo, fhi = (float)rhi;
      clip(fu, iu, -0.5f - fx, flo, fhi);
      clip(-fu, -iu, fx - (float)W + 0.5f, flo, fhi);
      clip(fv, iv, -0.5f - fy, flo, fhi);
      clip(-fv, -iv, fy - (float)H + 0.5f, flo, fhi);
      // bounding box of the target segment, widened by the largest halo and rounding
      const float ax = fx + fu * rlo, bxp = fx + fu * rhi, ay = fy + fv * rlo, byp = fy + fv * rhi;
      const float sx0 = fminf(ax, bxp) - hal - 1.f, sx1 = fmaxf(ax, bxp) + hal + 1.f;
      const float sy0 = fminf(ay, byp) - hal - 1.f, sy1 = fmaxf(ay, byp) + hal + 1.f;
      if (wx1 - wx0 < 3 && wy1 - wy0 < 3) {
        // window of at most 3 x 3 tiles (the usual case): clip and ballot every tile first
        // (lane k keeps tile k's ballot), reserve all the window's list slots with one
        // round of atomics (lane k: tile k), then write; one global round trip per 32 rays
        uint32_t rng[9];
        unsigned kbal = 0, hits = 0;
        // a tile's clip is the intersection of a row part (frame + the tile row's two
        // half-planes) and a column part (the tile column's two), each evaluated once per row or
        // column, branch-free against the four slopes' reciprocals (per ray)
        const float ay1 = fv + m, ay2 = m - fv, ax1 = fu + m, ax2 = m - fu;
        const float iy1 = rcp0(ay1), iy2 = rcp0(ay2), ix1 = rcp0(ax1), ix2 = rcp0(ax2);
        float xlo[3], xhi[3];
#pragma unroll
        for (int kx = 0; kx < 3; ++kx) {
          const int X0 = (wx0 + kx) * TX;
          xlo[kx] = -1e30f;
          xhi[kx] = 1e30f;
          clip(ax1, ix1, (float)X0 - 1.5f - c - fx, xlo[kx], xhi[kx]);
          clip(ax2, ix2, fx - (float)(X0 + TX) - 0.5f - c, xlo[kx], xhi[kx]);
        }
#pragma unroll
        for (int ky = 0; ky < 3; ++ky) {
          const int ty = wy0 + ky, Y0 = ty * TY;
          float ylo = flo, yhi = fhi;
          clip(ay1, iy1, (float)Y0 - 1.5f - c - fy, ylo, yhi);
          clip(ay2, iy2, fy - (float)(Y0 + TY) - 0.5f - c, ylo, yhi);
          const bool yhit = valid && ty <= wy1 && sy1 >= Y0 && sy0 <= Y0 + TY - 1 && yhi >= ylo - 2.f;
#pragma unroll
          for (int kx = 0; kx < 3; ++kx) {
            const int k = 3 * ky + kx, tx = wx0 + kx, X0 = tx * TX;
            const float lo = fmaxf(ylo, xlo[kx]), hi = fminf(yhi, xhi[kx]);
            const int ra = max((int)floorf(lo) - 1, rlo), rb = min((int)ceilf(hi) + 1, rhi);
            const bool hit = yhit && tx <= wx1 && sx1 >= X0 && sx0 <= X0 + TX - 1 && hi >= lo - 2.f && ra <= rb;
            rng[k] = (uint32_t)(ra - rlo) | ((uint32_t)(rb - rlo) << 16);
            const unsigned bal = __ballot_sync(0xffffffffu, hit);
            if (lane == k) kbal = bal;
            hits |= (unsigned)hit << k;
          }
        }
        int base = 0;
        if (kbal) base = atomicAdd(&P.ray_count[tile0 + (wy0 + lane / 3) * P.ntx + wx0 + lane % 3], __popc(kbal));
#pragma unroll
        for (int k = 0; k < 9; ++k) {
          const unsigned bal = __shfl_sync(0xffffffffu, kbal, k);
          if (!bal) continue;
          const int b = __shfl_sync(0xffffffffu, base, k);
          if (!((hits >> k) & 1u)) continue;
          const int e = b + __popc(bal & ((1u << lane) - 1u));
          RD_CHECK(wy0 + k / 3 < P.nty && wx0 + k % 3 < P.ntx, CK_K15_TILE);
          if (e < P.entry_cap) {
            const int64_t o = (tile0 + (wy0 + k / 3) * P.ntx + wx0 + k % 3) * P.entry_cap + e;
            P.ray_d[o] = make_double2(u, v);
            P.ray_xy[o] = xy;
            if (P.k2_rr16) reinterpret_cast<uint16_t*>(P.ray_r)[o] = (uint16_t)((rng[k] & 0xFFu) | ((rng[k] >> 16) << 8));
            else P.ray_r[o] = rng[k];
          } else {
            atomicOr(&P.flags[f], OVF_ENTRIES);
          }
        }
        continue;
      }
      for (int ty = wy0; ty <= wy1; ++ty) {
        const int Y0 = ty * TY;
        float ylo = flo, yhi = fhi;
        half_ge(fv + m, (float)Y0 - 1.5f - c - fy, ylo, yhi);
        half_ge(m - fv, fy - (float)(Y0 + TY) - 0.5f - c, ylo, yhi);
        const bool yhit = valid && sy1 >= Y0 && sy0 <= Y0 + TY - 1 && yhi >= ylo - 2.f;
        if (!__any_sync(0xffffffffu, yhit)) continue;
        for (int tx = wx0; tx <= wx1; ++tx) {
          const int X0 = tx * TX;
          bool hit = yhit && sx1 >= X0 && sx0 <= X0 + TX - 1;
          int ra = 0, rb = -1;
          if (hit) {
            float lo = ylo, hi = yhi;
            half_ge(fu + m, (float)X0 - 1.5f - c - fx, lo, hi);
            half_ge(m - fu, fx - (float)(X0 + TX) - 0.5f - c, lo, hi);
            ra = max((int)floorf(lo) - 1, rlo);
            rb = min((int)ceilf(hi) + 1, rhi);
            hit = hi >= lo - 2.f && ra <= rb;
          }
          const unsigned bal = __ballot_sync(0xffffffffu, hit);
          if (!bal) continue;
          const int64_t t = tile0 + ty * P.ntx + tx;
          int base = 0;
          if (lane == __ffs(bal) - 1) base = atomicAdd(&P.ray_count[t], __popc(bal));
          base = __shfl_sync(0xffffffffu, base, __ffs(bal) - 1);
          if (!hit) continue;
          const int e = base + __popc(bal & ((1u << lane) - 1u));
          if (e < P.entry_cap) {
            const int64_t o = t * P.entry_cap + e;
            P.ray_d[o] = make_double2(u, v);
            P.ray_xy[o] = xy;
            if (P.k2_rr16) reinterpret_cast<uint16_t*>(P.ray_r)[o] = (uint16_t)((ra - rlo) | ((rb - rlo) << 8));
            else P.ray_r[o] = (uint32_t)(ra - rlo) | ((uint32_t)(rb - rlo) << 16);
          } else {
            atomicOr(&P.flags[f], OVF_ENTRIES);
          }
        }
      }
    }
  }
  my_votes = __reduce_add_sync(0xffffffffu, my_votes);
  if (lane == 0 && my_votes) atomicAdd(&P.stats[f].votes, (unsigned long long)my_votes);
  // ridges per bin the frame needed (per-frame slot; k_scan folds the frames into P.need)
  need_r = __reduce_max_sync(0xffffffffu, need_r);
  if (lane == 0 && need_r) atomicMax(&P.need_ridges[f], need_r);
}

cudaError_t launch_rays(int n_frames, const Params& P, cudaStream_t st) {
  k_rays<<<dim3((P.nbx * P.nby + K15_WPB - 1) / K15_WPB, n_frames), 32 * K15_WPB, 0, st>>>(P);
  return cudaGetLastError();
}

}  // namespace rd
