// k_fit.cu — K3: canonical ordering of the peaks, non-exclusive annulus classification
// of the ridge pixels and the Kasa circle fit, one CTA per frame, one warp per ring.
//
// Rows A9-A11 of DESIGN.md §2 ("for each peak an annulus mask is formed
// and a best fitting circle is found for all ridge coordinates within the annulus";
// SI step 5).  Membership is an exact integer test
// (r-w)_+^2 <= d^2 <= (r+w)^2 over the ridge bins the annulus overlaps; the moments are
// int64 sums (order-free, hence bit-exact); the 3x3 normal equations are solved by
// Cramer's rule with exact int128 determinants and one rounding per unknown.
#include <algorithm>

#include "rd_internal.cuh"

namespace rd {

__device__ __forceinline__ long long warp_sum_ll(long long v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ double warp_sum_d(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__device__ __forceinline__ __int128 det3(__int128 a, __int128 b, __int128 c, __int128 d, __int128 e, __int128 f,
                                         __int128 g, __int128 h, __int128 i) {
  return a * (e * i - f * h) - b * (d * i - f * g) + c * (d * h - e * g);
}

__global__ void __launch_bounds__(K3_THREADS) k_fit(Params P) {
  extern __shared__ __align__(16) unsigned char smem[];
  Peak* sp = reinterpret_cast<Peak*>(smem);                    // [ring_cap]
  int* order = reinterpret_cast<int*>(sp + P.ring_cap);         // [ring_cap]
  const int f = blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int npk = P.peak_count[f];
  const int flags = P.flags[f];
  if (flags != 0 || npk > P.ring_cap) return;   // k_emit reports the frame with count -1
  for (int i = tid; i < npk; i += K3_THREADS) sp[i] = P.peaks[(int64_t)f * P.ring_cap + i];
  __syncthreads();
  // canonical (r, cy, cx) order: rank of each (unique) key
  for (int i = tid; i < npk; i += K3_THREADS) {
    const Peak a = sp[i];
    int rank = 0;
    for (int j = 0; j < npk; ++j) {
      const Peak b = sp[j];
      rank += (b.r < a.r) || (b.r == a.r && (b.y < a.y || (b.y == a.y && b.x < a.x)));
    }
    RD_CHECK(rank < npk, CK_K3_ORDER);
    order[rank] = i;
  }
  __syncthreads();
  const int64_t fbins = (int64_t)f * P.nbx * P.nby;
  // the frame's rings are dealt to gridDim.y CTAs (each ranks all peaks: the sort is cheap)
  for (int p = warp * gridDim.y + blockIdx.y; p < npk; p += (K3_THREADS / 32) * gridDim.y) {
    const Peak pk = sp[order[p]];
    const int w = P.lvlAnn[pk.r - P.r_lo];
    const long long lo = max(pk.r - w, 0), hi = (long long)pk.r + w;
    const long long lo2 = lo * lo, hi2 = hi * hi;
    const int bx0 = max((pk.x - (int)hi) / T1, 0), bx1 = min((pk.x + (int)hi) / T1, P.nbx - 1);
    const int by0 = max((pk.y - (int)hi) / T1, 0), by1 = min((pk.y + (int)hi) / T1, P.nby - 1);
    long long n = 0, Su = 0, Sv = 0, Suu = 0, Svv = 0, Suv = 0, Sz = 0, Suz = 0, Svz = 0;
    for (int by = by0; by <= by1; ++by)
      for (int bx = bx0; bx <= bx1; ++bx) {
        const int64_t b = fbins + by * P.nbx + bx;
        const int cnt = min(P.bin_count[b], P.ridge_cap);
        RD_CHECK(cnt >= 0 && cnt <= P.ridge_cap && bx < P.nbx && by < P.nby, CK_K3_BIN);
        const uint32_t* xy = P.bin_xy + b * P.ridge_cap;
        for (int k = lane; k < cnt; k += 32) {
          uint32_t v = xy[k];
          long long u = (long long)(v & 0xFFFFu) - pk.x, vv = (long long)(v >> 16) - pk.y;
          long long z = u * u + vv * vv;
          if (z < lo2 || z > hi2) continue;
          ++n; Su += u; Sv += vv; Suu += u * u; Svv += vv * vv; Suv += u * vv; Sz += z; Suz += u * z; Svz += vv * z;
        }
      }
    n = warp_sum_ll(n); Su = warp_sum_ll(Su); Sv = warp_sum_ll(Sv); Suu = warp_sum_ll(Suu); Svv = warp_sum_ll(Svv);
    Suv = warp_sum_ll(Suv); Sz = warp_sum_ll(Sz); Suz = warp_sum_ll(Suz); Svz = warp_sum_ll(Svz);
    // Kasa: [Suu Suv Su; Suv Svv Sv; Su Sv n] [D E F]^T = -[Suz Svz Sz]^T
    bool ok = false;
    double uc = 0, vc = 0, R = 0;
    if (n >= 3) {
      __int128 det = det3(Suu, Suv, Su, Suv, Svv, Sv, Su, Sv, n);
      if (det != 0) {
        __int128 nD = det3(-Suz, Suv, Su, -Svz, Svv, Sv, -Sz, Sv, n);
        __int128 nE = det3(Suu, -Suz, Su, Suv, -Svz, Sv, Su, -Sz, n);
        __int128 nF = det3(Suu, Suv, -Suz, Suv, Svv, -Svz, Su, Sv, -Sz);
        double dd = (double)det;
        double D = (double)nD / dd, E = (double)nE / dd, F = (double)nF / dd;
        uc = -0.5 * D;
        vc = -0.5 * E;
        double R2 = uc * uc + vc * vc - F;
        if (R2 >= 0.0) { R = sqrt(R2); ok = true; }
      }
    }
    double rms = 0.0;
    if (ok) {
      double acc = 0.0;
      for (int by = by0; by <= by1; ++by)
        for (int bx = bx0; bx <= bx1; ++bx) {
          const int64_t b = fbins + by * P.nbx + bx;
          const int cnt = min(P.bin_count[b], P.ridge_cap);
          const uint32_t* xy = P.bin_xy + b * P.ridge_cap;
          for (int k = lane; k < cnt; k += 32) {
            uint32_t v = xy[k];
            long long u = (long long)(v & 0xFFFFu) - pk.x, vv = (long long)(v >> 16) - pk.y;
            long long z = u * u + vv * vv;
            if (z < lo2 || z > hi2) continue;
            double du = (double)u - uc, dv = (double)vv - vc;
            double e = sqrt(du * du + dv * dv) - R;
            acc += e * e;
          }
        }
      acc = warp_sum_d(acc);
      rms = sqrt(acc / (double)n);
    }
    if (lane == 0) {
      Ring g;
      g.cx = pk.x; g.cy = pk.y; g.r = pk.r; g.raw_votes = pk.raw; g.score_fixed = pk.S;
      g.inliers = (int32_t)n; g.fit_ok = ok ? 1 : 0;
      g.fx = ok ? pk.x + uc : (double)pk.x;
      g.fy = ok ? pk.y + vc : (double)pk.y;
      g.fr = ok ? R : (double)pk.r;
      g.rms = rms;
      P.rings[(int64_t)f * P.ring_cap + p] = g;
    }
  }
  if (tid == 0 && blockIdx.y == 0) P.stats[f].peaks = (unsigned long long)npk;
}

// Classification output (A9): the ridge pixels of every ring of
// frame f, rings in the canonical order of K3's output.  One CTA; a warp per ring scans the
// ridge bins its annulus overlaps in the same order and with the same exact test as K3.
// write == 0: offsets[p + 1] = member count of ring p (offsets[0] = 0, prefix summed here);
// write == 1: members (x | y << 16) of ring p at offsets[p] .., in bin order (bin rows, bin
// columns, row-major within a bin).  The frame must not have overflowed (K3 wrote -1).
__global__ void __launch_bounds__(K3_THREADS) k_members(Params P, int f, int write, int* offsets,
                                                         uint32_t* members) {
  extern __shared__ __align__(16) unsigned char smem[];
  Peak* sp = reinterpret_cast<Peak*>(smem);                    // [ring_cap]
  int* order = reinterpret_cast<int*>(sp + P.ring_cap);         // [ring_cap]
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int npk = min(P.peak_count[f], P.ring_cap);
  for (int i = tid; i < npk; i += K3_THREADS) sp[i] = P.peaks[(int64_t)f * P.ring_cap + i];
  __syncthreads();
  for (int i = tid; i < npk; i += K3_THREADS) {   // canonical (r, cy, cx) order, as K3
    const Peak a = sp[i];
    int rank = 0;
    for (int j = 0; j < npk; ++j) {
      const Peak b = sp[j];
      rank += (b.r < a.r) || (b.r == a.r && (b.y < a.y || (b.y == a.y && b.x < a.x)));
    }
    order[rank] = i;
  }
  __syncthreads();
  const int64_t fbins = (int64_t)f * P.nbx * P.nby;
  for (int p = warp; p < npk; p += K3_THREADS / 32) {
    const Peak pk = sp[order[p]];
    const int w = P.lvlAnn[pk.r - P.r_lo];
    const long long lo = max(pk.r - w, 0), hi = (long long)pk.r + w;
    const long long lo2 = lo * lo, hi2 = hi * hi;
    const int bx0 = max((pk.x - (int)hi) / T1, 0), bx1 = min((pk.x + (int)hi) / T1, P.nbx - 1);
    const int by0 = max((pk.y - (int)hi) / T1, 0), by1 = min((pk.y + (int)hi) / T1, P.nby - 1);
    int n = write ? offsets[p] : 0;
    for (int by = by0; by <= by1; ++by)
      for (int bx = bx0; bx <= bx1; ++bx) {
        const int64_t b = fbins + by * P.nbx + bx;
        const int cnt = min(P.bin_count[b], P.ridge_cap);
        const uint32_t* xy = P.bin_xy + b * P.ridge_cap;
        for (int k0 = 0; k0 < cnt; k0 += 32) {
          const int k = k0 + lane;
          uint32_t v = 0;
          bool in = false;
          if (k < cnt) {
            v = xy[k];
            const long long u = (long long)(v & 0xFFFFu) - pk.x, vv = (long long)(v >> 16) - pk.y;
            const long long z = u * u + vv * vv;
            in = z >= lo2 && z <= hi2;
          }
          const unsigned bal = __ballot_sync(0xffffffffu, in);
          if (write && in) members[n + __popc(bal & ((1u << lane) - 1u))] = v;
          n += __popc(bal);
        }
      }
    if (!write && lane == 0) offsets[p + 1] = n;
  }
  if (!write) {
    __syncthreads();
    if (tid == 0) {
      offsets[0] = 0;
      for (int p = 0; p < npk; ++p) offsets[p + 1] += offsets[p];
    }
  }
}

cudaError_t launch_members(const Params& P, int f, int write, int* offsets, uint32_t* members, cudaStream_t st) {
  const size_t sm = (size_t)P.ring_cap * (sizeof(Peak) + sizeof(int));
  cudaFuncSetAttribute(k_members, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  k_members<<<1, K3_THREADS, sm, st>>>(P, f, write, offsets, members);
  return cudaGetLastError();
}

size_t k_fit_smem(const Params& P) { return (size_t)P.ring_cap * (sizeof(Peak) + sizeof(int)); }

cudaError_t launch_fit(int n_frames, const Params& P, cudaStream_t st) {
  size_t sm = k_fit_smem(P);
  cudaFuncSetAttribute(k_fit, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  // CTAs per frame (rings dealt across them; each ranks all peaks): enough to cover the SMs
  // at small batches, one per frame at large ones (cfg3, 256 frames: 0.69 -> 0.56 us/frame
  // against 4 per frame)
  const int split = std::max(1, std::min(4, (P.n_sm + n_frames - 1) / n_frames));
  k_fit<<<dim3(n_frames, split), K3_THREADS, sm, st>>>(P);
  return cudaGetLastError();
}

// Output assembly (A11): per-frame counts and CSR offsets over the call's
// frames, one CTA.  A frame is valid iff no internal capacity overflowed; its rings occupy
// [offsets[f], offsets[f] + counts[f]) of the caller's buffer.  offsets advance by every
// frame's peak count (0 for invalid frames), so offsets[n] is the capacity the call needed; a
// valid frame whose range passes out_cap gets count -1 and OVF_OUTPUT.  base_in (may be null:
// 0) is the first offset, base_out (may be null) receives offsets[n] (host-path chunks chain);
// flags_out (may be null) receives the frames' overflow bits.
__global__ void __launch_bounds__(1024) k_scan(Params P, int n_frames, int out_cap, int* __restrict__ counts,
                                               int* __restrict__ offsets, const int* base_in, int* base_out,
                                               int* flags_out) {
  __shared__ int wsum[32];
  __shared__ int carry;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) carry = base_in ? *base_in : 0;
  int mx = 0, mxr = 0;
  __syncthreads();
  for (int f0 = 0; f0 < n_frames; f0 += 1024) {
    const int f = f0 + tid;
    int npk = 0;
    bool valid = false;
    if (f < n_frames) {
      mxr = max(mxr, P.need_ridges[f]);
      npk = P.peak_count[f];
      valid = P.flags[f] == 0 && npk <= P.ring_cap;
      mx = max(mx, npk);
    }
    const int v = valid ? npk : 0;
    int incl = v;   // block-inclusive scan
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int t = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += t;
    }
    if (lane == 31) wsum[warp] = incl;
    __syncthreads();
    if (warp == 0) {
      int w = wsum[lane];
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int t = __shfl_up_sync(0xffffffffu, w, o);
        if (lane >= o) w += t;
      }
      wsum[lane] = w;
    }
    __syncthreads();
    const int c0 = carry;
    const int excl = c0 + (warp ? wsum[warp - 1] : 0) + incl - v;
    if (f < n_frames) {
      offsets[f] = excl;
      int cnt = valid ? npk : -1;
      if (valid && (long long)excl + npk > (long long)out_cap) {
        cnt = -1;
        P.flags[f] |= OVF_OUTPUT;
      }
      counts[f] = cnt;
      if (flags_out) flags_out[f] = P.flags[f];
    }
    __syncthreads();
    if (tid == 0) carry = c0 + wsum[31];
    __syncthreads();
  }
  mx = __reduce_max_sync(0xffffffffu, mx);
  if (lane == 0 && mx) atomicMax(&P.need[NEED_RINGS], mx);
  mxr = __reduce_max_sync(0xffffffffu, mxr);
  if (lane == 0 && mxr) atomicMax(&P.need[NEED_RIDGES], mxr);
  if (tid == 0) {
    offsets[n_frames] = carry;
    if (base_out) *base_out = carry;
  }
}

// Copies each valid frame's rings from the per-frame scratch to the caller's buffer at its
// offset (16-byte words; the destination may be mapped host memory on the host path).
__global__ void __launch_bounds__(128) k_copy(Params P, Ring* __restrict__ out, const int* __restrict__ counts,
                                              const int* __restrict__ offsets) {
  const int f = blockIdx.x, n = counts[f];
  if (n <= 0) return;
  RD_CHECK(n <= P.ring_cap, CK_EMIT);
  const uint4* src = reinterpret_cast<const uint4*>(P.rings + (int64_t)f * P.ring_cap);
  uint4* dst = reinterpret_cast<uint4*>(out + offsets[f]);
  for (int i = threadIdx.x; i < 4 * n; i += blockDim.x) dst[i] = src[i];
}

cudaError_t launch_emit(int n_frames, const Params& P, void* out, int out_cap, int* counts, int* offsets,
                        const int* base_in, int* base_out, int* flags_out, cudaStream_t st) {
  k_scan<<<1, 1024, 0, st>>>(P, n_frames, out_cap, counts, offsets, base_in, base_out, flags_out);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  k_copy<<<n_frames, 128, 0, st>>>(P, reinterpret_cast<Ring*>(out), counts, offsets);
  return cudaGetLastError();
}

}  // namespace rd
