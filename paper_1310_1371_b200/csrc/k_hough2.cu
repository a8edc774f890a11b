// k_hough2.cu — K2 (persistent form): directed voting, hotspot registration, radius-
// dependent smoothing with 1/r normalisation and 3x3x3 peak extraction.
//
// Rows A5-A8 of DESIGN.md §1 (SI steps 2-4, PAPER.md:931-978;
// range extension PAPER.md:998-1001).  Persistent CTAs (MINB per SM) take (frame, T x T
// tile) work items from a global counter.  For its tile a CTA sweeps r upward G levels
// per step, keeping on chip G levels of packed counters (CB = 1 or 2 bytes) over the tile
// + (K_max+1) halo and the hotspot lists of the last G + 2 levels (the paper's rolling
// level window).  The tile's ray list (routed by K1.5) arrives by bulk
// copies: every entry's 2-byte level interval below 255 levels (R16), else the first rcap
// rays whole.  A step has three phases separated by CTA barriers:
//   (1) votes: one thread per active ray (ridge pixel x sense of rho) casts its votes for
//       the G levels of the step; the atomic that lifts a counter past T_raw registers the
//       hotspot;
//   (2) S at each hotspot — lanes over window rows, dp4a against the
//       step's weight words (bulk-copied a step ahead) — and the candidate test
//       S > T_norm(r) in the same pass;
//   (3) every second step the rays active in the next two steps are listed; the step's
//       level buffers are cleared by one bulk copy of zeros on the TMA engine (the paper
//       resets the cells it registered, PAPER.md:426-434 — with byte counters a whole-buffer
//       clear is cheaper than tracking the touched words), which the next step's votes wait
//       for on an mbarrier; 3x3x3 peak extraction of the levels whose upper neighbour is
//       complete, one warp per candidate.
// Byte counters (CB = 1) are exact while no counter passes 255: the atomic that finds 255
// (P.u8_limit; lower only in tests) marks the frame, whose K2 results are then discarded and recomputed by the CB = 2
// instance (k_redo_reset + the redo list), so results never depend on the counter width.
// The shared-memory layout is computed on the host (Params::k2o, constant bank).  Only
// peak records (and optional debug hotspots) leave the SM.
#include <algorithm>
#include <type_traits>

#include "k_hough_common.cuh"
#include "rd_internal.cuh"

namespace rd {

namespace {

inline size_t al16(size_t v) { return (v + 15) & ~size_t(15); }

#ifndef RD_K2_SETUP3
#define RD_K2_SETUP3 1   // list the next step's rays in phase (3) (1: first, 2: after the clear) instead of (2)
#endif
#ifndef RD_K2_HSL
#define RD_K2_HSL 0
#endif
#ifndef RD_K2_HSL_MIN
#define RD_K2_HSL_MIN 2   // fewest lanes per hotspot in the byte-counter S phase (8: 14.75, 4: 14.19, 2: 13.95, 1: 13.95 us/frame)
#endif
#ifndef RD_K2_HSL_TGT
#define RD_K2_HSL_TGT 32   // lanes per hotspot: the widest hsl with hsl x (hotspots per warp) <= this (16: 14.29, 64: 14.94, 32: 13.99 us/frame)
#endif
#ifndef RD_K2_LP
#define RD_K2_LP 2   // steps per active-ray listing (rays idle in one step of the pair vote masked)
#endif
constexpr int LP = RD_K2_LP;

constexpr int HSL = RD_K2_HSL;   // byte-counter S tasks: lanes per hotspot (power of two <= 32; 0: per step)
constexpr int SMALL_K = 7;   // window rows 2K+1 <= 15: a half-warp per hotspot
// timing ablations (RD_K2_ABLATE bits, see Params::ablate) exist in profiling builds only
#ifdef RD_K2_PROF
#define ABL P.ablate
#else
#define ABL 0
#endif

}  // namespace
using namespace hk;

// Host: the K2 shared-memory layout for (G, threads, counter bytes) with the capacities in
// P (hot_cap, entry_cap, k2_rcap); returns the bytes.
size_t k_hough2_layout(Params& P, int G, int nt, int cb) {
  K2Layout& L = P.k2o;
  const int NSLOT = G + 2;
  (void)nt;
  const int hot_cap = P.hot_cap, nlev = P.n_levels;
  L.cb = cb;
  L.raws = P.k2ty + 2 * P.hal;   // rows
  L.rawc = P.k2t + 2 * P.hal;    // columns
  // row pitch of an odd number of 32-bit words: the rows of a window fall in distinct banks
  const int cpw = 4 / cb;   // cells per word
  L.rawp = ((L.rawc + cpw - 1) / cpw) | 1;
  L.rawp *= cpw;
  L.lvlc = (L.raws * L.rawp + 15) & ~15;   // 16-byte aligned level buffers (bulk clears)
  size_t o = 0;
  L.raw = o;   o = al16(o + (size_t)cb * G * L.lvlc);
  L.hS = o;    o = al16(o + 8 * (size_t)NSLOT * hot_cap);
  L.sd = o;    o = al16(o + 16 * (size_t)P.k2_rcap);
  L.rr = o;    o = al16(o + 4 * (size_t)P.k2_rcap);
  L.xy = o;    o = al16(o + 4 * (size_t)P.k2_rcap);
  L.rr16 = o;  o = al16(o + (P.k2_rr16 ? 2 * (size_t)P.entry_cap : 0));   // every entry's 2-byte interval
  L.hcell = o; o = al16(o + 2 * (size_t)NSLOT * hot_cap);
  // byte counters keep a hotspot's raw count in the low byte of its S word and take their
  // S tasks straight from the level lists: no raw or task arrays
  L.hraw = o;  o = al16(o + (cb == 1 ? 0 : 2 * (size_t)NSLOT * hot_cap));
  L.task = o;  o = al16(o + (cb == 1 ? 0 : 2 * (size_t)G * hot_cap));
  L.cand = o;  o = al16(o + 2 * (size_t)G * hot_cap);
  L.cdef = o;  o = al16(o + 2 * 2 * (size_t)hot_cap);
  L.act = o;   o = al16(o + 2 * (size_t)P.entry_cap);   // one list: written in phase (2), read in (1)
  L.hcnt = o;  o = al16(o + 4 * (size_t)(nlev + 16));
  L.w = o;     o = al16(o + 2 * (size_t)nlev * P.wstride);
  L.wst = o;   o = al16(o + (cb == 1 ? 32 * (size_t)P.wp_nw * G : 0));   // the step's dp4a weight words (bulk copy)
  L.k = o;     o = al16(o + 4 * (size_t)nlev);
  L.tn = o;    o = al16(o + 8 * (size_t)nlev);
  L.dummy = o; o = al16(o + 4 * 32);
  L.mbar = o;  o = al16(o + 16);         // [0] the tile's bulk ray copies, [1] the level-buffer clear
  L.total = (int)o;
  L.rawp_magic = (uint32_t)((1ull << 32) / (uint64_t)L.rawp + 1);
  return o;
}

template <bool kWide, int G, int NT, int MINB, int CB, bool R16>
__global__ void __launch_bounds__(NT, MINB) k_hough2(const __grid_constant__ Params P, int n_frames) {
  constexpr int NSLOT = G + 2;
  constexpr int NW = NT / 32;
  constexpr int CSH = CB == 1 ? 2 : 1;          // log2(cells per 32-bit word)
  constexpr int BITS = 8 * CB;
  constexpr uint32_t CMASK = CB == 1 ? 0xFFu : 0xFFFFu;
  constexpr unsigned FULL = 0xffffffffu;
  typedef typename std::conditional<CB == 1, uint8_t, uint16_t>::type cell_t;
  extern __shared__ __align__(16) unsigned char smem[];
#define SM(type, field) reinterpret_cast<type*>(smem + P.k2o.field)
  uint32_t* raw32 = SM(uint32_t, raw);          // [G] levels of packed counters
  cell_t* rawc = SM(cell_t, raw);
  unsigned long long* hS = SM(unsigned long long, hS);   // [NSLOT][hot_cap] S
  double2* sd = SM(double2, sd);                // [rcap] the tile's rays: (s*dx, s*dy)
  uint32_t* rr_s = SM(uint32_t, rr);            // [rcap] level interval ra | rb<<16
  uint32_t* sxy = SM(uint32_t, xy);             // [rcap] x | y<<16 (frame coordinates)
  uint16_t* rr16 = SM(uint16_t, rr16);          // [entry_cap] ra | rb<<8 of every entry (Params::k2_rr16)
  uint16_t* hcell = SM(uint16_t, hcell);        // [NSLOT][hot_cap] iy<<8 | ix (ring coordinates)
  uint16_t* hraw = SM(uint16_t, hraw);          // [NSLOT][hot_cap] raw count
  uint16_t* tasks = SM(uint16_t, task);         // [G*hot_cap] g<<12 | h (small K front, large K back)
  uint16_t* cand = SM(uint16_t, cand);          // [G*hot_cap] g<<12 | h
  uint16_t* cdef = SM(uint16_t, cdef);          // [2][hot_cap] h, top level of a step
  uint16_t* act = SM(uint16_t, act);            // [entry_cap] rays active in the step (next step's from phase 2)
  int* hcnt = SM(int, hcnt);                    // [nlev] hotspots per level + counters
  uint16_t* tW = SM(uint16_t, w);               // [nlev][wstride] w_r(d)
  int* tK = SM(int, k);                         // [nlev] K_r
  double* tTn = SM(double, tn);                 // [nlev] T_norm(r)
  uint32_t* dummy_w = SM(uint32_t, dummy);      // [32] targets of masked-out votes (+0)
  uint64_t* mbar = SM(uint64_t, mbar);          // bulk ray copies of a tile
#undef SM
  const int nlev = P.n_levels;
  int* cnt = hcnt + nlev;
  int* s_flags = cnt + 0;
  int* s_nact = cnt + 2;    // [2] by step parity
  int* s_ntask = cnt + 4;   // [2] small-K tasks from the front, large-K from the back
  int* s_ncand = cnt + 6;
  int* s_ndef = cnt + 8;    // [2] by step parity
  int* s_item = cnt + 12;
  int* s_ovf = cnt + 13;    // a byte counter passed 255

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int TX = P.k2t, TY = P.k2ty, hal = P.hal, hot_cap = P.hot_cap;
  const int rawp = P.k2o.rawp, lvlc = P.k2o.lvlc, rcap = P.k2_rcap, ecap = P.entry_cap;
  const int ntiles = P.ntx * P.nty;
  const uint32_t T_raw = (uint32_t)P.T_raw;
  // CB = 2 is also the redo pass: work items are then the tiles of the frames in the redo list
  const bool redo_pass = CB == 2 && P.redo_list != nullptr;
  const int n_work_frames = redo_pass ? P.redo_list[0] : n_frames;

  unsigned long long t_acc[6] = {0, 0, 0, 0, 0, 0};
  int need_e = 0, need_h = 0;   // capacities the CTA's tiles needed (rd_query_overflow)
  long long t_last = clock64();
#ifdef RD_K2_PROF   // per-phase cycle accounting (rd_phase_cycles); compiled in on request only
#define PMARK(i)                                      \
  if (P.prof && tid == 0) {                           \
    const long long t_ = clock64();                   \
    t_acc[i] += (unsigned long long)(t_ - t_last);    \
    t_last = t_;                                      \
  }
#else
#define PMARK(i)
#endif

  // once per CTA: level tables, zeroed counters and raw levels (the undo keeps them zero)
  for (int i = tid; i < nlev * P.wstride; i += NT) tW[i] = (uint16_t)P.lvlW[i];
  for (int i = tid; i < nlev; i += NT) {
    tK[i] = P.lvlK[i];
    tTn[i] = P.lvlTn[i];
  }
  {
    uint4* r4 = reinterpret_cast<uint4*>(raw32);
    for (int i = tid; i < (CB * G * lvlc) / 16; i += NT) r4[i] = make_uint4(0, 0, 0, 0);
  }
  for (int i = tid; i < 32; i += NT) {
    if (i < 16) cnt[i] = 0;
    dummy_w[i] = 0;
  }
  // the tile's resident rays arrive by bulk copies (TMA engine) when every array slice is
  // 16-byte aligned (entry_cap and rcap multiples of 4), else by per-thread cp.async
  const bool bulk = ((P.entry_cap | rcap) & 3) == 0;
  uint32_t mpar = 0;   // mbarrier phase
  uint32_t cpar = 0;   // clear mbarrier phase
  bool clear_pending = false;   // bulk copies on mbar[1] (clear, weight words) are in flight
  if (tid == 0) {
    mbar_init(mbar, 1);
    mbar_init(mbar + 1, 1);
    mbar_fence_init();
  }
  __syncthreads();
  // byte counters: the dp4a weight words of a step's levels (all four row alignments, one
  // contiguous block of the table) are bulk-copied into shared memory one step ahead, with the
  // clear, on mbar[1]; the first tile's first step's here
  const uint32_t wlev = CB == 1 ? 32u * (uint32_t)P.wp_nw : 0u;   // bytes per level
  auto issue_w = [&](int L0s) {   // (one thread; the caller has armed mbar[1] for the bytes)
    const uint32_t nb = wlev * (uint32_t)min(G, nlev - L0s);
    if (nb) bulk_g2s(smem + P.k2o.wst, P.lvlWP + (size_t)L0s * 8 * P.wp_nw, nb, mbar + 1);
  };
  if (CB == 1) {
    if (tid == 0) {
      mbar_expect_tx(mbar + 1, wlev * (uint32_t)min(G, nlev));
      issue_w(0);
    }
    clear_pending = true;
  }

  for (;;) {
    if (tid == 0) *s_item = atomicAdd(redo_pass ? P.k2_work + 1 : P.k2_work, 1);
    for (int i = tid; i < nlev; i += NT) hcnt[i] = 0;
    __syncthreads();
    const int item = *s_item;
    if (item >= n_work_frames * ntiles) break;
    const int fw = item / ntiles, tile = item - fw * ntiles;
    const int f = redo_pass ? P.redo_list[1 + fw] : fw;
    const int tyi = tile / P.ntx, txi = tile - tyi * P.ntx;
    const int X0 = txi * TX, Y0 = tyi * TY;
    const int RX0 = X0 - hal, RY0 = Y0 - hal;   // raw buffer origin (frame coordinates)
    const int64_t tl = (int64_t)f * ntiles + tile;
    const int ne_all = P.ray_count[tl];
    const int ne = min(ne_all, P.entry_cap);
    need_e = max(need_e, ne_all);   // (one global atomicMax per CTA at exit)
    const int64_t gbase = tl * P.entry_cap;
    int my_hot = 0;   // interior hotspots (the per-frame vote count comes from K1.5)

    auto rr_of16 = [&](int e) { const uint32_t v = rr16[e]; return (v & 0xFFu) | ((v >> 8) << 16); };
    // list the rays active in the LP steps starting at level L0s (count: s_nact[p])
    auto setup = [&](int L0s, int p) {
      const int Lhs = min(L0s + LP * G - 1, nlev - 1);
      for (int e0 = warp * 32; e0 < ne; e0 += NT) {
        const int e = e0 + lane;
        const uint32_t rr = e < ne ? (R16 ? rr_of16(e) : e < rcap ? rr_s[e] : __ldg(P.ray_r + gbase + e)) : 0xFFFFu;
        const bool a = (int)(rr & 0xFFFFu) <= Lhs && (int)(rr >> 16) >= L0s;
        const unsigned bal = __ballot_sync(FULL, a);
        if (!bal) continue;
        int base = 0;
        if (lane == 0) base = atomicAdd(&s_nact[p], __popc(bal));
        base = __shfl_sync(FULL, base, 0);
        RD_CHECK(!a || base + __popc(bal & lanemask_lt()) < ecap, CK_K2_LIST);
        if (a) act[base + __popc(bal & lanemask_lt())] = (uint16_t)e;
      }
    };
    // the tile's rays (up to rcap) become resident in shared memory
    const int nres = min(ne, rcap);
    if (R16) {   // every entry's interval (2 bytes) by one bulk copy; no resident rays (Params::k2_rr16)
      if (ne > 0) {
        if (tid == 0) {
          const int n8 = (ne + 7) & ~7;   // whole 16-byte lines (n8 <= entry_cap, a multiple of 8)
          fence_proxy_async_smem();
          mbar_expect_tx(mbar, (uint32_t)(2 * n8));
          bulk_g2s(rr16, reinterpret_cast<const uint16_t*>(P.ray_r) + gbase, 2u * n8, mbar);
        }
        mbar_wait(mbar, mpar);
        mpar ^= 1u;
      }
    } else if (bulk) {
      if (nres > 0) {
        if (tid == 0) {
          const int n4 = (nres + 3) & ~3;   // x | y and the intervals: whole 16-byte lines (n4 <= rcap)
          fence_proxy_async_smem();         // this CTA's reads of the previous tile's rays (behind a barrier) first
          mbar_expect_tx(mbar, (uint32_t)(16 * nres + 8 * n4));
          bulk_g2s(sd, P.ray_d + gbase, 16u * nres, mbar);
          bulk_g2s(sxy, P.ray_xy + gbase, 4u * n4, mbar);
          bulk_g2s(rr_s, P.ray_r + gbase, 4u * n4, mbar);
        }
        mbar_wait(mbar, mpar);
        mpar ^= 1u;
      }
    } else {
      for (int e = tid; e < nres; e += NT) {
        cp_async16(&sd[e], P.ray_d + gbase + e);
        cp_async4(&sxy[e], P.ray_xy + gbase + e);
        cp_async4(&rr_s[e], P.ray_r + gbase + e);
      }
      cp_async_wait_all();
    }
    __syncthreads();
    setup(0, 0);
    PMARK(0);

    for (int L0 = 0, step = 0; L0 < nlev; L0 += G, ++step) {
      const int Lhi = min(L0 + G - 1, nlev - 1);
      const int par = step & 1, lpar = (step / LP) & 1;   // step parity, listing parity
      const bool list_next = (step + 1) % LP == 0;       // this step lists the next LP steps' rays
      __syncthreads();
      PMARK(1);
      if (tid == 0) {   // counters whose last reader is behind the barrier above; first used after the next
        s_nact[lpar ^ 1] = 0;
        s_ncand[0] = 0;
        s_ndef[par] = 0;
      }
#ifdef RD_CHECKED
      if (P.jitter) __nanosleep(((unsigned)(warp * 2654435761u + step * 40503u + blockIdx.x * 97u) >> 7) & 2047u);
#endif
      if (clear_pending) {   // the previous step's levels are zero again, this step's weight words staged
        mbar_wait(mbar + 1, cpar);
        cpar ^= 1u;
        clear_pending = false;
      }
      // ---------------- (1) votes of levels L0..Lhi
      {
        const int nact = s_nact[lpar];
        const double rb0 = (double)(P.r_lo + L0);
        int slot_of[G];   // hotspot-list slot of each level of the step
#pragma unroll
        for (int g = 0; g < G; ++g) slot_of[g] = (L0 + g) % NSLOT;
        const uint32_t raw_base = smem_u32(raw32);
        const uint32_t dummy = smem_u32(dummy_w) + 4u * lane;   // masked votes add 0 to a private word
        const int bx0 = max(0, -RX0), bxs = min(P.k2o.rawc - 1, P.W - 1 - RX0) - bx0;
        const int by0 = max(0, -RY0), bys = min(P.k2o.raws - 1, P.H - 1 - RY0) - by0;
        bool ovf = false;
        // the votes of GL levels (GL = G, or 1 for a last step with a single level: no masked
        // work for the absent levels)
        auto run_votes = [&](auto GLc) {
          constexpr int GL = decltype(GLc)::value;
          if (ABL & 16) return;   // timing experiments only: no votes
          // a chunk's ray entries are loaded one chunk ahead (most come from L2: the load of
          // the next chunk overlaps this chunk's votes; 15.82 vs 15.96 us/frame on cfg3)
          auto load_ray = [&](int i, double2& d, uint32_t& xy, uint32_t& rr) {
            d = make_double2(0.0, 0.0);
            xy = 0u;
            rr = 0xFFFFu;   // empty interval
            if (i < nact) {
              const int e = act[i];
              RD_CHECK(e >= 0 && e < ne, CK_K2_RAY);
              if (R16) {   // pixel and direction from L2 (the interval is read at use, below)
                xy = __ldg(P.ray_xy + gbase + e);
                d = __ldg(P.ray_d + gbase + e);
              } else if (e < rcap) {
                d = sd[e];
                xy = sxy[e];
                rr = rr_s[e];
              } else {   // beyond the resident capacity: from global memory
                xy = __ldg(P.ray_xy + gbase + e);
                d = __ldg(P.ray_d + gbase + e);
                rr = __ldg(P.ray_r + gbase + e);
              }
            }
          };
          double2 nd;
          uint32_t nxy, nrr;
          load_ray(warp * 32 + lane, nd, nxy, nrr);
          for (int i0 = warp * 32; i0 < nact; i0 += NT) {
            const double2 d = nd;
            const uint32_t xy = nxy;
            uint32_t rr = nrr;
            if (R16) {   // the resident interval, not carried in the prefetch registers
              const int i = i0 + lane;
              rr = i < nact ? rr_of16(act[i]) : 0xFFFFu;
            }
            if (i0 + NT < nact) load_ray(i0 + NT + lane, nd, nxy, nrr);
            // levels ga..gb of the step lie inside the ray's interval (empty: ga > gb); compared with
            // each g directly (chained predicates: a level bitmask cost ~10 more instructions a chunk)
            const int ga = (int)(rr & 0xFFFFu) - L0, gb = (int)(rr >> 16) - L0;
            const double dx = d.x, dy = d.y;
            const int xr = (int)(xy & 0xFFFFu) - RX0, yr = (int)(xy >> 16) - RY0;
            // targets of the G levels, branch-free: a vote counts if its level is in the ray's
            // interval and its cell lies in the raw buffer and in the frame (cells outside a
            // level's box, tile + K_r + 1, are never read by that level's windows; the clear
            // resets them)
            uint32_t addr[GL], sh[GL], old[GL];
            const uint32_t pb = raw_base + (uint32_t)(CB * (yr * rawp + xr));   // the ray's own cell (bytes)
            const int ux = xr - bx0, uy = yr - by0;
            const double hx = copysign(0.5, dx), hy = copysign(0.5, dy);   // (r_lo >= 1)
            int qx = 0, qy = 0;   // (32: timing experiment only, integer fixed-point targets)
            if (ABL & 32) {
              qx = __double2int_rn(dx * 65536.0);
              qy = __double2int_rn(dy * 65536.0);
            }
  #pragma unroll
            for (int g = 0; g < GL; ++g) {
              const double rd = rb0 + (double)g;
              int ox, oy;
              if (ABL & 32) {
                ox = ((P.r_lo + L0 + g) * qx + 32768) >> 16;
                oy = ((P.r_lo + L0 + g) * qy + 32768) >> 16;
              } else {
                // llround: r > 0, so the product has the direction's sign and the half is the ray's
                ox = __double2int_rz(__dadd_rz(__dmul_rn(rd, dx), hx));
                oy = __double2int_rz(__dadd_rz(__dmul_rn(rd, dy), hy));
              }
              const bool ok = (g >= ga) & (g <= gb) & ((unsigned)(ux + ox) <= (unsigned)bxs) &
                              ((unsigned)(uy + oy) <= (unsigned)bys);
              const uint32_t bc = pb + (uint32_t)(g * lvlc * CB) + (uint32_t)(CB * (oy * rawp + ox));   // byte address
              // masked votes: shift 32 (shl/shr clamp to 0) on the lane's dummy word
              sh[g] = ok ? (bc & 3u) * 8u : 32u;
              addr[g] = ok ? (bc & ~3u) : dummy;
            }
  #pragma unroll
            for (int g = 0; g < GL; ++g)
              RD_CHECK(sh[g] == 32u ? addr[g] == dummy : (addr[g] - raw_base >= (uint32_t)(g * lvlc * CB) &&
                                                          addr[g] - raw_base < (uint32_t)((g + 1) * lvlc * CB)),
                       CK_K2_VOTE);
  #pragma unroll
            for (int g = 0; g < GL; ++g)
              old[g] = (ABL & 8) ? 0u : atom_add_shared(addr[g], shl_clamp(1u, sh[g]));   // (8: no atomics)
            uint32_t omax = 0;
  #pragma unroll
            for (int g = 0; g < GL; ++g) {
              const uint32_t oc = shr_clamp(old[g], sh[g]) & CMASK;   // 0 for masked votes
              omax = max(omax, oc);
              if (oc == T_raw) {   // this vote lifted the counter past T_raw (T_raw >= 1)
                const int cell = (int)((addr[g] - raw_base - (uint32_t)(g * lvlc * CB)) >> (CB - 1)) + (int)(sh[g] / BITS);
                const int cy = (int)__umulhi((uint32_t)cell, P.k2o.rawp_magic), cx = cell - cy * rawp;
                const int ix = cx - (hal - 1), iy = cy - (hal - 1);
                if ((unsigned)ix >= (unsigned)(TX + 2) || (unsigned)iy >= (unsigned)(TY + 2)) continue;   // not in the ring
                const int li = L0 + g;
                RD_CHECK(li < nlev && iy < TY + 2 && ix < TX + 2 && ix < 256, CK_K2_LIST);
                const int h = atomicAdd(&hcnt[li], 1);
                if (h < hot_cap) {
                  hcell[slot_of[g] * hot_cap + h] = (uint16_t)((iy << 8) | ix);
                  if (CB == 2) {   // (byte counters take their S tasks straight from the level lists)
                    const int slot = tK[li] <= SMALL_K ? atomicAdd(&s_ntask[0], 1)
                                                       : G * hot_cap - 1 - atomicAdd(&s_ntask[1], 1);
                    RD_CHECK(slot >= 0 && slot < G * hot_cap, CK_K2_TASK);
                    tasks[slot] = (uint16_t)((g << 12) | h);
                  }
                } else {
                  atomicOr(s_flags, OVF_HOTSPOTS);
                }
              }
            }
            if (CB == 1) ovf |= omax >= (uint32_t)P.u8_limit;
          }
        };
        const int nl = min(G, nlev - L0);
        if (nl == 1 && G > 1) run_votes(std::integral_constant<int, 1>{});
        else run_votes(std::integral_constant<int, G>{});
        if (CB == 1 && __any_sync(FULL, ovf) && lane == 0) *s_ovf = 1;
      }
      __syncthreads();
      PMARK(2);
#ifdef RD_CHECKED
      if (P.jitter) __nanosleep(((unsigned)(warp * 97u + step * 7919u + blockIdx.x * 2654435761u) >> 8) & 2047u);
#endif
      // ---------------- (2) the next step's rays; S = sum_i w(i) sum_j w(j) raw(y+i, x+j) at
      //     each hotspot and the candidate test
      {
#if !RD_K2_SETUP3
        if (L0 + G < nlev && list_next) setup(L0 + G, lpar ^ 1);
#endif
        if (CB == 1) {
          // byte counters: HSL lanes per hotspot, lane hl sums window rows hl, hl + HSL, ...;
          // a row is summed over whole 32-bit words with dp4a against the level's byte-plane
          // weights for the row's alignment (w = 64 wh + wl): exact integer S as below
          // weight words per row: (3 + 2K + 1 + 3) / 4 <= 9 for K <= 15; the task loop is
          // instantiated for 3, 5, 7 and 9 words and the step takes the narrowest that holds its
          // levels' windows (rows are read NWW words wide unconditionally, see below)
          // S tasks: the step's level lists back to back (task t -> level g, list index h)
          // the step's level counts, once (task decode below uses the prefix sums)
          int pre[G];   // pre[g] = tasks of levels 0 .. g
          int ntask = 0;
#pragma unroll
          for (int g = 0; g < G; ++g) {
            ntask += L0 + g < nlev ? min(hcnt[L0 + g], hot_cap) : 0;
            pre[g] = ntask;
          }
          if (ABL & 4) ntask = 0;
#if RD_K2_HSL == 0
          // lanes per hotspot: the widest power of two that still gives every warp its share
          // (hsl = 32 >> lgs with lgs = ceil(log2(per_warp)) capped: shifts, no loop and no division)
          const int per_warp = (ntask + NW - 1) / NW;
          static_assert(RD_K2_HSL_TGT == 32 && (RD_K2_HSL_MIN & (RD_K2_HSL_MIN - 1)) == 0, "closed form below");
          constexpr int LGS_MAX = RD_K2_HSL_MIN == 1 ? 5 : RD_K2_HSL_MIN == 2 ? 4 : RD_K2_HSL_MIN == 4 ? 3 : RD_K2_HSL_MIN == 8 ? 2 : RD_K2_HSL_MIN == 16 ? 1 : 0;
          const int lgs = per_warp <= 1 ? 0 : min(32 - __clz(per_warp - 1), LGS_MAX);
          const int hsl = 32 >> lgs;
#else
          constexpr int hsl = HSL;
          constexpr int lgs = HSL == 32 ? 0 : HSL == 16 ? 1 : HSL == 8 ? 2 : HSL == 4 ? 3 : HSL == 2 ? 4 : 5;
#endif
          const int NGW = 1 << lgs;   // hotspots per warp pass
          const int grp = lane >> (5 - lgs), hl = lane & (hsl - 1);
          auto run_s = [&](auto NWc) {
          constexpr int NWW = decltype(NWc)::value;
          for (int t0 = NGW * warp; t0 < ntask; t0 += NGW * NW) {
            const int t = t0 + grp;
            const bool valid = t < ntask;
            const int tv = valid ? t : t0;
            int g = 0, h = tv;
#pragma unroll
            for (int gg = 0; gg < G - 1; ++gg)
              if (tv >= pre[gg]) g = gg + 1, h = tv - pre[gg];
            const int tk = (g << 12) | h;
            const int li = L0 + g, sl = li % NSLOT;
            const int K = tK[li];
            const int c = hcell[sl * hot_cap + h];
            const int iy = c >> 8, ix = c & 0xFF;
            const int cx0 = ix - 1 + hal - K;        // first window column (raw-local)
            const int al = cx0 & 3, nw = (al + 2 * K + 4) >> 2;
            const uint2* wp = reinterpret_cast<const uint2*>(smem + P.k2o.wst) + (size_t)(g * 4 + al) * P.wp_nw;
            uint32_t wl[NWW], wh[NWW];   // (bulk-copied a step ahead: 32 B per level and word)
#pragma unroll
            for (int k = 0; k < NWW; ++k) {
              const uint2 w2 = wp[k];   // zero beyond the row's nw words (NWW <= wp_nw, which is odd)
              wl[k] = w2.x;
              wh[k] = w2.y;
            }
            const uint16_t* w = tW + li * P.wstride;
            const uint32_t* lvlw = raw32 + ((g * lvlc) >> 2);
            RD_CHECK(!valid || (g < G && h < hot_cap && iy - 1 + hal - K >= 0 && iy - 1 + hal + K < P.k2o.raws &&
                                cx0 - al >= 0 && cx0 - al + 4 * nw <= rawp * CB && nw <= NWW),
                     CK_K2_WINDOW);
            unsigned long long acc = 0;
            if (valid && !(ABL & 1)) {
              for (int row = hl; row <= 2 * K; row += hsl) {
                const uint32_t* rowp = lvlw + (((iy - 1 + hal + row - K) * rawp + cx0 - al) >> 2);
                uint32_t lo = 0, hi = 0;
                // every word of the row is read unconditionally (a branch per word serialised
                // the loads: 13.90 vs 13.31 us/frame): words k >= nw have zero weights (wl = wh
                // = 0) and lie inside shared memory (the raw levels are followed by the hotspot
                // arrays), so they add 0
#pragma unroll
                for (int k = 0; k < NWW; ++k) {
                  const uint32_t v = rowp[k];
                  lo = __dp4a(v, wl[k], lo);
                  hi = __dp4a(v, wh[k], hi);
                }
                acc += (unsigned long long)(hi * 64u + lo) * (unsigned long long)w[abs(row - K)];
              }
            }
#pragma unroll
            for (int o = hsl / 2; o > 0; o >>= 1) acc += __shfl_xor_sync(FULL, acc, o);
            const unsigned long long S = acc;
            if (valid && hl == 0) {
              const uint16_t rv = rawc[g * lvlc + (iy - 1 + hal) * rawp + (ix - 1 + hal)];
              hS[sl * hot_cap + h] = (S << 8) | rv;   // S < 2^46, raw < 256
              if (ix >= 1 && ix <= TX && iy >= 1 && iy <= TY) {   // interior hotspot
                ++my_hot;
                if (P.debug) {
                  const int kd = atomicAdd(&P.dbg_count[f], 1);
                  if (kd < P.dbg_cap) {
                    HotRec rec;
                    rec.r = P.r_lo + li; rec.y = Y0 - 1 + iy; rec.x = X0 - 1 + ix; rec.raw = rv;
                    rec.S = (long long)S;
                    P.dbg_hot[(int64_t)f * P.dbg_cap + kd] = rec;
                  } else {
                    atomicOr(&P.flags[f], OVF_DEBUG);
                  }
                }
                // candidate: r in [r_min, r_max] and S > T_norm(r);
                // the top level of the step waits for the next step's S of its upper neighbour
                if (li >= 1 && li <= nlev - 2 && (double)(long long)S > tTn[li]) {
                  if (li == Lhi) {
                    const int q = atomicAdd(&s_ndef[par], 1);
                    RD_CHECK(q < hot_cap, CK_K2_TASK);
                    cdef[par * hot_cap + q] = (uint16_t)h;
                  } else {
                    const int q = atomicAdd(s_ncand, 1);
                    RD_CHECK(q < G * hot_cap, CK_K2_TASK);
                    cand[q] = (uint16_t)tk;
                  }
                }
              }
            }
          }
          };
          // the widest window of the step's levels: its last level's (K_r = ceil(3 sigma(r)) does not
          // decrease with r: rd_create requires sig_a >= 0)
          const int Kst = tK[min(L0 + G - 1, nlev - 1)];
          const int nwst = (3 + 2 * Kst + 4) >> 2;
          if (nwst <= 3) run_s(std::integral_constant<int, 3>{});
          else if (nwst <= 5) run_s(std::integral_constant<int, 5>{});
          else if (nwst <= 7) run_s(std::integral_constant<int, 7>{});
          else run_s(std::integral_constant<int, 9>{});
        } else {
        const int nsmall = (ABL & 4) ? 0 : s_ntask[0], nlarge = (ABL & 4) ? 0 : s_ntask[1];
        const int half = lane >> 4;
        // small-K hotspots: a half-warp each; large-K: a warp each (lanes over window rows)
        const int nsp = (nsmall + 1) >> 1;
        for (int t = warp; t < nsp + nlarge; t += NW) {
          const bool small = t < nsp;
          int tk;
          bool valid = true;
          if (small) {
            const int ts = 2 * t + half;
            valid = ts < nsmall;
            tk = tasks[valid ? ts : 2 * t];
          } else {
            tk = tasks[G * hot_cap - 1 - (t - nsp)];
          }
          const int g = tk >> 12, h = tk & 0xFFF;
          const int li = L0 + g, sl = li % NSLOT;
          const int K = tK[li];
          const uint16_t* w = tW + li * P.wstride;
          const int c = hcell[sl * hot_cap + h];
          const int iy = c >> 8, ix = c & 0xFF;
          const cell_t* ctr = rawc + g * lvlc + (iy - 1 + hal) * rawp + (ix - 1 + hal);   // the hotspot's cell
          RD_CHECK(!valid || (g < G && h < hot_cap && iy - 1 + hal - K >= 0 && iy - 1 + hal + K < P.k2o.raws &&
                              ix - 1 + hal - K >= 0 && ix - 1 + hal + K < P.k2o.rawc),
                   CK_K2_WINDOW);
          const int sub = small ? (lane & 15) : lane;
          unsigned long long acc = 0;   // lane sum over window rows sub, sub + 32, ... (K > 15: 2K + 1 > 32 rows)
          if (valid && !(ABL & 1)) {
            for (int row = sub; row <= 2 * K; row += small ? 16 : 32) {
              const cell_t* rowp = ctr + (row - K) * rawp;
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
          }
          unsigned long long S;
          if (kWide) {
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
              const unsigned long long v = __shfl_xor_sync(FULL, acc, o);
              if (!(small && o == 16)) acc += v;
            }
            S = acc;
          } else {   // lane sums < 2^47 (K <= 48: at most 4 rows of < 2^44): 24-bit halves, single-instruction reductions
            const unsigned lo = (unsigned)(acc & 0xFFFFFFull), hi = (unsigned)(acc >> 24);
            unsigned slo, shi;
            if (small) {   // (warp-uniform branch) the two halves reduce separately
              const unsigned lo0 = __reduce_add_sync(FULL, half ? 0u : lo);
              const unsigned hi0 = __reduce_add_sync(FULL, half ? 0u : hi);
              const unsigned lo1 = __reduce_add_sync(FULL, half ? lo : 0u);
              const unsigned hi1 = __reduce_add_sync(FULL, half ? hi : 0u);
              slo = half ? lo1 : lo0;
              shi = half ? hi1 : hi0;
            } else {
              slo = __reduce_add_sync(FULL, lo);
              shi = __reduce_add_sync(FULL, hi);
            }
            S = ((unsigned long long)shi << 24) + slo;
          }
          if (valid && sub == 0) {
            hS[sl * hot_cap + h] = S;
            const uint16_t rv = *ctr;
            hraw[sl * hot_cap + h] = rv;
            if (ix >= 1 && ix <= TX && iy >= 1 && iy <= TY) {   // interior hotspot
              ++my_hot;
              if (P.debug) {
                const int kd = atomicAdd(&P.dbg_count[f], 1);
                if (kd < P.dbg_cap) {
                  HotRec rec;
                  rec.r = P.r_lo + li; rec.y = Y0 - 1 + iy; rec.x = X0 - 1 + ix; rec.raw = rv;
                  rec.S = (long long)S;
                  P.dbg_hot[(int64_t)f * P.dbg_cap + kd] = rec;
                } else {
                  atomicOr(&P.flags[f], OVF_DEBUG);
                }
              }
              // candidate: r in [r_min, r_max] and S > T_norm(r);
              // the top level of the step waits for the next step's S of its upper neighbour
              if (li >= 1 && li <= nlev - 2 && (double)(long long)S > tTn[li]) {
                if (li == Lhi) {
                  const int q = atomicAdd(&s_ndef[par], 1);
                  RD_CHECK(q < hot_cap, CK_K2_TASK);
                  cdef[par * hot_cap + q] = (uint16_t)h;
                } else {
                  const int q = atomicAdd(s_ncand, 1);
                  RD_CHECK(q < G * hot_cap, CK_K2_TASK);
                  cand[q] = (uint16_t)tk;
                }
              }
            }
          }
        }
        }   // CB == 2
      }
      __syncthreads();
      PMARK(3);
#ifdef RD_CHECKED
      if (P.jitter) __nanosleep(((unsigned)(warp * 40503u + step * 2654435761u + blockIdx.x * 31u) >> 9) & 2047u);
#endif
      // ---------------- (3) undo the step's counters, then peaks of levels L0-1 .. Lhi-1
      if (P.debug) {   // level fingerprints over the tile's own cells (each frame voxel once)
        const int x1 = min(X0 + TX, P.W), y1 = min(Y0 + TY, P.H), nx = x1 - X0, ncell = nx * (y1 - Y0);
        for (int g = 0; g < min(G, nlev - L0); ++g) {
          unsigned long long acc[3] = {0, 0, 0};
          for (int i = tid; i < ncell; i += NT) {
            const int yy = Y0 + i / nx, xx = X0 + i % nx;
            const unsigned long long c = rawc[g * lvlc + (yy - RY0) * rawp + (xx - RX0)];
            acc[0] += c;
            acc[1] += c * c;
            acc[2] += c * (unsigned long long)((long long)yy * P.W + xx);
          }
#pragma unroll
          for (int k = 0; k < 3; ++k) {
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) acc[k] += __shfl_xor_sync(FULL, acc[k], o);
            if (lane == 0 && acc[k]) atomicAdd(&P.dbg_fpr[((int64_t)f * nlev + L0 + g) * 3 + k], acc[k]);
          }
        }
        __syncthreads();   // read before the clear below
      }
      {
#if RD_K2_SETUP3 == 1
        if (L0 + G < nlev && list_next) setup(L0 + G, lpar ^ 1);
#endif
        {   // clear the step's level buffers: one bulk copy of zeros (TMA engine)
          if (tid == 0) {
            const uint32_t nb = (uint32_t)(CB * min(G, nlev - L0) * lvlc);   // the levels the step used
            const int Ln = L0 + G < nlev ? L0 + G : 0;   // the next step (of this tile or the next one)
            fence_proxy_async_smem();   // the S phase's reads (behind the barrier above) before the async writes
            mbar_expect_tx(mbar + 1, nb + wlev * (uint32_t)min(G, nlev - Ln));
            bulk_g2s(raw32, P.zeros, nb, mbar + 1);
            issue_w(Ln);
          }
          clear_pending = true;
        }
        if (tid == 0) {
          s_ntask[0] = 0;
          s_ntask[1] = 0;
        }
#if RD_K2_SETUP3 == 2
        if (L0 + G < nlev && list_next) setup(L0 + G, lpar ^ 1);
#endif
        const int nd = (L0 > 0 && !(ABL & 2)) ? s_ndef[par ^ 1] : 0, nc = (ABL & 2) ? 0 : s_ncand[0];
        for (int p = warp; p < nd + nc; p += NW) {
          int lc, h;
          if (p < nd) {
            lc = L0 - 1;
            h = cdef[(par ^ 1) * hot_cap + p];
          } else {
            const int tk = cand[p - nd];
            lc = L0 + (tk >> 12);
            h = tk & 0xFFF;
          }
          const int sc = lc % NSLOT;
          RD_CHECK(h < min(hcnt[lc], hot_cap) && lc >= 1 && lc <= nlev - 2, CK_K2_NMS);
          const int c = hcell[sc * hot_cap + h];
          const int iy = c >> 8, ix = c & 0xFF;
          constexpr int SSH = CB == 1 ? 8 : 0;   // byte counters: raw count in the low byte
          const unsigned long long hw = hS[sc * hot_cap + h];
          const long long S = (long long)(hw >> SSH);
          const long long rc = P.r_lo + lc;
          bool beaten = false;
#pragma unroll
          for (int dl = -1; dl <= 1; ++dl) {
            const int l = lc + dl, sl = l % NSLOT;
            const int n = min(hcnt[l], hot_cap);
            const long long ru = P.r_lo + l;
            for (int j = lane; j < n; j += 32) {
              const int u = hcell[sl * hot_cap + j];
              const int dy = (u >> 8) - iy, dx = (u & 0xFF) - ix;
              if (dy < -1 || dy > 1 || dx < -1 || dx > 1 || (dl == 0 && dy == 0 && dx == 0)) continue;
              const long long Su = (long long)(hS[sl * hot_cap + j] >> SSH);
              const long long lhs = S * ru, rhs = Su * rc;
              const bool v_first = dl > 0 || (dl == 0 && (dy > 0 || (dy == 0 && dx > 0)));
              if (!(lhs > rhs || (lhs == rhs && v_first))) beaten = true;
            }
          }
          if (__any_sync(FULL, beaten)) continue;
          if (lane == 0) {
            const int kk = atomicAdd(&P.peak_count[f], 1);
            if (kk < P.ring_cap) {
              Peak pk;
              pk.x = X0 - 1 + ix; pk.y = Y0 - 1 + iy; pk.r = (int)rc; pk.raw = CB == 1 ? (int)(hw & 0xFFu) : hraw[sc * hot_cap + h]; pk.S = S;
              P.peaks[(int64_t)f * P.ring_cap + kk] = pk;
            } else {
              atomicOr(&P.flags[f], OVF_RINGS);
            }
          }
        }
      }
      PMARK(4);
    }
    // ---------------- per-frame counters of this tile
    if (warp == 0) {   // hotspots per level this tile needed (rd_query_overflow)
      int m = 0;
      for (int i = lane; i < nlev; i += 32) m = max(m, hcnt[i]);
      need_h = max(need_h, __reduce_max_sync(FULL, m));
    }
    my_hot = __reduce_add_sync(FULL, my_hot);
    if (lane == 0 && my_hot) atomicAdd(&P.stats[f].hotspots, (unsigned long long)my_hot);
    __syncthreads();
    if (tid == 0) {
      if (*s_flags) atomicOr(&P.flags[f], *s_flags);
      if (CB == 1 && *s_ovf) atomicExch(&P.redo[f], 1);
      for (int i = 0; i < 14; ++i)
        if (i != 12) cnt[i] = 0;   // flags and all step counters, for the next tile
      if (P.prof) atomicAdd(&P.prof[15], 1ull);
    }
  }
  if (clear_pending) mbar_wait(mbar + 1, cpar);   // no bulk write may outlive the CTA
  if (tid == 0 && need_e) atomicMax(&P.need[NEED_ENTRIES], need_e);
  if (tid == 0 && need_h) atomicMax(&P.need[NEED_HOTSPOTS], need_h);
  if (P.prof && tid == 0) {
#pragma unroll
    for (int i = 0; i < 6; ++i) atomicAdd(&P.prof[i], t_acc[i]);
  }
#undef PMARK
}

// Frames marked by the byte-counter pass: discard their K2 results (peaks, the hotspot
// count, debug records and K2 flag bits) and list them for the 16-bit pass.  One CTA.
__global__ void k_redo_reset(Params P, int n_frames) {
  __shared__ int n;
  if (threadIdx.x == 0) n = 0;
  __syncthreads();
  for (int f = threadIdx.x; f < n_frames; f += blockDim.x) {
    if (!P.redo[f] && !P.force_redo) continue;
    P.peak_count[f] = 0;
    P.stats[f].hotspots = 0;
    P.dbg_count[f] = 0;
    P.flags[f] &= ~(OVF_HOTSPOTS | OVF_RINGS | OVF_DEBUG);
    if (P.dbg_fpr)
      for (int i = 0; i < 3 * P.n_levels; ++i) P.dbg_fpr[(int64_t)f * 3 * P.n_levels + i] = 0;
    P.redo_list[1 + atomicAdd(&n, 1)] = f;
  }
  __syncthreads();
  if (threadIdx.x == 0) P.redo_list[0] = n;
}

template <bool Wd, int Gv, int NT, int MB, int CB, bool R16>
static cudaError_t launch2_one(int n_frames, const Params& P, int n_sm, cudaStream_t st) {
  const size_t sm = (size_t)P.k2o.total;
  cudaError_t e =
      cudaFuncSetAttribute(k_hough2<Wd, Gv, NT, MB, CB, R16>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  if (e != cudaSuccess) return e;
  int per_sm = 0;
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_hough2<Wd, Gv, NT, MB, CB, R16>, NT, sm);
  if (e != cudaSuccess) return e;
  if (per_sm < 1) return cudaErrorInvalidConfiguration;
  if (P.k2_ctas_per_sm > 0) per_sm = std::min(per_sm, P.k2_ctas_per_sm);   // leave room for concurrent kernels
  const int items = n_frames * P.ntx * P.nty;
  const int grid = std::min(items, per_sm * n_sm);
  k_hough2<Wd, Gv, NT, MB, CB, R16><<<grid, NT, sm, st>>>(P, n_frames);
  return cudaGetLastError();
}

bool k_hough2_has_shape(int cb, int G, int nt, int minb) {
  if (cb == 1)
    return (G == 4 && nt == 384 && minb == 2) || (G == 4 && nt == 512 && minb == 2) ||
           (G == 8 && nt == 384 && minb == 2) || (G == 8 && nt == 512 && minb == 1) ||
           (G == 4 && nt == 256 && minb == 3) || (G == 8 && nt == 256 && minb == 2) ||
           (G == 4 && nt == 512 && minb == 1) || (G == 4 && nt == 768 && minb == 1);
  return (G == 4 && nt == 384 && minb == 2) || (G == 4 && nt == 512 && minb == 2) ||
         (G == 8 && nt == 512 && minb == 1) || (G == 4 && nt == 512 && minb == 1);
}

// one launch of the persistent K2 in shape (G, threads, CTAs/SM) with counter width cb
cudaError_t launch_hough2(int n_frames, const Params& P, bool wide, int G, int nt, int minb, int cb, int n_sm,
                          cudaStream_t st) {
  const int key = (cb << 20) | (G << 12) | (nt << 2) | (minb << 1) | (wide ? 1 : 0);
#define CASE(CBv, Gv, NTv, MBv)                                                                       \
  case (CBv << 20) | (Gv << 12) | (NTv << 2) | (MBv << 1) | 0:                                       \
    return P.k2_rr16 ? launch2_one<false, Gv, NTv, MBv, CBv, true>(n_frames, P, n_sm, st)          \
                     : launch2_one<false, Gv, NTv, MBv, CBv, false>(n_frames, P, n_sm, st);        \
  case (CBv << 20) | (Gv << 12) | (NTv << 2) | (MBv << 1) | 1:                                       \
    return P.k2_rr16 ? launch2_one<true, Gv, NTv, MBv, CBv, true>(n_frames, P, n_sm, st)           \
                     : launch2_one<true, Gv, NTv, MBv, CBv, false>(n_frames, P, n_sm, st);
  switch (key) {
    CASE(1, 4, 384, 2)
    CASE(1, 4, 512, 2)
    CASE(1, 8, 384, 2)
    CASE(1, 8, 512, 1)
    CASE(1, 4, 256, 3)
    CASE(1, 8, 256, 2)
    CASE(1, 4, 512, 1)
    CASE(1, 4, 768, 1)
    CASE(2, 4, 384, 2)
    CASE(2, 4, 512, 2)
    CASE(2, 8, 512, 1)
    CASE(2, 4, 512, 1)
    default: return cudaErrorInvalidValue;
  }
#undef CASE
}

cudaError_t launch_redo_reset(int n_frames, const Params& P, cudaStream_t st) {
  k_redo_reset<<<1, 256, 0, st>>>(P, n_frames);
  return cudaGetLastError();
}

}  // namespace rd
