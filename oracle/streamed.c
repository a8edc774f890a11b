/* streamed.c — the paper's own streamed voting and peak search (SI "Detailed algorithm",
 * steps 2-4), a second CPU oracle for the Hough stage.
 *
 * TEST INFRASTRUCTURE ONLY (see oracle.h).  The paper states that its optimisations change
 * memory and speed, not values: votes are collected per ridge pixel
 * (SI step 2), the vote stack is fully sorted by a bijective integer
 * code (SI step 3), and the parameter space is populated level by level
 * in two 3-level sub-spaces (raw and smoothed/normalised) indexed by r mod 3, with
 * registration of modified elements and undo of the bottom level (SI step 4,
 * PAPER.md:941-978).  Here it is written in that order and notation; tests check that it
 * yields exactly the hotspots and peaks of the full-array oracle (orc_peaks), which pins
 * the "streamed == full array" claim.  Readings R8-R14 apply.
 */
#include <math.h>
#include <stdlib.h>
#include <string.h>

#include "oracle.h"

static int cmp_u32(const void* a, const void* b) {
  uint32_t x = *(const uint32_t*)a, y = *(const uint32_t*)b;
  return x < y ? -1 : (x > y ? 1 : 0);
}

/* S at cell c of the raw level `lvl` (radius r): the radius-dependent Gaussian window sum
 * (reading R11) */
static int64_t window(const orc_params* p, const int32_t* lvl, int32_t r, int64_t c) {
  const int W = p->width, H = p->height;
  const int y = (int)(c / W), x = (int)(c % W);
  const int K = orc_level_halfwidth(p, r);
  int64_t wt[256];
  for (int d = 0; d <= K && d < 256; ++d) wt[d] = orc_level_weight(p, r, d);
  int64_t S = 0;
  for (int i = -K; i <= K; ++i) {
    if (y + i < 0 || y + i >= H) continue;
    for (int j = -K; j <= K; ++j) {
      if (x + j < 0 || x + j >= W) continue;
      S += wt[i < 0 ? -i : i] * wt[j < 0 ? -j : j] * (int64_t)lvl[(size_t)(y + i) * W + (x + j)];
    }
  }
  return S;
}

typedef struct { int64_t* v; int64_t n, cap; } vec64;
static int push(vec64* a, int64_t x) {
  if (a->n == a->cap) {
    a->cap = a->cap ? 2 * a->cap : 1024;
    a->v = (int64_t*)realloc(a->v, sizeof(int64_t) * (size_t)a->cap);
    if (!a->v) return -1;
  }
  a->v[a->n++] = x;
  return 0;
}

int64_t orc_stream_peaks(const orc_params* p, const orc_ridge* ridges, int64_t n_ridges, orc_hotspot* peaks,
                         int64_t peak_cap, orc_hotspot* hot_out, int64_t hot_cap, int64_t* n_hot) {
  const int W = p->width, H = p->height;
  const int r_lo = p->r_min - 1, r_hi = p->r_max + 1;
  const int64_t HW = (int64_t)W * H;
  /* SI step 2: votes collected per ridge pixel, each as one integer code (bijection of
   * (r, row, col), SI step 3) */
  vec64 stack = {0, 0, 0};
  for (int64_t k = 0; k < n_ridges; ++k)
    for (int r = r_lo; r <= r_hi; ++r) {
      long long ox = llround((double)r * ridges[k].dx), oy = llround((double)r * ridges[k].dy);
      for (int s = 1; s >= -1; s -= 2) {
        long long tx = ridges[k].x + s * ox, ty = ridges[k].y + s * oy;
        if (tx < 0 || tx >= W || ty < 0 || ty >= H) continue;
        if (push(&stack, ((int64_t)(r - r_lo) * H + ty) * W + tx)) return -1;
      }
    }
  /* SI step 3: full sort of the vote stack (radius, then row, then column) */
  uint32_t* codes = (uint32_t*)malloc(sizeof(uint32_t) * (size_t)(stack.n ? stack.n : 1));
  if (!codes) return -1;
  for (int64_t i = 0; i < stack.n; ++i) codes[i] = (uint32_t)stack.v[i];
  free(stack.v);
  qsort(codes, (size_t)stack.n, sizeof(uint32_t), cmp_u32);

  /* SI step 4: two sub-spaces of three consecutive levels, addressed by r mod 3 */
  int32_t* raw = (int32_t*)calloc((size_t)(3 * HW), sizeof(int32_t));
  int64_t* nrm = (int64_t*)calloc((size_t)(3 * HW), sizeof(int64_t));
  vec64 mod[3] = {{0, 0, 0}, {0, 0, 0}, {0, 0, 0}}, hot[3] = {{0, 0, 0}, {0, 0, 0}, {0, 0, 0}};
  if (!raw || !nrm) { free(codes); free(raw); free(nrm); return -1; }
  int64_t i = 0, npk = 0, nh = 0;
  for (int r = r_lo; r <= r_hi; ++r) {
    const int sl = (r - r_lo) % 3;
    int32_t* lvl = raw + sl * HW;
    /* populate level r: votes of one voxel come out of the sorted stack in a row */
    int64_t prev = -1;
    while (i < stack.n && (int64_t)codes[i] / HW == r - r_lo) {
      const int64_t c = (int64_t)codes[i] % HW;
      if (c != prev) {
        if (push(&mod[sl], c)) return -1;                          /* registered as modified */
        if (prev >= 0 && lvl[prev] > p->vote_threshold_raw && push(&hot[sl], prev)) return -1;  /* "surpassed" */
        prev = c;
      }
      lvl[c] += 1;
      ++i;
    }
    if (prev >= 0 && lvl[prev] > p->vote_threshold_raw && push(&hot[sl], prev)) return -1;
    /* map the hotspots of level r to the smoothed, normalised sub-space */
    for (int64_t k = 0; k < hot[sl].n; ++k) {
      const int64_t c = hot[sl].v[k];
      nrm[sl * HW + c] = window(p, lvl, r, c);
      if (hot_out && nh < hot_cap) {
        hot_out[nh].r = r;
        hot_out[nh].y = (int32_t)(c / W);
        hot_out[nh].x = (int32_t)(c % W);
        hot_out[nh].raw = lvl[c];
        hot_out[nh].S = nrm[sl * HW + c];
      }
      ++nh;
    }
    /* local maxima among the hotspots of level r-1 passing the float threshold (3x3x3) */
    const int rc = r - 1;
    if (rc >= p->r_min && rc <= p->r_max) {
      const int sc = (rc - r_lo) % 3;
      for (int64_t k = 0; k < hot[sc].n; ++k) {
        const int64_t c = hot[sc].v[k];
        const int64_t S = nrm[sc * HW + c];
        if (!((double)S > orc_norm_threshold(p, rc))) continue;
        const int y = (int)(c / W), x = (int)(c % W);
        int win = 1;
        for (int dr = -1; dr <= 1 && win; ++dr)
          for (int dy = -1; dy <= 1 && win; ++dy)
            for (int dx = -1; dx <= 1 && win; ++dx) {
              if (!dr && !dy && !dx) continue;
              if (y + dy < 0 || y + dy >= H || x + dx < 0 || x + dx >= W) continue;
              const int ru = rc + dr, su = (ru - r_lo) % 3;
              const int64_t Su = nrm[su * HW + (int64_t)(y + dy) * W + (x + dx)];
              const __int128 lhs = (__int128)S * ru, rhs = (__int128)Su * rc;
              const int v_first = dr > 0 || (dr == 0 && (dy > 0 || (dy == 0 && dx > 0)));
              if (!(lhs > rhs || (lhs == rhs && v_first))) win = 0;
            }
        if (!win) continue;
        if (npk < peak_cap) {
          peaks[npk].r = rc;
          peaks[npk].y = y;
          peaks[npk].x = x;
          peaks[npk].raw = raw[sc * HW + c];
          peaks[npk].S = S;
        }
        ++npk;
      }
    }
    /* undo every modification of level r-2: it becomes level r+1 (cyclic permutation) */
    if (r - 2 >= r_lo) {
      const int su = (r - 2 - r_lo) % 3;
      for (int64_t k = 0; k < mod[su].n; ++k) {
        raw[su * HW + mod[su].v[k]] = 0;
        nrm[su * HW + mod[su].v[k]] = 0;
      }
      mod[su].n = 0;
      hot[su].n = 0;
    }
  }
  for (int k = 0; k < 3; ++k) { free(mod[k].v); free(hot[k].v); }
  free(codes);
  free(raw);
  free(nrm);
  if (n_hot) *n_hot = nh;
  return npk;
}
