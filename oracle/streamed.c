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
    int64_t* nv = (int64_t*)realloc(a->v, sizeof(int64_t) * (size_t)(a->cap ? 2 * a->cap : 1024));
    if (!nv) return -1;
    a->v = nv;
    a->cap = a->cap ? 2 * a->cap : 1024;
  }
  a->v[a->n++] = x;
  return 0;
}

/* Per-thread state kept across frames, as in the paper's workers: the two 3-level
 * sub-spaces (all zero between frames, restored by the undo), the vote stack and the
 * registries. */
struct orc_stream_ws {
  int64_t HW;
  int32_t* raw;   /* [3][H*W] raw votes, level r at slot (r - r_lo) mod 3 */
  int64_t* nrm;   /* [3][H*W] S of hotspots (0 elsewhere) */
  uint32_t *codes, *tmp;
  int64_t code_cap;
  vec64 mod[3], hot[3];
  int64_t votes;  /* votes of the last frame */
};

orc_stream_ws* orc_stream_ws_create(const orc_params* p) {
  orc_stream_ws* w = (orc_stream_ws*)calloc(1, sizeof(orc_stream_ws));
  if (!w) return NULL;
  w->HW = (int64_t)p->width * p->height;
  w->raw = (int32_t*)calloc((size_t)(3 * w->HW), sizeof(int32_t));
  w->nrm = (int64_t*)calloc((size_t)(3 * w->HW), sizeof(int64_t));
  if (!w->raw || !w->nrm) { orc_stream_ws_free(w); return NULL; }
  return w;
}

void orc_stream_ws_free(orc_stream_ws* w) {
  if (!w) return;
  free(w->raw);
  free(w->nrm);
  free(w->codes);
  free(w->tmp);
  for (int k = 0; k < 3; ++k) { free(w->mod[k].v); free(w->hot[k].v); }
  free(w);
}

/* undo every registered modification of one slot */
static void undo(orc_stream_ws* w, int sl) {
  for (int64_t k = 0; k < w->mod[sl].n; ++k) {
    w->raw[sl * w->HW + w->mod[sl].v[k]] = 0;
    w->nrm[sl * w->HW + w->mod[sl].v[k]] = 0;
  }
  w->mod[sl].n = 0;
  w->hot[sl].n = 0;
}

int64_t orc_stream_peaks_ws(const orc_params* p, orc_stream_ws* w, const orc_ridge* ridges, int64_t n_ridges,
                            orc_hotspot* peaks, int64_t peak_cap, orc_hotspot* hot_out, int64_t hot_cap,
                            int64_t* n_hot) {
  const int W = p->width, H = p->height;
  const int r_lo = p->r_min - 1, r_hi = p->r_max + 1;
  const int64_t HW = w->HW;
  /* SI step 2: votes collected per ridge pixel, each pushed as one integer code, the
   * bijection ((r - r_lo) * H + row) * W + col of SI step 3 */
  const int64_t max_votes = n_ridges * 2 * (r_hi - r_lo + 1);
  if (max_votes > w->code_cap) {
    free(w->codes);
    free(w->tmp);
    w->code_cap = max_votes > 1024 ? max_votes : 1024;
    w->codes = (uint32_t*)malloc(sizeof(uint32_t) * (size_t)w->code_cap);
    w->tmp = (uint32_t*)malloc(sizeof(uint32_t) * (size_t)w->code_cap);
    if (!w->codes || !w->tmp) { w->code_cap = 0; return -1; }
  }
  int64_t n = 0;
  for (int64_t k = 0; k < n_ridges; ++k)
    for (int r = r_lo; r <= r_hi; ++r) {
      long long ox = llround((double)r * ridges[k].dx), oy = llround((double)r * ridges[k].dy);
      for (int s = 1; s >= -1; s -= 2) {
        long long tx = ridges[k].x + s * ox, ty = ridges[k].y + s * oy;
        if (tx < 0 || tx >= W || ty < 0 || ty >= H) continue;
        w->codes[n++] = (uint32_t)(((int64_t)(r - r_lo) * H + ty) * W + tx);
      }
    }
  w->votes = n;
  /* SI step 3: full sort of the vote stack (radius, then row, then column); a plain
   * least-significant-digit radix sort, 4 passes of 8 bits */
  uint32_t *a = w->codes, *b = w->tmp;
  for (int sh = 0; sh < 32; sh += 8) {
    int64_t cnt[257] = {0};
    for (int64_t i = 0; i < n; ++i) ++cnt[((a[i] >> sh) & 255) + 1];
    for (int d = 0; d < 256; ++d) cnt[d + 1] += cnt[d];
    for (int64_t i = 0; i < n; ++i) b[cnt[(a[i] >> sh) & 255]++] = a[i];
    uint32_t* t = a; a = b; b = t;
  }
  const uint32_t* codes = a;   /* after an even number of passes: w->codes */

  /* SI step 4: two sub-spaces of three consecutive levels, addressed by r mod 3 */
  int64_t i = 0, npk = 0, nh = 0;
  for (int r = r_lo; r <= r_hi; ++r) {
    const int sl = (r - r_lo) % 3;
    int32_t* lvl = w->raw + sl * HW;
    vec64 *mod = &w->mod[sl], *hot = &w->hot[sl];
    /* populate level r: the votes of one voxel come out of the sorted stack in a row */
    int64_t prev = -1;
    while (i < n && (int64_t)codes[i] / HW == r - r_lo) {
      const int64_t c = (int64_t)codes[i] % HW;
      if (c != prev) {
        if (push(mod, c)) return -1;                                                   /* "modified" */
        if (prev >= 0 && lvl[prev] > p->vote_threshold_raw && push(hot, prev)) return -1; /* "surpassed" */
        prev = c;
      }
      lvl[c] += 1;
      ++i;
    }
    if (prev >= 0 && lvl[prev] > p->vote_threshold_raw && push(hot, prev)) return -1;
    /* map the hotspots of level r to the smoothed, normalised sub-space */
    for (int64_t k = 0; k < hot->n; ++k) {
      const int64_t c = hot->v[k];
      w->nrm[sl * HW + c] = window(p, lvl, r, c);
      if (hot_out && nh < hot_cap) {
        hot_out[nh].r = r;
        hot_out[nh].y = (int32_t)(c / W);
        hot_out[nh].x = (int32_t)(c % W);
        hot_out[nh].raw = lvl[c];
        hot_out[nh].S = w->nrm[sl * HW + c];
      }
      ++nh;
    }
    /* local maxima among the hotspots of level r-1 passing the float threshold (3x3x3;
     * exact cross-multiplied comparison of S/r, lexicographic ties: readings R13-R14) */
    const int rc = r - 1;
    if (rc >= p->r_min && rc <= p->r_max) {
      const int sc = (rc - r_lo) % 3;
      const double Tn = orc_norm_threshold(p, rc);
      for (int64_t k = 0; k < w->hot[sc].n; ++k) {
        const int64_t c = w->hot[sc].v[k];
        const int64_t S = w->nrm[sc * HW + c];
        if (!((double)S > Tn)) continue;
        const int y = (int)(c / W), x = (int)(c % W);
        int win = 1;
        for (int dr = -1; dr <= 1 && win; ++dr)
          for (int dy = -1; dy <= 1 && win; ++dy)
            for (int dx = -1; dx <= 1 && win; ++dx) {
              if (!dr && !dy && !dx) continue;
              if (y + dy < 0 || y + dy >= H || x + dx < 0 || x + dx >= W) continue;
              const int ru = rc + dr, su = (ru - r_lo) % 3;
              const int64_t Su = w->nrm[su * HW + (int64_t)(y + dy) * W + (x + dx)];
              const __int128 lhs = (__int128)S * ru, rhs = (__int128)Su * rc;
              const int v_first = dr > 0 || (dr == 0 && (dy > 0 || (dy == 0 && dx > 0)));
              if (!(lhs > rhs || (lhs == rhs && v_first))) win = 0;
            }
        if (!win) continue;
        if (npk < peak_cap) {
          peaks[npk].r = rc;
          peaks[npk].y = y;
          peaks[npk].x = x;
          peaks[npk].raw = w->raw[sc * HW + c];
          peaks[npk].S = S;
        }
        ++npk;
      }
    }
    /* undo every modification of level r-2: its slot becomes level r+1 */
    if (r - 2 >= r_lo) undo(w, (r - 2 - r_lo) % 3);
  }
  /* leave the sub-spaces zero for the next frame */
  for (int k = 0; k < 3; ++k) undo(w, k);
  if (n_hot) *n_hot = nh;
  return npk;
}

int64_t orc_stream_peaks(const orc_params* p, const orc_ridge* ridges, int64_t n_ridges, orc_hotspot* peaks,
                         int64_t peak_cap, orc_hotspot* hot_out, int64_t hot_cap, int64_t* n_hot) {
  orc_stream_ws* w = orc_stream_ws_create(p);
  if (!w) return -1;
  int64_t n = orc_stream_peaks_ws(p, w, ridges, n_ridges, peaks, peak_cap, hot_out, hot_cap, n_hot);
  orc_stream_ws_free(w);
  return n;
}

int64_t orc_stream_votes(const orc_stream_ws* w) { return w->votes; }
