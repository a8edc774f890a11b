/* synth.c — seeded synthetic ring frames (input module shared by tests, oracle
 * and bench; holds none of the detection method's arithmetic).
 *
 * Recipe (BASELINE.json configs):
 *   value(x,y) = background + sum_i amp_i * exp(-(d_i - r_i)^2 / (2 sigma_p^2)) * mask_i
 *   d_i = |(x,y) - c_i|, mask_i = 0 on a removed polar arc (occlusion), else 1;
 *   noise: Poisson shot noise (normal approximation N(lambda, lambda); lambda >= 100
 *   everywhere for the u16 configs) plus Gaussian read noise, drawn as one normal
 *   with variance lambda + read^2; round half up, clip to [0, max_value].
 */
#define _GNU_SOURCE
#include "synth.h"

#include <math.h>
#include <pthread.h>
#include <stdlib.h>
#include <string.h>
#include <unistd.h>

#ifndef M_PI
#define M_PI 3.14159265358979323846
#endif

/* ---------------------------------------------------------------- RNG */
static inline uint64_t mix64(uint64_t z) {
  z += 0x9E3779B97F4A7C15ULL;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}
uint64_t synth_key(uint64_t a, uint64_t b, uint64_t c) {
  return mix64(mix64(mix64(a) ^ b) ^ c);
}
static inline uint64_t rbits(uint64_t key, uint64_t ctr) { return mix64(key ^ mix64(ctr)); }
double synth_u01(uint64_t key, uint64_t ctr) { return (double)(rbits(key, ctr) >> 11) * 0x1.0p-53; }

typedef struct { uint64_t key, ctr; } stream_t;
static inline double su01(stream_t* s) { return synth_u01(s->key, s->ctr++); }
static inline double suni(stream_t* s, double a, double b) { return a + (b - a) * su01(s); }
static inline int sint(stream_t* s, int n) { /* uniform in [0, n) */
  int v = (int)(su01(s) * n);
  return v >= n ? n - 1 : v;
}
static inline double normal_at(uint64_t key, uint64_t idx) {
  double u1 = synth_u01(key, 2 * idx), u2 = synth_u01(key, 2 * idx + 1);
  return sqrt(-2.0 * log(1.0 - u1)) * cos(2.0 * M_PI * u2);
}

/* ---------------------------------------------------------------- configs */
int synth_config_shape(int cfg, int32_t* w, int32_t* h, int32_t* pb, int32_t* mv, int32_t* batch) {
  int32_t W, H, PB, MV, B;
  switch (cfg) {
    case 1: case 11: W = 128; H = 128; PB = 1; MV = 255; B = 1; break;
    case 2: W = 640; H = 480; PB = 1; MV = 255; B = 16; break;
    case 3: W = 1024; H = 688; PB = 2; MV = 4095; B = 256; break;
    case 4: W = 1024; H = 1024; PB = 2; MV = 4095; B = 512; break;
    case 5: W = 1024; H = 688; PB = 2; MV = 4095; B = 8192; break;
    default: return -1;
  }
  if (w) *w = W;
  if (h) *h = H;
  if (pb) *pb = PB;
  if (mv) *mv = MV;
  if (batch) *batch = B;
  return 0;
}

int synth_config_scene(int cfg, synth_scene* s) {
  if (synth_config_shape(cfg, &s->width, &s->height, &s->pixel_bytes, &s->max_value, NULL)) return -1;
  switch (cfg) {
    case 1: s->background = 20; s->sigma_p = 1.0; s->read_sigma = 5; s->poisson = 0; break;
    case 11: s->background = 20; s->sigma_p = 1.0; s->read_sigma = 0; s->poisson = 0; break;
    case 2: s->background = 15; s->sigma_p = 1.2; s->read_sigma = 6; s->poisson = 0; break;
    case 3: case 5: s->background = 100; s->sigma_p = 1.5; s->read_sigma = 8; s->poisson = 1; break;
    case 4: s->background = 100; s->sigma_p = 1.5; s->read_sigma = 10; s->poisson = 1; break;
    default: return -1;
  }
  return 0;
}

/* annuli of two rings intersect: |ri - rj| < d < ri + rj */
static int intersects(const synth_ring* a, const synth_ring* b) {
  double d = hypot(a->cx - b->cx, a->cy - b->cy);
  return d > fabs(a->r - b->r) && d < a->r + b->r;
}
/* well separated: no intersection, no nesting, a gap of `gap` px */
static int separated(const synth_ring* a, const synth_ring* b, double gap) {
  return hypot(a->cx - b->cx, a->cy - b->cy) >= a->r + b->r + gap;
}
static void place_uniform(stream_t* s, const synth_scene* sc, double r, double margin_extra, int integer,
                          synth_ring* out) {
  double m = r + margin_extra;
  double lox = m, hix = sc->width - 1 - m, loy = m, hiy = sc->height - 1 - m;
  if (hix < lox) hix = lox = 0.5 * (sc->width - 1);
  if (hiy < loy) hiy = loy = 0.5 * (sc->height - 1);
  if (integer) {
    int ilx = (int)ceil(lox), ihx = (int)floor(hix), ily = (int)ceil(loy), ihy = (int)floor(hiy);
    out->cx = ilx + sint(s, ihx - ilx + 1);
    out->cy = ily + sint(s, ihy - ily + 1);
  } else {
    out->cx = suni(s, lox, hix);
    out->cy = suni(s, loy, hiy);
  }
}
static int in_bounds(const synth_scene* sc, const synth_ring* g, double margin_extra) {
  double m = g->r + margin_extra;
  return g->cx >= m && g->cx <= sc->width - 1 - m && g->cy >= m && g->cy <= sc->height - 1 - m;
}
static void init_ring(synth_ring* g) { memset(g, 0, sizeof *g); g->group = -1; }

/* cfg1 / cfg11: 3 well-separated rings of radii 10, 15, 20 */
static int layout_cfg1(stream_t* s, const synth_scene* sc, int integer, synth_ring* out) {
  static const double radii[3] = {10, 15, 20};
  for (int attempt = 0; attempt < 100000; ++attempt) {
    int ok = 1;
    for (int i = 0; i < 3 && ok; ++i) {
      init_ring(&out[i]);
      out[i].r = radii[i];
      out[i].amp = 180;
      if (integer) place_uniform(s, sc, radii[i], 5, 1, &out[i]);
      else { out[i].cx = suni(s, 20, 108); out[i].cy = suni(s, 20, 108); }
      for (int j = 0; j < i; ++j)
        if (!separated(&out[i], &out[j], 3 * sc->sigma_p)) ok = 0;
    }
    if (ok) return 3;
  }
  return 3;
}

static int try_single(stream_t* s, const synth_scene* sc, synth_ring* rings, int n, double r, double amp,
                      int tries, synth_ring* g) {
  double margin = 3 * sc->sigma_p + 3;
  for (int t = 0; t < tries; ++t) {
    init_ring(g);
    g->r = r;
    g->amp = amp;
    place_uniform(s, sc, r, margin, 0, g);
    int ok = 1;
    for (int j = 0; j < n && ok; ++j)
      if (!separated(g, &rings[j], 3 * sc->sigma_p)) ok = 0;
    if (ok) return 1;
  }
  return 0;
}

/* a partner that intersects ring `a` and is separated from all the others */
static int try_partner(stream_t* s, const synth_scene* sc, synth_ring* rings, int n, const synth_ring* a, double r,
                       double amp, int tries, synth_ring* g) {
  double margin = 3 * sc->sigma_p + 3, sp = sc->sigma_p;
  for (int t = 0; t < tries; ++t) {
    double lo = fabs(a->r - r) + 2 * sp, hi = a->r + r - 2 * sp;
    if (hi <= lo) return 0;
    double d = suni(s, lo, hi), th = suni(s, 0, 2 * M_PI);
    init_ring(g);
    g->r = r;
    g->amp = amp;
    g->cx = a->cx + d * cos(th);
    g->cy = a->cy + d * sin(th);
    if (!in_bounds(sc, g, margin)) continue;
    int ok = 1;
    for (int j = 0; j < n && ok; ++j)
      if (&rings[j] != a && !separated(g, &rings[j], 3 * sp)) ok = 0;
    if (ok) return 1;
  }
  return 0;
}

static void occlude(stream_t* s, synth_ring* rings, int n, int n_occ) {
  /* choose n_occ distinct rings (partial Fisher-Yates over indices) */
  int idx[4096];
  if (n > 4096) n = 4096;
  for (int i = 0; i < n; ++i) idx[i] = i;
  for (int k = 0; k < n_occ && k < n; ++k) {
    int j = k + sint(s, n - k);
    int t = idx[k]; idx[k] = idx[j]; idx[j] = t;
    synth_ring* g = &rings[idx[k]];
    g->occ_len = suni(s, M_PI / 3, M_PI);          /* 60..180 degrees */
    g->occ_start = suni(s, 0, 2 * M_PI);
  }
}

/* cfg2: 20 rings, radii U[8,40], 20% placed overlapping a neighbour */
static int layout_cfg2(stream_t* s, const synth_scene* sc, synth_ring* rings, int cap) {
  const int N = 20, n_ov = 4;
  int n = 0, group = 0;
  if (cap < N) return -1;
  while (n < N - n_ov) {
    synth_ring g;
    double r = suni(s, 8, 40), amp = suni(s, 120, 240) - sc->background;
    if (!try_single(s, sc, rings, n, r, amp, 200, &g)) { /* relax: accept overlap */
      init_ring(&g); g.r = r; g.amp = amp; place_uniform(s, sc, r, 3 * sc->sigma_p + 3, 0, &g);
    }
    rings[n++] = g;
  }
  for (int k = 0; k < n_ov; ++k) {
    synth_ring g;
    int placed = 0;
    for (int t = 0; t < 200 && !placed; ++t) {
      int a = sint(s, N - n_ov);
      double r = suni(s, 8, 40), amp = suni(s, 120, 240) - sc->background;
      if (try_partner(s, sc, rings, n, &rings[a], r, amp, 20, &g)) {
        placed = 1;
        if (rings[a].group < 0) rings[a].group = group++;
        rings[a].kind = 1;
        g.group = rings[a].group;
        g.kind = 1;
      }
    }
    if (!placed) {
      init_ring(&g); g.r = suni(s, 8, 40); g.amp = suni(s, 120, 240) - sc->background;
      place_uniform(s, sc, g.r, 3 * sc->sigma_p + 3, 0, &g);
    }
    rings[n++] = g;
  }
  return n;
}

/* cfg3/5: 50 rings, radii U[10,60]: 8 overlapping pairs, 3 nested concentric
 * pairs (dr ~ U[6,20]), 28 well-separated singles; 5 rings occluded by an arc */
static int layout_cfg3(stream_t* s, const synth_scene* sc, synth_ring* rings, int cap) {
  const int N = 50, n_nest = 3, n_ov = 8;
  int n = 0, group = 0;
  double margin = 3 * sc->sigma_p + 3;
  if (cap < N) return -1;
  for (int k = 0; k < n_nest; ++k) {
    double ro = suni(s, 16, 60);
    double dmax = fmin(20, ro - 10);
    double dr = suni(s, 6, dmax);
    synth_ring g;
    if (!try_single(s, sc, rings, n, ro, suni(s, 800, 3000) - sc->background, 500, &g)) {
      init_ring(&g); g.r = ro; g.amp = suni(s, 800, 3000) - sc->background; place_uniform(s, sc, ro, margin, 0, &g);
    }
    g.group = group; g.kind = 2;
    rings[n++] = g;
    synth_ring in = g;
    in.r = ro - dr;
    in.amp = suni(s, 800, 3000) - sc->background;
    rings[n++] = in;
    group++;
  }
  for (int k = 0; k < n_ov; ++k) {
    int done = 0;
    for (int t = 0; t < 100 && !done; ++t) {
      synth_ring a, b;
      double ra = suni(s, 10, 60), rb = suni(s, 10, 60);
      if (!try_single(s, sc, rings, n, ra, suni(s, 800, 3000) - sc->background, 50, &a)) continue;
      if (!try_partner(s, sc, rings, n, &a, rb, suni(s, 800, 3000) - sc->background, 50, &b)) continue;
      a.group = b.group = group++;
      a.kind = b.kind = 1;
      rings[n++] = a;
      rings[n++] = b;
      done = 1;
    }
    if (!done) { /* relax */
      synth_ring a; init_ring(&a); a.r = suni(s, 10, 60); a.amp = suni(s, 800, 3000) - sc->background;
      place_uniform(s, sc, a.r, margin, 0, &a); rings[n++] = a;
      synth_ring b; init_ring(&b); b.r = suni(s, 10, 60); b.amp = suni(s, 800, 3000) - sc->background;
      place_uniform(s, sc, b.r, margin, 0, &b); rings[n++] = b;
    }
  }
  while (n < N) {
    synth_ring g;
    double r = suni(s, 10, 60), amp = suni(s, 800, 3000) - sc->background;
    if (!try_single(s, sc, rings, n, r, amp, 500, &g)) {
      init_ring(&g); g.r = r; g.amp = amp; place_uniform(s, sc, r, margin, 0, &g);
    }
    rings[n++] = g;
  }
  occlude(s, rings, n, 5);
  return n;
}

/* cfg4: 200 rings, radii U[10,80]; sequential placement steering the mean number
 * of annulus-intersecting neighbours per ring towards 3 */
static int layout_cfg4(stream_t* s, const synth_scene* sc, synth_ring* rings, int cap) {
  const int N = 200;
  const double target_mean = 3.0;
  double margin = 3 * sc->sigma_p + 3;
  long edges = 0;
  if (cap < N) return -1;
  for (int k = 0; k < N; ++k) {
    double want = 0.5 * target_mean * (k + 1) - (double)edges;
    synth_ring best;
    int best_o = -1;
    double best_err = 1e300;
    for (int c = 0; c < 16; ++c) {
      synth_ring g;
      init_ring(&g);
      g.r = suni(s, 10, 80);
      g.amp = suni(s, 800, 3000) - sc->background;
      g.kind = 3;
      place_uniform(s, sc, g.r, margin, 0, &g);
      int o = 0;
      for (int j = 0; j < k; ++j) o += intersects(&g, &rings[j]);
      double err = fabs((double)o - want);
      if (err < best_err) { best_err = err; best = g; best_o = o; }
    }
    rings[k] = best;
    edges += best_o;
  }
  return N;
}

int synth_layout(int cfg, uint64_t seed, int64_t frame_idx, synth_ring* rings, int32_t cap) {
  synth_scene sc;
  if (synth_config_scene(cfg, &sc)) return -1;
  int key_cfg = (cfg == 5) ? 3 : cfg;    /* cfg5 frame i == cfg3 frame i */
  stream_t s = {synth_key((uint64_t)key_cfg, seed, (uint64_t)frame_idx), 0};
  switch (cfg) {
    case 1: return cap >= 3 ? layout_cfg1(&s, &sc, 0, rings) : -1;
    case 11: return cap >= 3 ? layout_cfg1(&s, &sc, 1, rings) : -1;
    case 2: return layout_cfg2(&s, &sc, rings, cap);
    case 3: case 5: return layout_cfg3(&s, &sc, rings, cap);
    case 4: return layout_cfg4(&s, &sc, rings, cap);
  }
  return -1;
}

/* ---------------------------------------------------------------- render */
int synth_render(const synth_scene* sc, const synth_ring* rings, int32_t n_rings, uint64_t noise_key, void* out,
                 int64_t pitch) {
  const int W = sc->width, H = sc->height;
  double* img = (double*)malloc(sizeof(double) * (size_t)W * H);
  if (!img) return -1;
  for (size_t i = 0; i < (size_t)W * H; ++i) img[i] = sc->background;
  const double sp = sc->sigma_p, reach = 5 * sp, inv2s2 = 1.0 / (2 * sp * sp);
  for (int k = 0; k < n_rings; ++k) {
    const synth_ring* g = &rings[k];
    int x0 = (int)floor(g->cx - g->r - reach), x1 = (int)ceil(g->cx + g->r + reach);
    int y0 = (int)floor(g->cy - g->r - reach), y1 = (int)ceil(g->cy + g->r + reach);
    if (x0 < 0) x0 = 0;
    if (y0 < 0) y0 = 0;
    if (x1 > W - 1) x1 = W - 1;
    if (y1 > H - 1) y1 = H - 1;
    for (int y = y0; y <= y1; ++y)
      for (int x = x0; x <= x1; ++x) {
        double ddx = x - g->cx, ddy = y - g->cy;
        double d = sqrt(ddx * ddx + ddy * ddy), t = d - g->r;
        if (fabs(t) > reach) continue;
        if (g->occ_len > 0) {
          double th = atan2(ddy, ddx);
          double rel = fmod(th - g->occ_start + 4 * M_PI, 2 * M_PI);
          if (rel < g->occ_len) continue;
        }
        img[(size_t)y * W + x] += g->amp * exp(-t * t * inv2s2);
      }
  }
  const double rs2 = sc->read_sigma * sc->read_sigma;
  for (int y = 0; y < H; ++y) {
    for (int x = 0; x < W; ++x) {
      size_t i = (size_t)y * W + x;
      double lam = img[i], var = rs2 + (sc->poisson ? (lam > 0 ? lam : 0) : 0);
      double v = lam;
      if (var > 0) v += sqrt(var) * normal_at(noise_key, i);
      double q = floor(v + 0.5);
      if (q < 0) q = 0;
      if (q > sc->max_value) q = sc->max_value;
      if (sc->pixel_bytes == 1) ((uint8_t*)out + y * pitch)[x] = (uint8_t)q;
      else ((uint16_t*)((uint8_t*)out + y * pitch))[x] = (uint16_t)q;
    }
  }
  free(img);
  return 0;
}

int synth_frame(int cfg, uint64_t seed, int64_t frame_idx, void* out, synth_ring* truth, int32_t truth_cap,
                int32_t* n_truth) {
  synth_scene sc;
  if (synth_config_scene(cfg, &sc)) return -1;
  synth_ring rings[512];
  int n = synth_layout(cfg, seed, frame_idx, rings, 512);
  if (n < 0) return -1;
  int key_cfg = (cfg == 5) ? 3 : cfg;
  uint64_t nk = synth_key((uint64_t)key_cfg + 1000, seed, (uint64_t)frame_idx);
  if (synth_render(&sc, rings, n, nk, out, (int64_t)sc.width * sc.pixel_bytes)) return -1;
  if (truth) {
    int m = n < truth_cap ? n : truth_cap;
    memcpy(truth, rings, sizeof(synth_ring) * (size_t)m);
  }
  if (n_truth) *n_truth = n;
  return 0;
}

typedef struct {
  int cfg;
  uint64_t seed;
  int64_t first;
  int32_t n;
  uint8_t* out;
  size_t stride;
  int next;
  pthread_mutex_t mu;
  int err;
} batch_job;

static void* batch_worker(void* arg) {
  batch_job* j = (batch_job*)arg;
  for (;;) {
    pthread_mutex_lock(&j->mu);
    int i = j->next++;
    pthread_mutex_unlock(&j->mu);
    if (i >= j->n) break;
    if (synth_frame(j->cfg, j->seed, j->first + i, j->out + (size_t)i * j->stride, NULL, 0, NULL)) j->err = 1;
  }
  return NULL;
}

int synth_batch(int cfg, uint64_t seed, int64_t first, int32_t n, void* out, int32_t nthreads) {
  int32_t W, H, PB;
  if (synth_config_shape(cfg, &W, &H, &PB, NULL, NULL)) return -1;
  if (nthreads <= 0) nthreads = (int32_t)sysconf(_SC_NPROCESSORS_ONLN);
  if (nthreads > n) nthreads = n > 0 ? n : 1;
  if (nthreads > 256) nthreads = 256;
  batch_job j = {cfg, seed, first, n, (uint8_t*)out, (size_t)W * H * PB, 0, PTHREAD_MUTEX_INITIALIZER, 0};
  pthread_t th[256];
  for (int t = 0; t < nthreads; ++t) pthread_create(&th[t], NULL, batch_worker, &j);
  for (int t = 0; t < nthreads; ++t) pthread_join(th[t], NULL);
  return j.err ? -1 : 0;
}
