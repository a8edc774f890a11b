/* oracle.c — plain CPU oracle of the ridge-directed circle-Hough ring detector.
 *
 * TEST INFRASTRUCTURE ONLY (see oracle.h): callable from tests/, smoke() and
 * bench.py's CPU-baseline legs; never from the product path.  Shares no code with
 * paper_1310_1371_b200/.
 *
 * Paper: /root/reference/PAPER.md (arXiv 1310.1371).  Step numbers follow
 * SURVEY.md §8(c); every reading where the paper is silent is listed in DESIGN.md
 * "Readings" (R1..R18).  Compile with -ffp-contract=off (no FMA contraction) so the
 * floating-point recipe of step 3 is the one written here.
 */
#define _GNU_SOURCE
#include "oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdlib.h>
#include <string.h>
#include <unistd.h>

#ifndef M_PI
#define M_PI 3.14159265358979323846
#endif

static inline int clampi(int v, int lo, int hi) { return v < lo ? lo : (v > hi ? hi : v); }

static inline int64_t pixel_at(const orc_params* p, const void* frame, int64_t pitch, int x, int y) {
  const uint8_t* row = (const uint8_t*)frame + (int64_t)y * pitch;
  return p->pixel_bytes == 1 ? (int64_t)row[x] : (int64_t)((const uint16_t*)row)[x];
}

/* ------------------------------------------------------------------ tables */

/* Step 1 taps ("Gaussian smoothing having the appropriate scale";
 * Methods PAPER.md:533-536 "smoothed using a Gaussian convolution").  Reading R2/R3:
 * K_s = ceil(3 sigma_s); q_i = llround(1024 exp(-i^2 / (2 sigma_s^2))), unnormalised. */
int32_t orc_gauss_taps(double sigma_s, int32_t* taps, int32_t cap) {
  int32_t K = (int32_t)ceil(3.0 * sigma_s);
  if (2 * K + 1 > cap) return -1;
  for (int32_t i = -K; i <= K; ++i) taps[i + K] = (int32_t)llround(1024.0 * exp(-(double)(i * i) / (2.0 * sigma_s * sigma_s)));
  return K;
}

/* sigma(r) = 0.05 r + 0.25 (Methods) written as (a r + b)/den. */
double orc_sigma(const orc_params* p, int32_t r) { return (double)(p->sig_a * r + p->sig_b) / (double)p->sig_den; }

/* K_r = ceil(3 sigma(r)) in exact integer form (reading R12). */
int32_t orc_level_halfwidth(const orc_params* p, int32_t r) {
  int32_t num = 3 * (p->sig_a * r + p->sig_b);
  return (num + p->sig_den - 1) / p->sig_den;
}

/* Gaussian weight exp(-d^2 / (2 sigma(r)^2)) of the radius-dependent smoothing
 * (PAPER.md:538-541 Methods; SI step 4 PAPER.md:962-965), 12-bit fixed point (R11). */
int32_t orc_level_weight(const orc_params* p, int32_t r, int32_t d) {
  int64_t s = (int64_t)p->sig_a * r + p->sig_b;
  double num = (double)((int64_t)d * d * p->sig_den * p->sig_den);
  double den = 2.0 * (double)(s * s);
  return (int32_t)llround(4096.0 * exp(-num / den));
}

/* Candidate threshold "a fraction of 2 pi", expressed in
 * the fixed-point units of S: N = S / (2^24 r) > tau 2 pi  <=>  S > tau 2 pi 2^24 r (R13). */
double orc_norm_threshold(const orc_params* p, int32_t r) {
  return ((p->vote_threshold_norm * (2.0 * M_PI)) * 16777216.0) * (double)r;
}

/* kappa threshold in the units of the unnormalised integer Hessian (R3, R5). */
double orc_curvature_threshold_int(const orc_params* p) {
  int32_t q[64];
  int32_t K = orc_gauss_taps(p->smoothing_sigma, q, 64);
  int64_t sq = 0;
  for (int i = 0; i <= 2 * K; ++i) sq += q[i];
  return p->curvature_threshold * (64.0 * (double)sq * (double)sq);
}

/* Annulus half-width (R15): max(2, ceil(2 sigma(r))) unless fixed by the caller. */
int32_t orc_annulus_halfwidth(const orc_params* p, int32_t r) {
  if (p->annulus_halfwidth > 0) return p->annulus_halfwidth;
  int32_t num = 2 * (p->sig_a * r + p->sig_b);
  int32_t w = (num + p->sig_den - 1) / p->sig_den;
  return w < 2 ? 2 : w;
}

/* ------------------------------------------------------------------ step 1 */
/* G[y][x] = sum_{i,j} q_i q_j I[clamp(y+i)][clamp(x+j)], evaluated as the separable
 * row-then-column pass OpenCV's GaussianBlur performs.  All
 * values are integers < 2^53, so the double result is exact. */
void orc_smooth(const orc_params* p, const void* frame, int64_t pitch, double* G) {
  const int W = p->width, H = p->height;
  int32_t q[64];
  int32_t K = orc_gauss_taps(p->smoothing_sigma, q, 64);
  int64_t* R = (int64_t*)malloc(sizeof(int64_t) * (size_t)W * H);
  for (int y = 0; y < H; ++y)
    for (int x = 0; x < W; ++x) {
      int64_t acc = 0;
      for (int j = -K; j <= K; ++j) acc += (int64_t)q[j + K] * pixel_at(p, frame, pitch, clampi(x + j, 0, W - 1), y);
      R[(size_t)y * W + x] = acc;
    }
  for (int y = 0; y < H; ++y)
    for (int x = 0; x < W; ++x) {
      int64_t acc = 0;
      for (int i = -K; i <= K; ++i) acc += (int64_t)q[i + K] * R[(size_t)clampi(y + i, 0, H - 1) * W + x];
      G[(size_t)y * W + x] = (double)acc;
    }
  free(R);
}

/* ------------------------------------------------------------------ step 2 */
/* 5x5 second-order Sobel (SI step 1 PAPER.md:921-923), correlation
 * form, reading R3: Ixx = s5_y (x) d2_x, Iyy = d2_y (x) s5_x, Ixy = d1_y (x) d1_x with
 * s5 = [1,4,6,4,1], d2 = [1,0,-2,0,1], d1 = [-1,-2,0,2,1].  Valid on [2,W-3]x[2,H-3]
 * (R7); elsewhere 0.  Exact integers in double. */
static const int S5[5] = {1, 4, 6, 4, 1};
static const int D2[5] = {1, 0, -2, 0, 1};
static const int D1[5] = {-1, -2, 0, 2, 1};

void orc_hessian(const orc_params* p, const double* G, double* Ixx, double* Iyy, double* Ixy) {
  const int W = p->width, H = p->height;
  memset(Ixx, 0, sizeof(double) * (size_t)W * H);
  memset(Iyy, 0, sizeof(double) * (size_t)W * H);
  memset(Ixy, 0, sizeof(double) * (size_t)W * H);
  /* separable evaluation (OpenCV Sobel = sepFilter2D): horizontal 1D pass, then vertical */
  double* hd2 = (double*)calloc((size_t)W * H, sizeof(double));
  double* hs5 = (double*)calloc((size_t)W * H, sizeof(double));
  double* hd1 = (double*)calloc((size_t)W * H, sizeof(double));
  for (int y = 0; y < H; ++y)
    for (int x = 2; x <= W - 3; ++x) {
      double a = 0, b = 0, c = 0;
      for (int j = -2; j <= 2; ++j) {
        double g = G[(size_t)y * W + x + j];
        a += D2[j + 2] * g;
        b += S5[j + 2] * g;
        c += D1[j + 2] * g;
      }
      hd2[(size_t)y * W + x] = a;
      hs5[(size_t)y * W + x] = b;
      hd1[(size_t)y * W + x] = c;
    }
  for (int y = 2; y <= H - 3; ++y)
    for (int x = 2; x <= W - 3; ++x) {
      double a = 0, b = 0, c = 0;
      for (int i = -2; i <= 2; ++i) {
        size_t k = (size_t)(y + i) * W + x;
        a += S5[i + 2] * hd2[k];
        b += D2[i + 2] * hs5[k];
        c += D1[i + 2] * hd1[k];
      }
      Ixx[(size_t)y * W + x] = a;
      Iyy[(size_t)y * W + x] = b;
      Ixy[(size_t)y * W + x] = c;
    }
  free(hd2);
  free(hs5);
  free(hd1);
}

/* Edge variant (NEXT-2): "replacing the Hessian by the Gradient ... the gradient magnitude
 * replacing kappa has to be a local maximum along the gradient direction".
 * Reading R19: OpenCV's first-order 5x5 Sobel, correlation form, Ix = s5_y (x) d1_x and
 * Iy = d1_y (x) s5_x, evaluated separably like orc_hessian; valid on [2,W-3]x[2,H-3]. */
void orc_gradient(const orc_params* p, const double* G, double* Ix, double* Iy) {
  const int W = p->width, H = p->height;
  memset(Ix, 0, sizeof(double) * (size_t)W * H);
  memset(Iy, 0, sizeof(double) * (size_t)W * H);
  double* hs5 = (double*)calloc((size_t)W * H, sizeof(double));
  double* hd1 = (double*)calloc((size_t)W * H, sizeof(double));
  for (int y = 0; y < H; ++y)
    for (int x = 2; x <= W - 3; ++x) {
      double b = 0, c = 0;
      for (int j = -2; j <= 2; ++j) {
        double g = G[(size_t)y * W + x + j];
        b += S5[j + 2] * g;
        c += D1[j + 2] * g;
      }
      hs5[(size_t)y * W + x] = b;
      hd1[(size_t)y * W + x] = c;
    }
  for (int y = 2; y <= H - 3; ++y)
    for (int x = 2; x <= W - 3; ++x) {
      double gx = 0, gy = 0;
      for (int i = -2; i <= 2; ++i) {
        size_t k = (size_t)(y + i) * W + x;
        gx += S5[i + 2] * hd1[k];
        gy += D1[i + 2] * hs5[k];
      }
      Ix[(size_t)y * W + x] = gx;
      Iy[(size_t)y * W + x] = gy;
    }
  free(hs5);
  free(hd1);
}

/* A ramp I = g x gives Ix = 8 (d1) * 16 (s5) * (sum q)^2 * g, so a threshold t_e in counts/px
 * is t_e * 128 (sum q)^2 in gradient units; squared (fp64) because magnitudes are compared
 * squared (R19). */
double orc_edge_threshold_int2(const orc_params* p) {
  int32_t q[64];
  int32_t K = orc_gauss_taps(p->smoothing_sigma, q, 64);
  int64_t sq = 0;
  for (int i = 0; i <= 2 * K; ++i) sq += q[i];
  double t = p->edge_threshold * (128.0 * (double)sq * (double)sq);
  return t * t;
}

/* ------------------------------------------------------------------ step 3 */
/* kappa = smaller eigenvalue of the Hessian [[a,b],[b,c]], rho = its unit
 * eigenvector ("the smaller principal curvature and the
 * corresponding eigenvector"; SI step 1 PAPER.md:923-925).  Fixed fp64 recipe (R3):
 *   T = a + c, e = a - c, D = e*e + 4*(b*b), s = sqrt(D), kappa = 0.5*(T - s);
 *   e >= 0: v = (-b, 0.5*(e + s)); else v = (0.5*(s - e), -b); rho = v / |v|.
 * Degenerate (e == 0 and b == 0): isotropic, direction undefined (R3). */
int orc_eigen(double a, double b, double c, double* kappa, double* dx, double* dy) {
  double T = a + c;
  double e = a - c;
  double bb = b * b;
  double ee = e * e;
  double D = ee + 4.0 * bb;
  double s = sqrt(D);
  *kappa = 0.5 * (T - s);
  if (e == 0.0 && b == 0.0) {
    *dx = 0.0;
    *dy = 0.0;
    return 1;
  }
  double vx, vy;
  if (e >= 0.0) {
    vx = -b;
    vy = 0.5 * (e + s);
  } else {
    vx = 0.5 * (s - e);
    vy = -b;
  }
  double n = sqrt(vx * vx + vy * vy);
  *dx = vx / n;
  *dy = vy / n;
  return 0;
}

/* ------------------------------------------------------------------ step 4 */
typedef struct ws_t {
  int W, H;
  double *G, *Ixx, *Iyy, *Ixy, *K, *DX, *DY;
  unsigned char* DEG;
} ws_t;

static int ws_alloc(ws_t* w, int W, int H) {
  size_t n = (size_t)W * H;
  w->W = W;
  w->H = H;
  w->G = (double*)malloc(n * sizeof(double));
  w->Ixx = (double*)malloc(n * sizeof(double));
  w->Iyy = (double*)malloc(n * sizeof(double));
  w->Ixy = (double*)malloc(n * sizeof(double));
  w->K = (double*)malloc(n * sizeof(double));
  w->DX = (double*)malloc(n * sizeof(double));
  w->DY = (double*)malloc(n * sizeof(double));
  w->DEG = (unsigned char*)malloc(n);
  return w->G && w->Ixx && w->Iyy && w->Ixy && w->K && w->DX && w->DY && w->DEG ? 0 : -1;
}
static void ws_free(ws_t* w) {
  free(w->G); free(w->Ixx); free(w->Iyy); free(w->Ixy); free(w->K); free(w->DX); free(w->DY); free(w->DEG);
}

/* Edge pixels (NEXT-2, reading R19): m2 = Ix*Ix + Iy*Iy (each operation
 * rounded, no FMA) replaces kappa; a candidate has m2 > (t_e 128 (sum q)^2)^2; rho = (Ix, Iy)/
 * sqrt(m2); m2 must be a local maximum along rho with the R6 tie rule mirrored:
 * m2_p >= m2(after) and m2_p > m2(before).  Candidates lie in [3,W-4]x[3,H-4].  The edge list
 * reuses orc_ridge records (kappa field = m2).  w->G holds the smoothed frame. */
static int64_t edges_ws(const orc_params* p, ws_t* w, orc_ridge* out, int64_t cap) {
  const int W = p->width, H = p->height;
  orc_gradient(p, w->G, w->Ixx, w->Iyy);   /* Ix, Iy in the Ixx, Iyy buffers */
  for (size_t k = 0; k < (size_t)W * H; ++k) {
    double gx = w->Ixx[k], gy = w->Iyy[k];
    double m2 = gx * gx + gy * gy;
    w->K[k] = m2;
    if (m2 > 0.0) {
      double n = sqrt(m2);
      w->DX[k] = gx / n;
      w->DY[k] = gy / n;
    } else {
      w->DX[k] = 0.0;
      w->DY[k] = 0.0;
    }
  }
  const double t2 = orc_edge_threshold_int2(p);
  int64_t n = 0;
  for (int y = 3; y <= H - 4; ++y)
    for (int x = 3; x <= W - 4; ++x) {
      size_t k = (size_t)y * W + x;
      double mp = w->K[k];
      if (!(mp > t2)) continue;
      int ox = (int)llround(w->DX[k]), oy = (int)llround(w->DY[k]);
      int after_plus = (oy > 0) || (oy == 0 && ox > 0);
      double m_plus = w->K[(size_t)(y + oy) * W + (x + ox)];
      double m_minus = w->K[(size_t)(y - oy) * W + (x - ox)];
      double m_after = after_plus ? m_plus : m_minus;
      double m_before = after_plus ? m_minus : m_plus;
      if (mp >= m_after && mp > m_before) {
        if (n < cap) {
          out[n].x = x;
          out[n].y = y;
          out[n].dx = w->DX[k];
          out[n].dy = w->DY[k];
          out[n].kappa = mp;
        }
        ++n;
      }
    }
  return n;
}

/* Ridge pixels ("(i) kappa < 0; (ii) kappa is a local minimum
 * along rho"; SI step 2 PAPER.md:926-931 "smaller than a pre-defined curvature
 * threshold (the latter is no greater than zero) ... local minimum along the
 * direction of rho").  Readings R5-R7: kappa < t_int; the two samples are the
 * 8-neighbours p +- (llround(dx), llround(dy)); the one after p in row-major order
 * must satisfy kappa_p <= kappa(after), the one before kappa_p < kappa(before);
 * candidates lie in [3,W-4]x[3,H-4]; degenerate pixels are never ridges. */
static int64_t ridges_ws(const orc_params* p, ws_t* w, const void* frame, int64_t pitch, orc_ridge* out,
                         int64_t cap) {
  const int W = p->width, H = p->height;
  orc_smooth(p, frame, pitch, w->G);
  if (p->feature == 1) return edges_ws(p, w, out, cap);
  orc_hessian(p, w->G, w->Ixx, w->Iyy, w->Ixy);
  for (int y = 2; y <= H - 3; ++y)
    for (int x = 2; x <= W - 3; ++x) {
      size_t k = (size_t)y * W + x;
      w->DEG[k] = (unsigned char)orc_eigen(w->Ixx[k], w->Ixy[k], w->Iyy[k], &w->K[k], &w->DX[k], &w->DY[k]);
    }
  const double t = orc_curvature_threshold_int(p);
  int64_t n = 0;
  for (int y = 3; y <= H - 4; ++y)
    for (int x = 3; x <= W - 4; ++x) {
      size_t k = (size_t)y * W + x;
      if (w->DEG[k]) continue;
      double kp = w->K[k];
      if (!(kp < t)) continue;
      int ox = (int)llround(w->DX[k]), oy = (int)llround(w->DY[k]);
      int after_plus = (oy > 0) || (oy == 0 && ox > 0); /* p + o follows p in row-major order */
      double k_plus = w->K[(size_t)(y + oy) * W + (x + ox)];
      double k_minus = w->K[(size_t)(y - oy) * W + (x - ox)];
      double k_after = after_plus ? k_plus : k_minus;
      double k_before = after_plus ? k_minus : k_plus;
      if (kp <= k_after && kp < k_before) {
        if (n < cap) {
          out[n].x = x;
          out[n].y = y;
          out[n].dx = w->DX[k];
          out[n].dy = w->DY[k];
          out[n].kappa = kp;
        }
        ++n;
      }
    }
  return n;
}

int64_t orc_ridges(const orc_params* p, const void* frame, int64_t pitch, orc_ridge* out, int64_t cap) {
  ws_t w;
  if (ws_alloc(&w, p->width, p->height)) { ws_free(&w); return -1; }
  int64_t n = ridges_ws(p, &w, frame, pitch, out, cap);
  ws_free(&w);
  return n;
}

/* ------------------------------------------------------------------ step 5 */
/* Directed votes ("each directed ridge pixel votes for all
 * candidate points ... directed along rho"; SI step 2 PAPER.md:931-933; range
 * [r_min-1, r_max+1] PAPER.md:998-1001; each vote "increments an accumulator by
 * one" PAPER.md:141-144).  Readings R8/R9: both senses s = +-1; target
 * (x + s*llround(r*dx), y + s*llround(r*dy)); out-of-frame votes are dropped. */
int64_t orc_votes(const orc_params* p, const orc_ridge* ridges, int64_t n_ridges, int32_t* raw) {
  const int W = p->width, H = p->height;
  const int r_lo = p->r_min - 1, r_hi = p->r_max + 1;
  int64_t votes = 0;
  for (int64_t k = 0; k < n_ridges; ++k) {
    for (int r = r_lo; r <= r_hi; ++r) {
      long long ox = llround((double)r * ridges[k].dx);
      long long oy = llround((double)r * ridges[k].dy);
      for (int s = 1; s >= -1; s -= 2) {
        long long tx = ridges[k].x + s * ox, ty = ridges[k].y + s * oy;
        if (tx < 0 || tx >= W || ty < 0 || ty >= H) continue;
        raw[(size_t)(r - r_lo) * W * H + (size_t)ty * W + (size_t)tx] += 1;
        ++votes;
      }
    }
  }
  return votes;
}

/* ------------------------------------------------------------------ step 7 */
/* Radius-dependent smoothing at a hotspot ("each equi-radius
 * level ... smoothed using Gaussian weights, whose width is proportional to the
 * radius"; Methods PAPER.md:538-544; SI step 4 PAPER.md:962-965 "a spatial average
 * ... weighted by a Gaussian function").  Reading R11: unnormalised square window
 * |i|,|j| <= K_r, weights w_r(i) w_r(j), out-of-frame cells 0; S in 2^-24 units. */
int64_t orc_window_sum(const orc_params* p, const int32_t* raw, int32_t r, int32_t y, int32_t x) {
  const int W = p->width, H = p->height;
  const int r_lo = p->r_min - 1;
  const int K = orc_level_halfwidth(p, r);
  const int32_t* lvl = raw + (size_t)(r - r_lo) * W * H;
  int64_t wt[256];
  if (K > 255) return -1;
  for (int d = 0; d <= K; ++d) wt[d] = orc_level_weight(p, r, d);
  int64_t S = 0;
  for (int i = -K; i <= K; ++i) {
    int yy = y + i;
    if (yy < 0 || yy >= H) continue;
    int64_t wi = wt[i < 0 ? -i : i];
    for (int j = -K; j <= K; ++j) {
      int xx = x + j;
      if (xx < 0 || xx >= W) continue;
      int64_t wj = wt[j < 0 ? -j : j];
      S += wi * wj * (int64_t)lvl[(size_t)yy * W + xx];
    }
  }
  return S;
}

/* ------------------------------------------------------------------ step 8 */
static int cmp_key(int32_t r1, int32_t y1, int32_t x1, int32_t r2, int32_t y2, int32_t x2) {
  if (r1 != r2) return r1 < r2 ? -1 : 1;
  if (y1 != y2) return y1 < y2 ? -1 : 1;
  if (x1 != x2) return x1 < x2 ? -1 : 1;
  return 0;
}
/* hotspot list is sorted by (r, y, x): binary search */
static const orc_hotspot* find_hot(const orc_hotspot* h, int64_t n, int32_t r, int32_t y, int32_t x) {
  int64_t lo = 0, hi = n - 1;
  while (lo <= hi) {
    int64_t mid = (lo + hi) / 2;
    int c = cmp_key(h[mid].r, h[mid].y, h[mid].x, r, y, x);
    if (c == 0) return &h[mid];
    if (c < 0) lo = mid + 1; else hi = mid - 1;
  }
  return NULL;
}

/* ------------------------------------------------------------------ step 10 */
/* Kasa algebraic circle fit ("a best fitting circle is found for
 * all ridge coordinates within the annulus"; reading R16): minimise
 * sum (z + D u + E v + F)^2, z = u^2 + v^2, on centred integer coordinates.
 * Normal equations solved by Gaussian elimination with partial pivoting. */
static int fit_moments(int64_t n, int64_t Su, int64_t Sv, int64_t Suu, int64_t Svv, int64_t Suv, int64_t Sz,
                       int64_t Suz, int64_t Svz, double* uc, double* vc, double* R) {
  if (n < 3) return 0;
  /* exact singularity test on the integer normal matrix */
  __int128 det = (__int128)Suu * ((__int128)Svv * n - (__int128)Sv * Sv)
               - (__int128)Suv * ((__int128)Suv * n - (__int128)Sv * Su)
               + (__int128)Su * ((__int128)Suv * Sv - (__int128)Svv * Su);
  if (det == 0) return 0;
  double A[3][4] = {{(double)Suu, (double)Suv, (double)Su, -(double)Suz},
                    {(double)Suv, (double)Svv, (double)Sv, -(double)Svz},
                    {(double)Su, (double)Sv, (double)n, -(double)Sz}};
  for (int c = 0; c < 3; ++c) {
    int piv = c;
    for (int r = c + 1; r < 3; ++r)
      if (fabs(A[r][c]) > fabs(A[piv][c])) piv = r;
    if (piv != c)
      for (int k = 0; k < 4; ++k) { double t = A[c][k]; A[c][k] = A[piv][k]; A[piv][k] = t; }
    for (int r = c + 1; r < 3; ++r) {
      double f = A[r][c] / A[c][c];
      for (int k = c; k < 4; ++k) A[r][k] -= f * A[c][k];
    }
  }
  double sol[3];
  for (int r = 2; r >= 0; --r) {
    double acc = A[r][3];
    for (int k = r + 1; k < 3; ++k) acc -= A[r][k] * sol[k];
    sol[r] = acc / A[r][r];
  }
  double D = sol[0], E = sol[1], F = sol[2];
  *uc = -D / 2.0;
  *vc = -E / 2.0;
  double R2 = (*uc) * (*uc) + (*vc) * (*vc) - F;
  if (!(R2 >= 0.0)) return 0;
  *R = sqrt(R2);
  return 1;
}

int orc_fit(const int32_t* xs, const int32_t* ys, int64_t n, int32_t cx, int32_t cy, double* fx, double* fy,
            double* fr, double* rms) {
  int64_t Su = 0, Sv = 0, Suu = 0, Svv = 0, Suv = 0, Sz = 0, Suz = 0, Svz = 0;
  for (int64_t k = 0; k < n; ++k) {
    int64_t u = xs[k] - cx, v = ys[k] - cy, z = u * u + v * v;
    Su += u; Sv += v; Suu += u * u; Svv += v * v; Suv += u * v; Sz += z; Suz += u * z; Svz += v * z;
  }
  double uc, vc, R;
  if (!fit_moments(n, Su, Sv, Suu, Svv, Suv, Sz, Suz, Svz, &uc, &vc, &R)) {
    *fx = cx; *fy = cy; *fr = 0; *rms = 0;
    return 0;
  }
  double acc = 0;
  for (int64_t k = 0; k < n; ++k) {
    double du = (double)(xs[k] - cx) - uc, dv = (double)(ys[k] - cy) - vc;
    double e = sqrt(du * du + dv * dv) - R;
    acc += e * e;
  }
  *fx = cx + uc;
  *fy = cy + vc;
  *fr = R;
  *rms = sqrt(acc / (double)n);
  return 1;
}

/* ------------------------------------------------------------------ pipeline */
typedef struct detect_ws {
  ws_t img;
  int32_t* raw;
  size_t raw_cells;
  orc_ridge* ridges;
  int64_t ridge_cap;
  orc_hotspot* hot;
  int64_t hot_cap;
  orc_hotspot* peaks;
  int64_t peak_cap;
  orc_stream_ws* sws;   /* non-NULL: steps 5-8 the streamed way (streamed.c) */
} detect_ws;

static int dws_init(detect_ws* d, const orc_params* p, int streamed) {
  memset(d, 0, sizeof *d);
  if (ws_alloc(&d->img, p->width, p->height)) return -1;
  if (streamed) {
    d->sws = orc_stream_ws_create(p);
    if (!d->sws) return -1;
  } else {
    int nr = p->r_max - p->r_min + 3;
    d->raw_cells = (size_t)nr * p->width * p->height;
    d->raw = (int32_t*)malloc(d->raw_cells * sizeof(int32_t));
    if (!d->raw) return -1;
  }
  d->ridge_cap = (int64_t)p->width * p->height;
  d->ridges = (orc_ridge*)malloc(sizeof(orc_ridge) * (size_t)d->ridge_cap);
  d->hot_cap = 1 << 16;
  d->hot = (orc_hotspot*)malloc(sizeof(orc_hotspot) * (size_t)d->hot_cap);
  d->peak_cap = 4096;
  d->peaks = (orc_hotspot*)malloc(sizeof(orc_hotspot) * (size_t)d->peak_cap);
  return d->ridges && d->hot && d->peaks ? 0 : -1;
}
static void dws_free(detect_ws* d) {
  ws_free(&d->img);
  orc_stream_ws_free(d->sws);
  free(d->raw);
  free(d->ridges);
  free(d->hot);
  free(d->peaks);
}

static int params_ok(const orc_params* p) {
  if (p->width < 5 || p->height < 5) return 0;
  if (p->pixel_bytes != 1 && p->pixel_bytes != 2) return 0;
  if (!(p->smoothing_sigma > 0) || p->smoothing_sigma > 10) return 0;
  if (p->feature != 0 && p->feature != 1) return 0;
  if (p->feature == 0 && !(p->curvature_threshold <= 0)) return 0;
  if (p->feature == 1 && !(p->edge_threshold > 0)) return 0;
  if (p->r_min < 2 || p->r_max <= p->r_min) return 0;
  if (p->vote_threshold_raw < 1 || !(p->vote_threshold_norm > 0)) return 0;
  if (p->sig_a < 0 || p->sig_den <= 0 || p->sig_a * p->r_min + p->sig_b <= 0) return 0;
  return 1;
}

/* steps 6-8 on a full raw accumulator.  Hotspots are appended to *hot (sorted by
 * (r, y, x)); peaks (as hotspot records, canonical order) to peaks[] up to
 * peak_cap.  Returns the number of peaks or -1 on allocation failure. */
static int64_t hot_and_peaks(const orc_params* p, const int32_t* raw, orc_hotspot** hot, int64_t* hot_cap,
                             int64_t* n_hot, orc_hotspot* peaks, int64_t peak_cap) {
  const int W = p->width, H = p->height;
  const int r_lo = p->r_min - 1, r_hi = p->r_max + 1;
  /* step 6: hotspots, "surpassed an integer threshold" (R10:
   * strict >), scanned in (r, y, x) order so the list is sorted */
  int64_t nh = 0;
  for (int r = r_lo; r <= r_hi; ++r) {
    const int32_t* lvl = raw + (size_t)(r - r_lo) * W * H;
    for (int y = 0; y < H; ++y)
      for (int x = 0; x < W; ++x) {
        int32_t v = lvl[(size_t)y * W + x];
        if (v > p->vote_threshold_raw) {
          if (nh == *hot_cap) {
            *hot_cap *= 2;
            *hot = (orc_hotspot*)realloc(*hot, sizeof(orc_hotspot) * (size_t)*hot_cap);
            if (!*hot) return -1;
          }
          orc_hotspot* h = &(*hot)[nh];
          h->r = r;
          h->y = y;
          h->x = x;
          h->raw = v;
          /* step 7: S(v) at the hotspot */
          h->S = orc_window_sum(p, raw, r, y, x);
          ++nh;
        }
      }
  }
  *n_hot = nh;
  const orc_hotspot* hs = *hot;
  /* step 8: candidates (r in [r_min, r_max], S > T_norm(r); PAPER.md:415-419,
   * 998-1001) that are 3x3x3 local maxima of N = S / (2^24 r) (PAPER.md:340,
   * 417-419, 969-972).  R14: non-hotspots have N = 0, out-of-frame neighbours are
   * ignored, ties go to the lexicographically smaller (r, y, x). */
  int64_t npk = 0;
  for (int64_t k = 0; k < nh; ++k) {
    const orc_hotspot* v = &hs[k];
    if (v->r < p->r_min || v->r > p->r_max) continue;
    if (!((double)v->S > orc_norm_threshold(p, v->r))) continue;
    int is_peak = 1;
    for (int dr = -1; dr <= 1 && is_peak; ++dr)
      for (int dy = -1; dy <= 1 && is_peak; ++dy)
        for (int dx = -1; dx <= 1 && is_peak; ++dx) {
          if (!dr && !dy && !dx) continue;
          int ur = v->r + dr, uy = v->y + dy, ux = v->x + dx;
          if (uy < 0 || uy >= H || ux < 0 || ux >= W) continue;
          const orc_hotspot* u = find_hot(hs, nh, ur, uy, ux);
          int64_t Su = u ? u->S : 0;
          __int128 lhs = (__int128)v->S * ur, rhs = (__int128)Su * v->r; /* N(v) vs N(u) */
          int wins = lhs > rhs || (lhs == rhs && cmp_key(v->r, v->y, v->x, ur, uy, ux) < 0);
          if (!wins) is_peak = 0;
        }
    if (!is_peak) continue;
    if (npk < peak_cap) peaks[npk] = *v;
    ++npk;
  }
  return npk;
}

int64_t orc_peaks(const orc_params* p, const int32_t* raw, orc_hotspot* peaks, int64_t peak_cap,
                  orc_hotspot* hot_out, int64_t hot_cap_out, int64_t* n_hot_out) {
  int64_t cap = 1 << 12, nh = 0;
  orc_hotspot* hot = (orc_hotspot*)malloc(sizeof(orc_hotspot) * (size_t)cap);
  if (!hot) return -1;
  int64_t npk = hot_and_peaks(p, raw, &hot, &cap, &nh, peaks, peak_cap);
  if (npk >= 0 && hot_out) memcpy(hot_out, hot, sizeof(orc_hotspot) * (size_t)(nh < hot_cap_out ? nh : hot_cap_out));
  if (n_hot_out) *n_hot_out = nh;
  free(hot);
  return npk;
}

/* steps 9-10 for one peak: annulus classification (non-exclusive; PAPER.md:342-349,
 * SI step 5 PAPER.md:979-984) over all ridges, then the Kasa fit (R15, R16). */
static void classify_fit(const orc_params* p, const orc_ridge* ridges, int64_t nr, const orc_hotspot* v,
                         orc_ring* g) {
  g->cx = v->x;
  g->cy = v->y;
  g->r = v->r;
  g->raw_votes = v->raw;
  g->score_fixed = v->S;
  int32_t w = orc_annulus_halfwidth(p, v->r);
  int64_t lo = v->r - w > 0 ? v->r - w : 0, hi = (int64_t)v->r + w;
  int64_t lo2 = lo * lo, hi2 = hi * hi;
  int64_t n = 0, Su = 0, Sv = 0, Suu = 0, Svv = 0, Suv = 0, Sz = 0, Suz = 0, Svz = 0;
  for (int64_t m = 0; m < nr; ++m) {
    int64_t u = ridges[m].x - v->x, vv = ridges[m].y - v->y, z = u * u + vv * vv;
    if (z < lo2 || z > hi2) continue;
    ++n; Su += u; Sv += vv; Suu += u * u; Svv += vv * vv; Suv += u * vv; Sz += z; Suz += u * z; Svz += vv * z;
  }
  g->inliers = (int32_t)n;
  double uc, vc, R;
  if (fit_moments(n, Su, Sv, Suu, Svv, Suv, Sz, Suz, Svz, &uc, &vc, &R)) {
    double acc = 0;
    for (int64_t m = 0; m < nr; ++m) {
      int64_t u = ridges[m].x - v->x, vv = ridges[m].y - v->y, z = u * u + vv * vv;
      if (z < lo2 || z > hi2) continue;
      double du = (double)u - uc, dv = (double)vv - vc;
      double e = sqrt(du * du + dv * dv) - R;
      acc += e * e;
    }
    g->fit_ok = 1;
    g->fx = v->x + uc;
    g->fy = v->y + vc;
    g->fr = R;
    g->rms = sqrt(acc / (double)n);
  } else {
    g->fit_ok = 0;
    g->fx = v->x;
    g->fy = v->y;
    g->fr = v->r;
    g->rms = 0;
  }
}

static int64_t detect_ws_run(const orc_params* p, detect_ws* d, const void* frame, int64_t pitch, orc_ring* rings,
                             int64_t ring_cap, orc_stats* stats, orc_ridge* ridges_out, int64_t ridge_cap,
                             orc_hotspot* hot_out, int64_t hot_cap) {
  /* steps 1-4 */
  int64_t nr = ridges_ws(p, &d->img, frame, pitch, d->ridges, d->ridge_cap);
  if (ridges_out)
    memcpy(ridges_out, d->ridges, sizeof(orc_ridge) * (size_t)(nr < ridge_cap ? nr : ridge_cap));
  int64_t votes, nh = 0, npk;
  if (d->sws) {
    /* steps 5-8 streamed (SI steps 2-4); hotspots are not collected */
    npk = orc_stream_peaks_ws(p, d->sws, d->ridges, nr, d->peaks, d->peak_cap, NULL, 0, &nh);
    if (npk > d->peak_cap) {
      d->peak_cap = npk;
      d->peaks = (orc_hotspot*)realloc(d->peaks, sizeof(orc_hotspot) * (size_t)d->peak_cap);
      if (!d->peaks) return -1;
      npk = orc_stream_peaks_ws(p, d->sws, d->ridges, nr, d->peaks, d->peak_cap, NULL, 0, &nh);
    }
    if (npk < 0) return -1;
    votes = orc_stream_votes(d->sws);
    hot_out = NULL;
  } else {
    /* step 5: full accumulator, zeroed per frame */
    memset(d->raw, 0, d->raw_cells * sizeof(int32_t));
    votes = orc_votes(p, d->ridges, nr, d->raw);
    /* steps 6-8 */
    npk = hot_and_peaks(p, d->raw, &d->hot, &d->hot_cap, &nh, d->peaks, d->peak_cap);
    if (npk < 0) return -1;
    if (npk > d->peak_cap) { /* grow and redo the (cheap) peak pass */
      d->peak_cap = npk;
      d->peaks = (orc_hotspot*)realloc(d->peaks, sizeof(orc_hotspot) * (size_t)d->peak_cap);
      if (!d->peaks) return -1;
      npk = hot_and_peaks(p, d->raw, &d->hot, &d->hot_cap, &nh, d->peaks, d->peak_cap);
    }
  }
  if (hot_out) memcpy(hot_out, d->hot, sizeof(orc_hotspot) * (size_t)(nh < hot_cap ? nh : hot_cap));
  /* steps 9-10, rings in canonical (r, cy, cx) order (the hotspot scan order) */
  for (int64_t k = 0; k < npk && k < ring_cap; ++k) classify_fit(p, d->ridges, nr, &d->peaks[k], &rings[k]);
  if (stats) {
    stats->ridges = nr;
    stats->votes = votes;
    stats->hotspots = nh;
    stats->peaks = npk;
  }
  return npk;
}

int64_t orc_detect(const orc_params* p, const void* frame, int64_t pitch, orc_ring* rings, int64_t ring_cap,
                   orc_stats* stats, orc_ridge* ridges_out, int64_t ridge_cap, orc_hotspot* hot_out,
                   int64_t hot_cap) {
  if (!params_ok(p)) return -1;
  detect_ws d;
  if (dws_init(&d, p, 0)) { dws_free(&d); return -1; }
  int64_t n = detect_ws_run(p, &d, frame, pitch, rings, ring_cap, stats, ridges_out, ridge_cap, hot_out, hot_cap);
  dws_free(&d);
  return n;
}

typedef struct {
  const orc_params* p;
  const uint8_t* frames;
  int64_t stride;
  int32_t n;
  orc_ring* rings;
  int32_t ring_stride;
  int32_t* counts;
  orc_stats* stats;
  int next;
  int err;
  int streamed;
  pthread_mutex_t mu;
} batch_t;

typedef struct {
  batch_t* b;
  detect_ws* ws;   /* a pool's workspace (kept across calls), or NULL: allocate per call */
  int* ready;
} worker_t;

static void* batch_worker(void* arg) {
  worker_t* w = (worker_t*)arg;
  batch_t* b = w->b;
  detect_ws local;
  detect_ws* dp = w->ws ? w->ws : &local;
  detect_ws d;
  if (!w->ws || !*w->ready) {
    if (dws_init(dp, b->p, b->streamed)) { dws_free(dp); b->err = 1; return NULL; }
    if (w->ws) *w->ready = 1;
  }
  d = *dp;
  for (;;) {
    pthread_mutex_lock(&b->mu);
    int i = b->next++;
    pthread_mutex_unlock(&b->mu);
    if (i >= b->n) break;
    orc_stats st;
    int64_t c = detect_ws_run(b->p, &d, b->frames + (size_t)i * b->stride, (int64_t)b->p->width * b->p->pixel_bytes,
                              b->rings + (size_t)i * b->ring_stride, b->ring_stride, &st, NULL, 0, NULL, 0);
    if (c < 0) b->err = 1;
    b->counts[i] = (int32_t)(c > b->ring_stride ? -1 : c);
    if (b->stats) b->stats[i] = st;
  }
  if (w->ws) *w->ws = d;   /* buffers may have grown */
  else dws_free(&d);
  return NULL;
}

static int detect_batch(const orc_params* p, const void* frames, int64_t stride, int32_t n, orc_ring* rings,
                        int32_t ring_stride, int32_t* counts, orc_stats* stats, int32_t nthreads, int streamed) {
  if (!params_ok(p)) return -1;
  if (nthreads <= 0) nthreads = (int32_t)sysconf(_SC_NPROCESSORS_ONLN);
  if (nthreads > n) nthreads = n > 0 ? n : 1;
  if (nthreads > 512) nthreads = 512;
  batch_t b = {p, (const uint8_t*)frames, stride, n, rings, ring_stride, counts, stats, 0, 0, streamed,
               PTHREAD_MUTEX_INITIALIZER};
  pthread_t th[512];
  worker_t w[512];
  for (int t = 0; t < nthreads; ++t) {
    w[t].b = &b;
    w[t].ws = NULL;
    w[t].ready = NULL;
    pthread_create(&th[t], NULL, batch_worker, &w[t]);
  }
  for (int t = 0; t < nthreads; ++t) pthread_join(th[t], NULL);
  return b.err ? -1 : 0;
}

/* A thread pool's per-thread workspaces kept across calls (bench.py's timing legs): the
 * arithmetic is that of orc_detect_batch; only the allocation of the full arrays (and its page
 * faults) is paid once instead of once per call.  Each frame still re-zeroes its arrays. */
struct orc_pool {
  orc_params p;
  int32_t nthreads, streamed;
  detect_ws ws[512];
  int ready[512];
};

orc_pool* orc_pool_create(const orc_params* p, int32_t nthreads, int32_t streamed) {
  if (!params_ok(p)) return NULL;
  orc_pool* pl = (orc_pool*)calloc(1, sizeof(orc_pool));
  if (!pl) return NULL;
  pl->p = *p;
  if (nthreads <= 0) nthreads = (int32_t)sysconf(_SC_NPROCESSORS_ONLN);
  pl->nthreads = nthreads > 512 ? 512 : nthreads;
  pl->streamed = streamed;
  return pl;
}

void orc_pool_free(orc_pool* pl) {
  if (!pl) return;
  for (int t = 0; t < pl->nthreads; ++t)
    if (pl->ready[t]) dws_free(&pl->ws[t]);
  free(pl);
}

int orc_pool_detect(orc_pool* pl, const void* frames, int64_t stride, int32_t n, orc_ring* rings, int32_t ring_stride,
                    int32_t* counts, orc_stats* stats) {
  if (!pl) return -1;
  batch_t b = {&pl->p, (const uint8_t*)frames, stride, n, rings, ring_stride, counts, stats, 0, 0, pl->streamed,
               PTHREAD_MUTEX_INITIALIZER};
  const int nt = pl->nthreads < n ? pl->nthreads : (n > 0 ? n : 1);
  pthread_t th[512];
  worker_t w[512];
  for (int t = 0; t < nt; ++t) {
    w[t].b = &b;
    w[t].ws = &pl->ws[t];
    w[t].ready = &pl->ready[t];
    pthread_create(&th[t], NULL, batch_worker, &w[t]);
  }
  for (int t = 0; t < nt; ++t) pthread_join(th[t], NULL);
  return b.err ? -1 : 0;
}

int orc_detect_batch(const orc_params* p, const void* frames, int64_t stride, int32_t n, orc_ring* rings,
                     int32_t ring_stride, int32_t* counts, orc_stats* stats, int32_t nthreads) {
  return detect_batch(p, frames, stride, n, rings, ring_stride, counts, stats, nthreads, 0);
}

int orc_detect_batch_streamed(const orc_params* p, const void* frames, int64_t stride, int32_t n, orc_ring* rings,
                              int32_t ring_stride, int32_t* counts, orc_stats* stats, int32_t nthreads) {
  return detect_batch(p, frames, stride, n, rings, ring_stride, counts, stats, nthreads, 1);
}
