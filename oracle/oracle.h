/* oracle.h — plain, slow, obviously-correct CPU oracle of the ridge-directed
 * circle-Hough ring detector (Afik, arXiv 1310.1371; /root/reference/PAPER.md).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load or call this library.  The
 * product path (paper_1310_1371_b200/) never links, imports or executes it, and it
 * shares no code, header, table generator or constant with that path.
 *
 * Every function follows SURVEY.md §8(c) steps 1-10 / DESIGN.md "Readings" and
 * cites the PAPER.md passage it implements.  The full (N_r x H x W) accumulator is
 * materialised: the paper states that its streamed 3-level evaluation reaches the
 * same result (SI step 4 at PAPER.md:941-978), so the full array
 * is the definition of record.  Built with -ffp-contract=off.
 */
#ifndef RD_ORACLE_H
#define RD_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct orc_params {
  int32_t width, height;
  int32_t pixel_bytes;          /* 1 (uint8) or 2 (uint16) */
  double smoothing_sigma;       /* sigma_s */
  double curvature_threshold;   /* t <= 0, counts/px^2 */
  int32_t r_min, r_max;         /* search range; Hough over [r_min-1, r_max+1] */
  int32_t vote_threshold_raw;   /* hotspot iff raw > this */
  double vote_threshold_norm;   /* tau: candidate iff N > tau*2*pi */
  int32_t sig_a, sig_b, sig_den;/* sigma(r) = (a r + b)/den = 0.05 r + 0.25 */
  int32_t annulus_halfwidth;    /* 0: max(2, ceil(2 sigma(r))) */
  int32_t feature;              /* 0: directed ridges (Hessian); 1: directed edges (gradient) */
  double edge_threshold;        /* edges: |grad| > this, counts/px of the sigma_s-smoothed image (R19) */
} orc_params;

typedef struct orc_ridge { int32_t x, y; double dx, dy, kappa; } orc_ridge;
typedef struct orc_hotspot { int32_t r, y, x, raw; int64_t S; } orc_hotspot;
typedef struct orc_ring {
  int32_t cx, cy, r, raw_votes;
  int64_t score_fixed;
  int32_t inliers, fit_ok;
  double fx, fy, fr, rms;
} orc_ring;
typedef struct orc_stats { int64_t ridges, votes, hotspots, peaks; } orc_stats;

/* ---- tables ---- */
int32_t orc_gauss_taps(double sigma_s, int32_t* taps, int32_t cap);          /* returns K_s; taps[0..2K_s] */
int32_t orc_level_halfwidth(const orc_params* p, int32_t r);                 /* K_r = ceil(3 sigma(r)) */
int32_t orc_level_weight(const orc_params* p, int32_t r, int32_t d);         /* w_r(d), 2^12 fixed point */
double orc_sigma(const orc_params* p, int32_t r);                            /* sigma(r) as a double */
double orc_norm_threshold(const orc_params* p, int32_t r);                   /* T_norm(r) in S units */
double orc_curvature_threshold_int(const orc_params* p);                     /* t * 64 * (sum q)^2 */
int32_t orc_annulus_halfwidth(const orc_params* p, int32_t r);

/* ---- stages ---- */
/* step 1: G = (q (x) q) * I with replicate border; exact integers in double */
void orc_smooth(const orc_params* p, const void* frame, int64_t pitch_bytes, double* G);
/* step 2: 5x5 second-order Sobel (correlation) on [2,W-3]x[2,H-3]; outside = 0 */
void orc_hessian(const orc_params* p, const double* G, double* Ixx, double* Iyy, double* Ixy);
/* step 2 (edge variant, R19): 5x5 first-order Sobel gradient Ix = s5_y (x) d1_x, Iy = d1_y (x) s5_x
 * on [2,W-3]x[2,H-3]; outside = 0 */
void orc_gradient(const orc_params* p, const double* G, double* Ix, double* Iy);
/* edge threshold in the units of the squared integer gradient: (t_e * 128 * (sum q)^2)^2 */
double orc_edge_threshold_int2(const orc_params* p);
/* step 3: least principal curvature and its unit eigenvector; returns 1 if degenerate */
int orc_eigen(double a, double b, double c, double* kappa, double* dx, double* dy);
/* steps 1-4: ridge list in row-major order; returns count (<= cap written) */
int64_t orc_ridges(const orc_params* p, const void* frame, int64_t pitch_bytes, orc_ridge* out, int64_t cap);
/* step 5: votes of a ridge list into raw[(r - (r_min-1))*H*W + y*W + x] (caller zeroes); returns votes */
int64_t orc_votes(const orc_params* p, const orc_ridge* ridges, int64_t n_ridges, int32_t* raw);
/* step 7: S at voxel (level r, y, x) of a raw array */
int64_t orc_window_sum(const orc_params* p, const int32_t* raw, int32_t r, int32_t y, int32_t x);

/* steps 6-8 on a caller-supplied raw accumulator [N_r][H][W]: peaks (hotspot
 * records, canonical order) and optionally all hotspots.  Returns #peaks or -1. */
int64_t orc_peaks(const orc_params* p, const int32_t* raw, orc_hotspot* peaks, int64_t peak_cap,
                  orc_hotspot* hot_out, int64_t hot_cap, int64_t* n_hot);

/* streamed.c: the paper's own streamed form of steps 5-8 (SI steps 2-4):
 * sorted vote stack, 3-level raw and normalised sub-spaces indexed by r mod 3, registration
 * and undo.  Same outputs and order as orc_peaks on the full accumulator of the same ridges.
 * Returns #peaks or -1 on allocation failure. */
int64_t orc_stream_peaks(const orc_params* p, const orc_ridge* ridges, int64_t n_ridges, orc_hotspot* peaks,
                         int64_t peak_cap, orc_hotspot* hot_out, int64_t hot_cap, int64_t* n_hot);
/* the same with a per-thread workspace reused across frames (zero between calls) */
typedef struct orc_stream_ws orc_stream_ws;
orc_stream_ws* orc_stream_ws_create(const orc_params* p);
void orc_stream_ws_free(orc_stream_ws* w);
int64_t orc_stream_peaks_ws(const orc_params* p, orc_stream_ws* w, const orc_ridge* ridges, int64_t n_ridges,
                            orc_hotspot* peaks, int64_t peak_cap, orc_hotspot* hot_out, int64_t hot_cap,
                            int64_t* n_hot);
int64_t orc_stream_votes(const orc_stream_ws* w);   /* votes of the last call */

/* orc_detect_batch with steps 5-8 done the streamed way (NEXT-1): identical outputs. */
int orc_detect_batch_streamed(const orc_params* p, const void* frames, int64_t frame_stride_bytes, int32_t n_frames,
                              orc_ring* rings, int32_t ring_stride, int32_t* counts, orc_stats* stats,
                              int32_t nthreads);

/* orc_detect_batch with per-thread workspaces kept across calls (timing legs of bench.py):
 * same outputs, the full arrays are allocated once per pool thread instead of once per call. */
typedef struct orc_pool orc_pool;
orc_pool* orc_pool_create(const orc_params* p, int32_t nthreads, int32_t streamed);
int orc_pool_detect(orc_pool* pool, const void* frames, int64_t frame_stride_bytes, int32_t n_frames, orc_ring* rings,
                    int32_t ring_stride, int32_t* counts, orc_stats* stats);
void orc_pool_free(orc_pool* pool);

/* Whole pipeline, steps 1-10, for one frame.  rings: canonical (r, cy, cx) order.
 * Optional debug outputs may be NULL.  Returns the number of rings (all are
 * written only if <= ring_cap), or -1 on allocation failure / bad parameters. */
int64_t orc_detect(const orc_params* p, const void* frame, int64_t pitch_bytes,
                   orc_ring* rings, int64_t ring_cap, orc_stats* stats,
                   orc_ridge* ridges_out, int64_t ridge_cap,
                   orc_hotspot* hot_out, int64_t hot_cap);

/* Many frames with a pool of host threads (dynamic, one frame at a time, as the
 * paper's producer/consumer).  rings[f*ring_stride ..], counts[f].
 * Returns 0 on success. */
int orc_detect_batch(const orc_params* p, const void* frames, int64_t frame_stride_bytes, int32_t n_frames,
                     orc_ring* rings, int32_t ring_stride, int32_t* counts, orc_stats* stats, int32_t nthreads);

/* Kasa fit of integer points around (cx, cy): used by pins (step 10). */
int orc_fit(const int32_t* xs, const int32_t* ys, int64_t n, int32_t cx, int32_t cy,
            double* fx, double* fy, double* fr, double* rms);

#ifdef __cplusplus
}
#endif
#endif
