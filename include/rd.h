/* rd.h — C ABI of librd.so, the B200 (sm_100a) ring detector.
 *
 * The library implements the data-parallel hot path of Afik's ridge-directed
 * circle-Hough ring detector (arXiv 1310.1371; /root/reference/PAPER.md), as
 * stated in the paper's problem statement: frames in; per frame, ring centre and
 * radius lists with their vote support out (PAPER.md:109-126 Introduction,
 * PAPER.md:218-226 and 275-276 Fig. 2(f) "best fit circle").  Steps:
 *   A1-A4 ridge extraction  (SI steps 1-2 PAPER.md:919-933)
 *   A5-A8 directed voting, radius-dependent smoothing, 1/r normalisation, 3x3x3
 *         peaks (SI steps 2-4 PAPER.md:931-978, 998-1001)
 *   A9-A11 annulus classification, circle fit, output (SI step 5
 *         PAPER.md:979-984)
 * Every integer result (ridge set, accumulator counts, S values, peaks, inlier
 * counts) is bit-identical to the CPU oracle (oracle/); fitted
 * centres/radii agree within 1e-4 px.
 *
 * Conventions
 *  - All functions return rd_status and never throw.  Plain pointers and sizes
 *    only; "d_" pointers are CUDA device pointers, "h_" pointers host pointers.
 *  - The caller owns frames and output buffers; the detector owns its scratch,
 *    allocated once in rd_create (no allocation inside rd_detect).
 *  - rd_detect is asynchronous and stream ordered on the caller's stream.  Errors
 *    found on the device (capacity overflow) are reported per frame (count = -1)
 *    and by rd_sync / rd_query_overflow.  Nothing is truncated silently.
 *  - One detector per host thread / stream at a time.  The library contains no
 *    collectives: multi-GPU sharding lives in the Python layer.
 */
#ifndef RD_H
#define RD_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define RD_ABI_VERSION 2

typedef enum rd_status {
  RD_OK = 0,
  RD_ERR_PARAM = 1,     /* invalid argument / config value (synchronous) */
  RD_ERR_DIM = 2,       /* frame geometry unsupported */
  RD_ERR_CONFIG = 3,    /* config inconsistent (e.g. overflow bound violated) */
  RD_ERR_CAPACITY = 4,  /* a per-frame/per-tile capacity overflowed on the device */
  RD_ERR_CUDA = 5,      /* CUDA runtime error (message: rd_last_error) */
  RD_ERR_STATE = 6      /* call out of order (e.g. dump before detect) */
} rd_status;

typedef enum rd_pixel { RD_U8 = 0, RD_U16 = 1 } rd_pixel;

/* Detector configuration.  Paper parameters
 * plus the capacities of this implementation.  rd_config_init fills defaults. */
typedef struct rd_config {
  int32_t width, height;          /* frame size in pixels, each >= 8 and <= 16384   -> RD_ERR_DIM */
  int32_t pixel;                  /* RD_U8 | RD_U16 */
  int32_t max_value;              /* upper bound of pixel values (255 / 4095 / 65535) */
  double smoothing_sigma;         /* sigma_s in (0, 5] px          -> RD_ERR_PARAM */
  double curvature_threshold;     /* t <= 0, counts/px^2 of the sigma_s-smoothed image */
  int32_t r_min, r_max;           /* 2 <= r_min < r_max <= 1000; Hough over [r_min-1, r_max+1] */
  int32_t vote_threshold_raw;     /* 1..60000; hotspot iff raw count > this */
  double vote_threshold_norm;     /* tau > 0; candidate iff S/(2^24 r) > tau*2*pi */
  int32_t sig_a, sig_b, sig_den;  /* sigma(r) = (a r + b)/den; 1, 5, 20 = 0.05 r + 0.25 */
  int32_t annulus_halfwidth;      /* 0: max(2, ceil(2 sigma(r))); else fixed w >= 1 */
  int32_t max_rings_per_frame;    /* output capacity per frame (default 1024) */
  int32_t max_ridges_per_tile;    /* ridges per 32x32 tile (default 512) */
  int32_t max_entries_per_tile;   /* voting rays per Hough tile (default 3072; tiles are 96x96 or 64x64) */
  int32_t max_hotspots_per_level; /* hotspots per Hough tile per level (0 = automatic: 160 for ridges,
                                     256 for edges; cfg3 ridges need < 128) */
  int32_t debug;                  /* 1: keep hotspot records for rd_dump_hotspots */
  /* ABI 2: feature selection ("replaced by directed edges ... replacing the
   * Hessian by the Gradient ... the gradient magnitude ... a local maximum along the gradient
   * direction"; reading R19).  RD_FEATURE_EDGE uses the 5x5 first-order Sobel gradient;
   * curvature_threshold is then ignored and edge_threshold (> 0, counts/px of the smoothed
   * image) selects candidates |grad| > edge_threshold.  Requires sigma_s <= 4.3 (K_s <= 13). */
  int32_t feature;                /* RD_FEATURE_RIDGE (0, default) | RD_FEATURE_EDGE (1)  -> RD_ERR_PARAM */
  double edge_threshold;          /* > 0 when feature == RD_FEATURE_EDGE                   -> RD_ERR_PARAM */
} rd_config;

enum { RD_FEATURE_RIDGE = 0, RD_FEATURE_EDGE = 1 };

/* One detected ring, 64 bytes.  (cx, cy, r, raw_votes, score_fixed, inliers,
 * fit_ok) are bit-exact; (fx, fy, fr, rms) agree with the oracle to 1e-4 px. */
typedef struct rd_ring {
  int32_t cx, cy, r;      /* integer Hough peak (PAPER.md:316-320 apex) */
  int32_t raw_votes;      /* raw accumulator count at the peak voxel */
  int64_t score_fixed;    /* S, Gaussian-weighted level sum in 2^-24 units; N = S / (2^24 r) */
  int32_t inliers;        /* ridge pixels inside the annulus (vote support, non-exclusive) */
  int32_t fit_ok;         /* 1 if inliers >= 3 and the Kasa system is regular */
  double fx, fy, fr;      /* sub-pixel centre and radius (Kasa fit) */
  double rms;             /* rms geometric residual of the inliers */
} rd_ring;

typedef struct rd_ridge { int32_t x, y; double dx, dy; } rd_ridge;          /* 24 B */
typedef struct rd_hotspot { int32_t r, y, x, raw; int64_t S; } rd_hotspot;  /* 24 B */
typedef struct rd_frame_stats { int64_t ridges, votes, hotspots, peaks; } rd_frame_stats;

typedef struct rd_detector rd_detector;

/* Library version / human-readable status / last CUDA error text (thread-local). */
int32_t rd_abi_version(void);
const char* rd_status_string(rd_status s);
const char* rd_last_error(void);

/* Defaults for a frame geometry: sigma_s 1.5, t -10, r in [8,70], T_raw 3,
 * tau 0.5, sigma(r) = (r+5)/20, default capacities.  cfg must be non-NULL. */
rd_status rd_config_init(rd_config* cfg, int32_t width, int32_t height, int32_t pixel);

/* Validates cfg, builds the level tables on the host and allocates all device
 * scratch for up to max_batch frames per rd_detect call on `device`. */
rd_status rd_create(const rd_config* cfg, int32_t max_batch, int32_t device, rd_detector** out);
rd_status rd_destroy(rd_detector* det);

/* Detects rings in n_frames frames resident on the device.
 *   d_frames: frame f, row y starts at d_frames + f*frame_stride_bytes + y*pitch_bytes;
 *             pixels are uint8 or uint16 per cfg.pixel (read only).
 *   d_rings:  n_frames * cfg.max_rings_per_frame records; frame f's rings start at
 *             d_rings + f*max_rings_per_frame, in canonical (r, cy, cx) order.
 *   d_counts: n_frames int32: number of rings, or -1 if a capacity overflowed.
 *   stream:   cudaStream_t (NULL = legacy default stream).
 * 1 <= n_frames <= max_batch.  Asynchronous. */
rd_status rd_detect(rd_detector* det, const void* d_frames, int64_t pitch_bytes, int64_t frame_stride_bytes,
                    int32_t n_frames, rd_ring* d_rings, int32_t* d_counts, void* stream);

/* End-to-end variant on HOST buffers (pinned memory recommended): copies frames
 * host->device in chunks (at most min(48, max_batch/2) frames, the first ones
 * smaller), up to 3 chunks ahead of the detection, which alternates between two
 * internal streams working on disjoint halves of the internal buffers, and copies
 * rings/counts back.  Any n_frames >= 1.  Synchronous: returns when h_rings/h_counts
 * are filled.  h_rings: n_frames * max_rings_per_frame records.  rd_sync,
 * rd_query_overflow and rd_get_stats do not describe rd_detect_host calls (the
 * counts of overflowed frames are -1 and the call returns RD_ERR_CAPACITY). */
rd_status rd_detect_host(rd_detector* det, const void* h_frames, int64_t pitch_bytes, int64_t frame_stride_bytes,
                         int32_t n_frames, rd_ring* h_rings, int32_t* h_counts);

/* Waits for the last rd_detect and reports RD_ERR_CAPACITY if any frame overflowed. */
rd_status rd_sync(rd_detector* det);

/* After rd_sync: per-frame overflow bit masks of the last call (bit0 ridges/tile,
 * bit1 voting rays/tile, bit2 hotspots/level, bit3 rings/frame, bit4 debug list). */
rd_status rd_query_overflow(rd_detector* det, int32_t n_frames, int32_t* h_flags);

/* After rd_sync: per-frame counters of the last call (ridges, in-frame votes,
 * hotspots, peaks).  Synchronous copy. */
rd_status rd_get_stats(rd_detector* det, int32_t n_frames, rd_frame_stats* h_stats);

/* Classification (A9) of frame `frame` of the last rd_detect
 * call: for each of the frame's rings, in the order rd_detect returned them, the ridge
 * pixels in its annulus (r-w)_+^2 <= (x-cx)^2 + (y-cy)^2 <= (r+w)^2 (non-exclusive: a pixel
 * may support several rings), packed x | y << 16, ordered by ridge bin (bin rows, bin
 * columns) and row-major within a bin.  Computed on the GPU on request (not part of
 * rd_detect).  h_offsets[0..min(offsets_cap, n_rings + 1)) receives the CSR offsets
 * (ring i owns members [h_offsets[i], h_offsets[i+1])), h_members the first min(cap,
 * total) members, *n_total the total (call again with a larger cap if needed; NULL
 * buffers with cap 0 query the sizes).  Synchronous.  RD_ERR_CAPACITY if the frame
 * overflowed (its ring count was -1); RD_ERR_STATE if there was no such frame. */
rd_status rd_ring_members(rd_detector* det, int32_t frame, int32_t* h_offsets, int32_t offsets_cap,
                          uint32_t* h_members, int64_t cap, int64_t* n_total);

/* Debug: ridge list of frame `frame` of the last call, in tile order (32x32 tiles,
 * row-major within a tile).  Writes min(n, cap) records, sets *n. */
rd_status rd_dump_ridges(rd_detector* det, int32_t frame, rd_ridge* h_out, int64_t cap, int64_t* n);

/* Debug (cfg.debug = 1): all hotspots (raw > T_raw) of frame `frame`, unordered. */
rd_status rd_dump_hotspots(rd_detector* det, int32_t frame, rd_hotspot* h_out, int64_t cap, int64_t* n);

/* Per-kernel timing with CUDA events recorded on the launching stream around each
 * of the detector's kernels (K1 ridges, K1.5 ray routing, K2 Hough, K3 fit).
 * rd_set_timing(det, 1) clears and enables accumulation; rd_kernel_times waits for the
 * recorded events and writes total milliseconds per kernel into h_ms[0..3] and the
 * number of timed rd_detect calls into *n_calls.  Disabled by default (no events). */
rd_status rd_set_timing(rd_detector* det, int32_t on);
rd_status rd_kernel_times(rd_detector* det, float* h_ms, int32_t* n_calls);

/* Profiling aid: per-phase SM-cycle counters of the Hough kernel, accumulated by one
 * thread per CTA at its barriers when enabled (on = 1 clears and enables; 0 disables).
 * h_cycles[0..15]: [0] ray gathering, [1] first step setup, [2] votes, [3] window sums,
 * [4] candidate bookkeeping + undo, [5] peaks + next setup, [15] number of CTAs.
 * Synchronous read; counters cost a few instructions per barrier while enabled. */
rd_status rd_phase_cycles(rd_detector* det, int32_t on, uint64_t* h_cycles);

/* Step A3 in isolation: the fp64 kappa / rho recipe on n
 * Hessians d_abc[3i..3i+2] = (Ixx, Ixy, Iyy) -> d_out[3i..3i+2] = (kappa, dx, dy),
 * d_degenerate[i] = 1 if isotropic.  Device pointers; asynchronous on stream. */
rd_status rd_eigen(const double* d_abc, int64_t n, double* d_out, int32_t* d_degenerate, void* stream);

#ifdef __cplusplus
}
#endif
#endif
