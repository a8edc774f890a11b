/* rd.h — C ABI of librd.so, the B200 (sm_100a) ring detector.
 *
 * The library implements the data-parallel hot path of Afik's ridge-directed
 * circle-Hough ring detector (arXiv 1310.1371; /root/reference/PAPER.md) as the paper
 * states the problem: frames in; per frame, the ring centres and radii with their vote
 * support out (PAPER.md:109-126 Introduction "classify/cluster the coordinates into
 * sub-sets, each sub-set matching a single ring"; Fig. 2(f) "the output:
 * best fit circle").  Steps:
 *   A1-A4 ridge extraction  (SI steps 1-2)
 *   A5-A8 directed voting, radius-dependent smoothing, 1/r normalisation, 3x3x3
 *         peaks (SI steps 2-4)
 *   A9-A11 annulus classification, circle fit, output (SI step 5,
 *         PAPER.md:979-984)
 * Every integer result (ridge set, accumulator counts, S values, peaks, inlier counts) is
 * bit-identical to the CPU oracle (oracle/); fitted centres/radii agree
 * within 1e-4 px.
 *
 * Conventions
 *  - Every function returns rd_status and never throws.  Plain pointers and sizes only;
 *    "d_" pointers are CUDA device pointers, "h_" pointers host pointers.
 *  - The caller owns frames and output buffers; the detector owns its scratch, allocated
 *    in rd_create (rd_detect never allocates; rd_detect_host allocates its staging once,
 *    on first use, and grows its ring staging only when a call asks for more).
 *  - rd_detect is asynchronous and stream ordered on the caller's stream.  Errors found on
 *    the device (a capacity overflowed) are reported per frame (count = -1) and by rd_sync /
 *    rd_query_overflow, which also returns the capacities that would have sufficed.
 *    Nothing is truncated silently.
 *  - One detector per host thread / stream at a time (calls on one detector are ordered:
 *    each call waits for the previous one's device work before reusing scratch).  The
 *    library contains no collectives: multi-GPU sharding lives in the Python layer.
 */
#ifndef RD_H
#define RD_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define RD_ABI_VERSION 4

typedef enum rd_status {
  RD_OK = 0,
  RD_ERR_PARAM = 1,     /* invalid argument / config value (synchronous) */
  RD_ERR_DIM = 2,       /* frame geometry unsupported */
  RD_ERR_CONFIG = 3,    /* config inconsistent (exactness bound violated, no kernel shape fits) */
  RD_ERR_CAPACITY = 4,  /* a capacity overflowed on the device: see rd_query_overflow */
  RD_ERR_CUDA = 5,      /* CUDA runtime error (message: rd_last_error) */
  RD_ERR_STATE = 6      /* call out of order (e.g. a dump before any rd_detect) */
} rd_status;

typedef enum rd_pixel { RD_U8 = 0, RD_U16 = 1 } rd_pixel;

/* Detector configuration: the paper's parameters (PAPER.md:289-292 sigma_s; 926-928 curvature
 * threshold; 538-544 sigma(r); 413-419 and 947-961 the two vote thresholds; 998-1001 the
 * extended Hough range) plus this implementation's capacities.  rd_config_init fills
 * defaults; readings R1-R19 fix what the paper leaves open. */
typedef struct rd_config {
  int32_t width, height;          /* frame size in pixels, each in [8, 16384]            -> RD_ERR_DIM   */
  int32_t pixel;                  /* RD_U8 | RD_U16                                      -> RD_ERR_PARAM */
  int32_t max_value;              /* upper bound of pixel values (255 / 4095 / 65535); sets the exactness
                                     bounds of the integer smoothing                     -> RD_ERR_CONFIG */
  double smoothing_sigma;         /* sigma_s > 0 with ceil(3 sigma_s) <= 13 */
  double curvature_threshold;     /* t <= 0, counts/px^2 of the sigma_s-smoothed image (R5) */
  int32_t r_min, r_max;           /* 2 <= r_min < r_max <= 1000; Hough over [r_min-1, r_max+1] */
  int32_t vote_threshold_raw;     /* 1..60000; hotspot iff raw count > this (R10) */
  double vote_threshold_norm;     /* tau > 0; candidate iff S/(2^24 r) > tau*2*pi (R13) */
  int32_t sig_a, sig_b, sig_den;  /* sigma(r) = (a r + b)/den; 1, 5, 20 = 0.05 r + 0.25 */
  int32_t annulus_halfwidth;      /* 0: w(r) = max(2, ceil(2 sigma(r))) (R15); else a fixed w >= 1 */
  int32_t max_rings_per_frame;    /* peaks kept per frame (default 1024) */
  int32_t max_ridges_per_tile;    /* ridges per 32x32 ridge bin (default 512, at most 1024) */
  int32_t max_entries_per_tile;   /* voting rays routed to one Hough tile (default 3072, at most 65535);
                                     rd_create picks the Hough tiling (rectangles of up to 254 px per side
                                     whose raw buffers fit shared memory, DESIGN.md §6 K2) */
  int32_t max_hotspots_per_level; /* hotspots per Hough tile per level (0 = automatic: 160 for ridges,
                                     256 for edges; at most 4095) */
  int32_t debug;                  /* 1: keep hotspot records and level fingerprints for rd_debug_dump */
  /* feature selection ("replaced by directed edges ... replacing the Hessian by
   * the Gradient ... the gradient magnitude ... a local maximum along the gradient direction";
   * reading R19).  RD_FEATURE_EDGE uses the 5x5 first-order Sobel gradient; curvature_threshold
   * is then ignored and edge_threshold (> 0, counts/px of the smoothed image) selects
   * candidates |grad| > edge_threshold. */
  int32_t feature;                /* RD_FEATURE_RIDGE (0, default) | RD_FEATURE_EDGE (1)  -> RD_ERR_PARAM */
  double edge_threshold;          /* > 0 when feature == RD_FEATURE_EDGE                   -> RD_ERR_PARAM */
} rd_config;

enum { RD_FEATURE_RIDGE = 0, RD_FEATURE_EDGE = 1 };

/* One detected ring, 64 bytes.  (cx, cy, r, raw_votes, score_fixed, inliers, fit_ok) are
 * bit-exact; (fx, fy, fr, rms) agree with the oracle to 1e-4 px. */
typedef struct rd_ring {
  int32_t cx, cy, r;      /* integer Hough peak: the apex of the vote cones */
  int32_t raw_votes;      /* raw accumulator count at the peak voxel */
  int64_t score_fixed;    /* S, Gaussian-weighted level sum in 2^-24 units; N = S / (2^24 r) */
  int32_t inliers;        /* ridge pixels inside the annulus = vote support, non-exclusive */
  int32_t fit_ok;         /* 1 if inliers >= 3 and the Kasa system is regular (R16) */
  double fx, fy, fr;      /* sub-pixel centre and radius (Kasa fit) */
  double rms;             /* rms geometric residual of the inliers */
} rd_ring;

typedef struct rd_ridge { int32_t x, y; double dx, dy; } rd_ridge;          /* 24 B */
typedef struct rd_hotspot { int32_t r, y, x, raw; int64_t S; } rd_hotspot;  /* 24 B */
typedef struct rd_frame_stats { int64_t ridges, votes, hotspots, peaks; } rd_frame_stats;
/* Per-level fingerprint of the raw accumulator of one frame (every voxel of the level once):
 * votes = sum raw, sq = sum raw^2, pos = sum raw * (y W + x) (mod 2^64). */
typedef struct rd_level_fpr { int32_t r, pad; int64_t votes, sq, pos; } rd_level_fpr;  /* 32 B */

/* Capacities a call needed (rd_query_overflow).  Each needed_* is the largest value the last
 * call met (not only when it overflowed), so a caller can size a detector for its data.  The
 * per-tile needs (rays per tile, hotspots per level) refer to the Hough tiling of that detector;
 * other capacities change the shared-memory layout and may change the tiling rd_create picks,
 * so resizing can take more than one round (Detector.sized_for in the Python binding iterates). */
typedef struct rd_overflow {
  int32_t frames_overflowed;         /* frames of the call whose count is -1 */
  int32_t flags;                     /* OR of the per-frame RD_OVF_* bits */
  int32_t needed_ridges_per_tile;    /* -> rd_config.max_ridges_per_tile */
  int32_t needed_entries_per_tile;   /* -> rd_config.max_entries_per_tile */
  int32_t needed_hotspots_per_level; /* -> rd_config.max_hotspots_per_level */
  int32_t needed_rings_per_frame;    /* -> rd_config.max_rings_per_frame */
  int64_t needed_rings_total;        /* -> ring_capacity_total of rd_detect / rd_detect_host */
} rd_overflow;

/* per-frame overflow bits (rd_query_flags) */
enum { RD_OVF_RIDGES = 1, RD_OVF_ENTRIES = 2, RD_OVF_HOTSPOTS = 4, RD_OVF_RINGS = 8, RD_OVF_DEBUG = 16,
       RD_OVF_OUTPUT = 32 };

typedef struct rd_detector rd_detector;

/* Library version / human-readable status / last CUDA or configuration error text
 * (thread-local). */
int32_t rd_abi_version(void);
const char* rd_status_string(rd_status s);
const char* rd_last_error(void);

/* Defaults for a frame geometry: sigma_s 1.5, t -10, r in [8,70], T_raw 3, tau 0.5,
 * sigma(r) = (r+5)/20, default capacities.  cfg must be non-NULL (else RD_ERR_PARAM). */
rd_status rd_config_init(rd_config* cfg, int32_t width, int32_t height, int32_t pixel);

/* Validates cfg (RD_ERR_DIM / RD_ERR_PARAM / RD_ERR_CONFIG, synchronously, before touching the
 * device), builds the level tables of the readings (taps q, K_r, w_r, T_norm(r), w(r)) on the
 * host, picks the kernel shapes and allocates all device scratch for up to max_batch >= 1
 * frames per rd_detect call on CUDA device `device`.  *out receives the detector (NULL on
 * error); the caller releases it with rd_destroy. */
rd_status rd_create(const rd_config* cfg, int32_t max_batch, int32_t device, rd_detector** out);
rd_status rd_destroy(rd_detector* det);   /* NULL is a no-op; waits for the detector's work */

/* Detects rings in n_frames frames resident on the device: the whole hot path A1-A11
 * (SI steps 1-5) as CUDA kernels on `stream`.
 *   d_frames:  frame f, row y starts at d_frames + f*frame_stride_bytes + y*pitch_bytes; pixels
 *              uint8 or uint16 per cfg.pixel (read only; pitch >= width * pixel bytes).
 *   d_rings:   ring_capacity_total records.  Frame f's rings are d_rings[d_offsets[f] ..
 *              d_offsets[f] + d_counts[f]) in canonical (r, cy, cx) order, frames back to back.
 *   d_counts:  n_frames int32: rings per frame, or -1 if a capacity overflowed for that frame
 *              (an internal one, or its rings do not fit in ring_capacity_total).
 *   d_offsets: n_frames + 1 int32: d_offsets[f] = sum of the rings of frames < f (frames with
 *              count -1 included by their true peak count, so d_offsets[n_frames] is the total
 *              the call needed; 0 for frames that overflowed an internal capacity).
 *   stream:    cudaStream_t (NULL = legacy default stream).
 * 1 <= n_frames <= max_batch.  Asynchronous; RD_ERR_PARAM for bad pointers/sizes. */
rd_status rd_detect(rd_detector* det, const void* d_frames, int64_t pitch_bytes, int64_t frame_stride_bytes,
                    int32_t n_frames, rd_ring* d_rings, int32_t ring_capacity_total, int32_t* d_counts,
                    int32_t* d_offsets, void* stream);

/* End-to-end variant on HOST buffers (pinned memory recommended): copies frames host->device
 * in chunks (at most min(48, max_batch/2) frames, the first ones smaller; behind a call in
 * flight, see rd_submit_host, min(96, max_batch/2) frames), up to 3 chunks ahead
 * of the detection, which alternates between two internal streams working on disjoint halves of
 * the internal buffers; the rings come back compacted as in rd_detect (only the rings found
 * cross the bus).  Any n_frames >= 1.  h_rings: ring_capacity_total records; h_counts: n_frames;
 * h_offsets: n_frames + 1.  Synchronous: returns when the outputs are filled; RD_ERR_CAPACITY if a
 * frame's count is -1 (rd_query_overflow then describes this call). */
rd_status rd_detect_host(rd_detector* det, const void* h_frames, int64_t pitch_bytes, int64_t frame_stride_bytes,
                         int32_t n_frames, rd_ring* h_rings, int32_t ring_capacity_total, int32_t* h_counts,
                         int32_t* h_offsets);

/* Pipelined form of rd_detect_host for streams of batches (the paper's frames arriving from
 * the camera while earlier ones are processed): rd_submit_host enqueues the
 * same work as rd_detect_host (same arguments and outputs) and returns at once, so the copies
 * of the next batch overlap the detection of this one; rd_wait_host completes the OLDEST
 * submitted call: it waits for it, then fills that call's h_rings / h_counts / h_offsets and
 * returns its status (RD_ERR_CAPACITY as rd_detect_host).  At most RD_HOST_DEPTH calls are in
 * flight: a further rd_submit_host, rd_wait_host with none in flight, and rd_detect_host /
 * rd_detect / every query while calls are in flight return RD_ERR_STATE.  h_frames must stay
 * unchanged and the output buffers valid until the call's rd_wait_host returns. */
enum { RD_HOST_DEPTH = 2 };
rd_status rd_submit_host(rd_detector* det, const void* h_frames, int64_t pitch_bytes, int64_t frame_stride_bytes,
                         int32_t n_frames, rd_ring* h_rings, int32_t ring_capacity_total, int32_t* h_counts,
                         int32_t* h_offsets);
rd_status rd_wait_host(rd_detector* det);

/* Waits for the last rd_detect; RD_ERR_CAPACITY if any frame overflowed. */
rd_status rd_sync(rd_detector* det);

/* After the last rd_detect / rd_detect_host (waits for it): what overflowed and the capacities
 * that would have sufficed (see rd_overflow).  RD_ERR_STATE before any call. */
rd_status rd_query_overflow(rd_detector* det, rd_overflow* h_out);

/* Per-frame RD_OVF_* bits of the last rd_detect (waits for it); n <= frames of that call. */
rd_status rd_query_flags(rd_detector* det, int32_t n_frames, int32_t* h_flags);

/* Per-frame counters of the last rd_detect (ridges, in-frame votes, hotspots, peaks).
 * Synchronous copy; RD_ERR_STATE after rd_detect_host (its chunks reuse the buffers). */
rd_status rd_get_stats(rd_detector* det, int32_t n_frames, rd_frame_stats* h_stats);

/* Classification (A9; "for each peak an annulus mask is formed ... ridge
 * coordinates within the annulus", SI step 5 PAPER.md:979-984) of frame `frame` of the last
 * rd_detect: for each of the frame's rings, in the order rd_detect returned them, the ridge
 * pixels in its annulus (r-w)_+^2 <= (x-cx)^2 + (y-cy)^2 <= (r+w)^2 (non-exclusive), packed
 * x | y << 16, ordered by ridge bin (bin rows, bin columns) and row-major within a bin.
 * Computed on the GPU on request on the detector's own stream (scratch preallocated, grown
 * only if a frame has more members than any before).  h_offsets[0..min(offsets_cap,
 * n_rings + 1)) receives the CSR offsets, h_members the first min(cap, total) members,
 * *n_total the total (NULL buffers with cap 0 query the sizes).  Synchronous.
 * RD_ERR_CAPACITY if the frame overflowed; RD_ERR_STATE if the last call had no such frame or
 * was rd_detect_host. */
rd_status rd_ring_members(rd_detector* det, int32_t frame, int32_t* h_offsets, int32_t offsets_cap,
                          uint32_t* h_members, int64_t cap, int64_t* n_total);

/* Stage-by-stage dumps of frame `frame` of the last rd_detect:
 *   RD_DUMP_RIDGES    rd_ridge[]      ridge list (A1-A4) in bin order (32x32 bins, row-major)
 *   RD_DUMP_LEVEL_FPR rd_level_fpr[]  one per level r_min-1 .. r_max+1 (A5; needs cfg.debug)
 *   RD_DUMP_HOTSPOTS  rd_hotspot[]    every hotspot with its S (A6-A7; needs cfg.debug), unordered
 *   RD_DUMP_MEMBERS   uint32_t[]      the members of rd_ring_members, all rings back to back
 * Writes at most cap_bytes into h_buf and sets *n_records to the full count (h_buf NULL with
 * cap_bytes 0 queries it).  Synchronous.  RD_ERR_STATE if unavailable (no call, host path,
 * debug off for the debug-only dumps). */
enum { RD_DUMP_RIDGES = 0, RD_DUMP_LEVEL_FPR = 1, RD_DUMP_HOTSPOTS = 2, RD_DUMP_MEMBERS = 3 };
rd_status rd_debug_dump(rd_detector* det, int32_t frame, int32_t what, void* h_buf, int64_t cap_bytes,
                        int64_t* n_records);

/* Per-kernel timing with CUDA events recorded on the launching stream around each of the
 * detector's kernels (K1 ridges, K1.5 ray routing, K2 Hough, K3 fit + output).
 * rd_set_timing(det, 1) clears and enables accumulation (a timed rd_detect runs on one stream);
 * rd_kernel_times waits for the recorded events and writes total milliseconds per kernel into
 * h_ms[0..3] and the number of timed rd_detect calls into *n_calls.  Off by default. */
rd_status rd_set_timing(rd_detector* det, int32_t on);
rd_status rd_kernel_times(rd_detector* det, float* h_ms, int32_t* n_calls);

/* Profiling aid (builds with -DRD_K2_PROF only): per-phase SM-cycle counters of the Hough
 * kernel.  h_cycles[0..15]: [0] ray gathering, [1] step setup, [2] votes, [3] window sums,
 * [4] clears + peaks, [15] CTAs.  on = 1 clears and enables; synchronous read. */
rd_status rd_phase_cycles(rd_detector* det, int32_t on, uint64_t* h_cycles);

/* Step A3 in isolation: the fp64 kappa / rho recipe (R3) on n Hessians
 * d_abc[3i..3i+2] = (Ixx, Ixy, Iyy) -> d_out[3i..3i+2] = (kappa, dx, dy); d_degenerate[i]: bit 0
 * set if isotropic, bits 1-2 = llround(dx) + 1 and bits 3-4 = llround(dy) + 1 as the ridge test
 * takes them (from the unnormalised direction, without the division).  Computed the way the
 * kernels split it (direction kept unnormalised by the ridge kernel, normalised by the ray
 * kernel).  Device pointers; asynchronous on stream. */
rd_status rd_eigen(const double* d_abc, int64_t n, double* d_out, int32_t* d_degenerate, void* stream);

#ifdef __cplusplus
}
#endif
#endif
