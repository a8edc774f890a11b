/* synth.h — seeded synthetic ring-frame generator (test/bench INPUT module).
 *
 * This module produces the frames that BOTH the CPU oracle (oracle/) and the CUDA
 * path (paper_1310_1371_b200/) consume.  It holds none of the detection method's
 * arithmetic: it only draws ring layouts and renders Gaussian-profile rings plus
 * noise, following the workload recipes of BASELINE.json `configs` as read in
 * SURVEY.md §8(d) / DESIGN.md "Input recipe".  The paper's own frames (PAPER.md
 * 611-627, 686-697: 968x728 8-bit CCD frames, ~50 particles) are not available;
 * these synthetic frames stand in for them.
 *
 * Randomness is counter based (SplitMix64 finaliser keyed by config, seed, frame
 * index, stream and counter), so frame i is identical regardless of how frames
 * are split across threads, processes or GPUs.
 */
#ifndef SYNTH_H
#define SYNTH_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct synth_ring {
  double cx, cy;      /* centre, pixel units (pixel (x,y) sits at integer coordinates) */
  double r;           /* ring radius (crest), pixels */
  double amp;         /* crest amplitude above background (counts) */
  double occ_start;   /* removed arc start angle (rad), valid if occ_len > 0 */
  double occ_len;     /* removed arc length (rad); 0 = not occluded */
  int32_t group;      /* -1 single; >=0 id of its overlapping / nested pair */
  int32_t kind;       /* 0 single, 1 overlapping pair member, 2 nested pair member, 3 steered (cfg4) */
} synth_ring;

typedef struct synth_scene {
  int32_t width, height;
  int32_t pixel_bytes;    /* 1 = uint8, 2 = uint16 */
  int32_t max_value;      /* clip value: 255 or 4095 */
  double background;      /* counts */
  double sigma_p;         /* radial Gaussian profile sigma (px) */
  double read_sigma;      /* additive Gaussian noise sigma (counts) */
  int32_t poisson;        /* 1: shot noise (Poisson(lambda), normal approximation, lambda>=background) */
} synth_scene;

/* Shapes of the BASELINE.json configs (cfg_id 1..5) and of test variants
 * (11 = "1x": cfg1 noiseless, integer centres).  Returns 0 on success, -1 for an
 * unknown id. batch = the config's batch size (cfg5: 8192). */
int synth_config_shape(int cfg_id, int32_t* width, int32_t* height, int32_t* pixel_bytes,
                       int32_t* max_value, int32_t* batch);

/* Scene parameters (profile, background, noise) of a config. */
int synth_config_scene(int cfg_id, synth_scene* out);

/* Draws the ring layout of frame `frame_idx` of config `cfg_id`. Writes at most
 * `cap` rings; returns the number of rings (or -1 on bad id). */
int synth_layout(int cfg_id, uint64_t seed, int64_t frame_idx, synth_ring* rings, int32_t cap);

/* Renders rings onto a frame with the scene's background, profile and noise.
 * out: pixel_bytes-wide pixels, row pitch `pitch_bytes`.  noise_key selects the
 * noise stream.  Returns 0 on success. */
int synth_render(const synth_scene* scene, const synth_ring* rings, int32_t n_rings,
                 uint64_t noise_key, void* out, int64_t pitch_bytes);

/* Layout + render of one config frame (contiguous rows).  truth may be NULL. */
int synth_frame(int cfg_id, uint64_t seed, int64_t frame_idx, void* out,
                synth_ring* truth, int32_t truth_cap, int32_t* n_truth);

/* Frames [first, first+n) of a config into a contiguous buffer (frame stride =
 * W*H*pixel_bytes), using `nthreads` host threads (<=0: all online cores). */
int synth_batch(int cfg_id, uint64_t seed, int64_t first_frame, int32_t n, void* out, int32_t nthreads);

/* Counter-based RNG exposed for tests: uniform double in [0,1) from (key, counter). */
double synth_u01(uint64_t key, uint64_t counter);
uint64_t synth_key(uint64_t a, uint64_t b, uint64_t c);

#ifdef __cplusplus
}
#endif
#endif
