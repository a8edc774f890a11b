/* rd_san.c — a small C driver of librd.so for compute-sanitizer.
 *
 * Runs the whole hot path through the C ABI on seeded synthetic frames: rd_detect on a batch
 * (two concurrent parts when n >= 128... and one part below), rd_detect_host (chunked, two
 * streams), rd_ring_members and the debug dumps, then checks that every frame's count is >= 0
 * and that both paths agree.  No PyTorch, so the sanitizer sees only this library's kernels.
 *
 *   rd_san cfg n sigma_s t r_min r_max [debug]        exit 0 on success
 * (RD_K2_FORCE_REDO=1 in the environment sends every frame through the 16-bit redo pass.)
 */
#include <cuda_runtime.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "rd.h"
#include "../../synth/synth.h"

#define CHECK(x)                                                                 \
  do {                                                                           \
    int s_ = (int)(x);                                                           \
    if (s_) {                                                                    \
      fprintf(stderr, "%s:%d %s -> %d (%s)\n", __FILE__, __LINE__, #x, s_, rd_last_error()); \
      return 2;                                                                  \
    }                                                                            \
  } while (0)

int main(int argc, char** argv) {
  if (argc < 7) {
    fprintf(stderr, "usage: rd_san cfg n sigma_s t r_min r_max [debug]\n");
    return 1;
  }
  const int cfg = atoi(argv[1]), n = atoi(argv[2]);
  int32_t W, H, pb, mv, batch;
  if (synth_config_shape(cfg, &W, &H, &pb, &mv, &batch)) return 1;
  const size_t fbytes = (size_t)W * H * pb;
  void* h_frames = malloc(fbytes * n);
  if (synth_batch(cfg, 0, 0, n, h_frames, 0)) return 1;
  rd_config c;
  CHECK(rd_config_init(&c, W, H, pb == 1 ? RD_U8 : RD_U16));
  c.max_value = mv;
  c.smoothing_sigma = atof(argv[3]);
  c.curvature_threshold = atof(argv[4]);
  c.r_min = atoi(argv[5]);
  c.r_max = atoi(argv[6]);
  c.debug = argc > 7 ? atoi(argv[7]) : 0;
  rd_detector* det = NULL;
  CHECK(rd_create(&c, n, 0, &det));
  void* d_frames = NULL;
  rd_ring *d_rings = NULL, *h_rings = NULL, *h_rings2 = NULL;
  int32_t *d_counts = NULL, *d_offsets = NULL;
  const int cap = n * c.max_rings_per_frame;
  CHECK(cudaMalloc(&d_frames, fbytes * n));
  CHECK(cudaMalloc((void**)&d_rings, sizeof(rd_ring) * cap));
  CHECK(cudaMalloc((void**)&d_counts, sizeof(int32_t) * n));
  CHECK(cudaMalloc((void**)&d_offsets, sizeof(int32_t) * (n + 1)));
  CHECK(cudaMemcpy(d_frames, h_frames, fbytes * n, cudaMemcpyHostToDevice));
  cudaStream_t st;
  CHECK(cudaStreamCreate(&st));
  CHECK(rd_detect(det, d_frames, (int64_t)W * pb, (int64_t)fbytes, n, d_rings, cap, d_counts, d_offsets, st));
  CHECK(rd_sync(det));
  int32_t* counts = (int32_t*)malloc(sizeof(int32_t) * n);
  int32_t* offsets = (int32_t*)malloc(sizeof(int32_t) * (n + 1));
  int32_t* counts2 = (int32_t*)malloc(sizeof(int32_t) * n);
  int32_t* offsets2 = (int32_t*)malloc(sizeof(int32_t) * (n + 1));
  CHECK(cudaMemcpy(counts, d_counts, sizeof(int32_t) * n, cudaMemcpyDeviceToHost));
  CHECK(cudaMemcpy(offsets, d_offsets, sizeof(int32_t) * (n + 1), cudaMemcpyDeviceToHost));
  h_rings = (rd_ring*)malloc(sizeof(rd_ring) * (offsets[n] + 1));
  CHECK(cudaMemcpy(h_rings, d_rings, sizeof(rd_ring) * offsets[n], cudaMemcpyDeviceToHost));
  long total = 0;
  for (int i = 0; i < n; ++i) {
    if (counts[i] < 0) { fprintf(stderr, "frame %d overflowed\n", i); return 3; }
    total += counts[i];
  }
  /* classification and dumps of frame 0 */
  int64_t nm = 0;
  CHECK(rd_ring_members(det, 0, NULL, 0, NULL, 0, &nm));
  int64_t nr = 0;
  CHECK(rd_debug_dump(det, 0, RD_DUMP_RIDGES, NULL, 0, &nr));
  if (c.debug) {
    int64_t nf = 0, nh = 0;
    rd_level_fpr fpr[256];
    CHECK(rd_debug_dump(det, n - 1, RD_DUMP_LEVEL_FPR, fpr, sizeof fpr, &nf));
    CHECK(rd_debug_dump(det, 0, RD_DUMP_HOTSPOTS, NULL, 0, &nh));
  }
  /* the host path on the same frames: identical output */
  h_rings2 = (rd_ring*)malloc(sizeof(rd_ring) * cap);
  CHECK(rd_detect_host(det, h_frames, (int64_t)W * pb, (int64_t)fbytes, n, h_rings2, cap, counts2, offsets2));
  if (memcmp(counts, counts2, sizeof(int32_t) * n) || memcmp(offsets, offsets2, sizeof(int32_t) * (n + 1)) ||
      memcmp(h_rings, h_rings2, sizeof(rd_ring) * offsets[n])) {
    fprintf(stderr, "host path differs from the device path\n");
    return 4;
  }
  rd_overflow ov;
  CHECK(rd_query_overflow(det, &ov));
  CHECK(rd_destroy(det));
  printf("rd_san ok: cfg %d, %d frames, %ld rings, %lld members in frame 0, %lld ridges in frame 0\n", cfg, n, total,
         (long long)nm, (long long)nr);
  cudaFree(d_frames);
  cudaFree(d_rings);
  cudaFree(d_counts);
  cudaFree(d_offsets);
  cudaStreamDestroy(st);
  free(h_frames);
  free(h_rings);
  free(h_rings2);
  free(counts);
  free(offsets);
  free(counts2);
  free(offsets2);
  return 0;
}
