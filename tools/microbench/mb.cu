// Micro-benchmarks for design decisions (smem atomics, fp64, llround) on B200.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__global__ void k_atoms(uint32_t* out, int iters, int spread_mask, int mode) {
  extern __shared__ uint32_t sm[];
  for (int i = threadIdx.x; i < 8192; i += blockDim.x) sm[i] = 0;
  __syncthreads();
  uint32_t x = threadIdx.x * 2654435761u + blockIdx.x * 97u;
  uint32_t acc = 0;
  for (int it = 0; it < iters; ++it) {
    x = x * 1664525u + 1013904223u;
    uint32_t a = (x >> 8) & spread_mask;
    if (mode == 0) atomicAdd(&sm[a], 1u);
    else if (mode == 1) acc += atomicAdd(&sm[a], 1u);
    else if (mode == 2) { uint32_t inc = 1u << ((a & 1) * 16); atomicAdd(&sm[a >> 1], inc); }
    else { sm[a] += 1; }  // non-atomic baseline (racy)
  }
  __syncthreads();
  if (threadIdx.x == 0) out[blockIdx.x] = sm[0] + acc;
}

__global__ void k_dfma(double* out, int iters) {
  double a = threadIdx.x * 1.0001, b = 0.999, c = 1e-3, d = 2.0, e = 3.0, f = 4.0;
  for (int i = 0; i < iters; ++i) {
    a = fma(a, b, c); d = fma(d, b, c); e = fma(e, b, c); f = fma(f, b, c);
  }
  if (a + d + e + f == 12345.0) out[0] = a;
}
__global__ void k_llround(long long* out, int iters) {
  double v = threadIdx.x * 0.37;
  long long s = 0;
  for (int i = 0; i < iters; ++i) {
    s += llround(v); v += 1.25;
    s += llround(v * 0.5);
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void k_dsqrt(double* out, int iters) {
  double v = threadIdx.x + 1.0, s = 0;
  for (int i = 0; i < iters; ++i) { s += sqrt(v); v += 1.0; }
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void k_ddiv(double* out, int iters) {
  double v = threadIdx.x + 1.0, s = 0, w = 3.0;
  for (int i = 0; i < iters; ++i) { s += w / v; v += 1.0; }
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
  cudaDeviceProp p; cudaGetDeviceProperties(&p, 0);
  printf("%s SMs=%d clock=%d kHz smemPerSM=%zu\n", p.name, p.multiProcessorCount, p.clockRate, p.sharedMemPerMultiprocessor);
  int nsm = p.multiProcessorCount;
  uint32_t* d_out; cudaMalloc(&d_out, 1 << 24);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const char* names[] = {"atom_noret", "atom_ret", "atom_packed16", "nonatomic_rmw"};
  for (int mode = 0; mode < 4; ++mode)
  for (int spread : {8191, 1023, 31, 0}) {
    for (int blocks_per_sm : {2, 4}) {
      int threads = 512, iters = 4096;
      int grid = nsm * blocks_per_sm;
      k_atoms<<<grid, threads, 32768>>>(d_out, 16, spread, mode);
      cudaEventRecord(e0);
      k_atoms<<<grid, threads, 32768>>>(d_out, iters, spread, mode);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      double ops = (double)grid * threads * iters;
      printf("%-14s spread=%5d bps=%d: %.3f ms  %.1f Gop/s  %.3f op/clk/SM (at %.0f MHz nominal)\n", names[mode], spread + 1, blocks_per_sm, ms,
             ops / ms / 1e6, ops / (ms * 1e-3) / nsm / (p.clockRate * 1e3), p.clockRate / 1e3);
    }
  }
  {
    int grid = nsm * 4, threads = 512, iters = 1 << 14;
    k_dfma<<<grid, threads>>>((double*)d_out, 16);
    cudaEventRecord(e0); k_dfma<<<grid, threads>>>((double*)d_out, iters); cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double ops = (double)grid * threads * iters * 4;
    printf("DFMA: %.1f Gop/s = %.2f TFLOP/s  %.2f /clk/SM\n", ops / ms / 1e6, 2 * ops / ms / 1e9, ops / (ms * 1e-3) / nsm / (p.clockRate * 1e3));
  }
  {
    int grid = nsm * 4, threads = 512, iters = 1 << 12;
    k_llround<<<grid, threads>>>((long long*)d_out, 16);
    cudaEventRecord(e0); k_llround<<<grid, threads>>>((long long*)d_out, iters); cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double ops = (double)grid * threads * iters * 2;
    printf("llround: %.1f Gop/s  %.2f /clk/SM\n", ops / ms / 1e6, ops / (ms * 1e-3) / nsm / (p.clockRate * 1e3));
  }
  {
    int grid = nsm * 4, threads = 512, iters = 1 << 12;
    k_dsqrt<<<grid, threads>>>((double*)d_out, 16);
    cudaEventRecord(e0); k_dsqrt<<<grid, threads>>>((double*)d_out, iters); cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double ops = (double)grid * threads * iters;
    printf("dsqrt: %.1f Gop/s  %.2f /clk/SM\n", ops / ms / 1e6, ops / (ms * 1e-3) / nsm / (p.clockRate * 1e3));
  }
  {
    int grid = nsm * 4, threads = 512, iters = 1 << 12;
    k_ddiv<<<grid, threads>>>((double*)d_out, 16);
    cudaEventRecord(e0); k_ddiv<<<grid, threads>>>((double*)d_out, iters); cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double ops = (double)grid * threads * iters;
    printf("ddiv: %.1f Gop/s  %.2f /clk/SM\n", ops / ms / 1e6, ops / (ms * 1e-3) / nsm / (p.clockRate * 1e3));
  }
  cudaError_t err = cudaGetLastError();
  printf("err=%s\n", cudaGetErrorString(err));
  return 0;
}
