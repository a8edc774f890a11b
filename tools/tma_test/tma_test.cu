// Standalone check of the TMA + mbarrier helpers of rd_internal.cuh on 3-D u8/u16 boxes.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cstdio>
#include <vector>
#include "../../paper_1310_1371_b200/csrc/rd_internal.cuh"
using namespace rd;

template <typename T>
__global__ void k(const __grid_constant__ CUtensorMap tmap, int bw, int bh, int x, int y, int z, T* out) {
  extern __shared__ __align__(128) unsigned char sm[];
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm);
  T* buf = reinterpret_cast<T*>(sm + 128);
  if (threadIdx.x == 0) { mbar_init(bar, 1); mbar_fence_init(); }
  __syncthreads();
  if (threadIdx.x == 0) {
    fence_proxy_async_smem();
    mbar_expect_tx(bar, bw * bh * sizeof(T));
    tma_load_3d(buf, &tmap, bar, x, y, z);
  }
  mbar_wait(bar, 0);
  for (int i = threadIdx.x; i < bw * bh; i += blockDim.x) out[i] = buf[i];
}

template <typename T>
int run(int W, int H, int N, int bw, int bh, int x, int y, int z) {
  PFN_cuTensorMapEncodeTiled_v12000 enc;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q);
  std::vector<T> h((size_t)W * H * N);
  for (size_t i = 0; i < h.size(); ++i) h[i] = (T)(i * 7 + 3);
  T *d, *o;
  cudaMalloc(&d, h.size() * sizeof(T));
  cudaMalloc(&o, bw * bh * sizeof(T));
  cudaMemcpy(d, h.data(), h.size() * sizeof(T), cudaMemcpyHostToDevice);
  CUtensorMap map;
  cuuint64_t dims[3] = {(cuuint64_t)W, (cuuint64_t)H, (cuuint64_t)N};
  cuuint64_t strides[2] = {(cuuint64_t)W * sizeof(T), (cuuint64_t)W * H * sizeof(T)};
  cuuint32_t box[3] = {(cuuint32_t)bw, (cuuint32_t)bh, 1}, es[3] = {1, 1, 1};
  CUresult r = enc(&map, sizeof(T) == 1 ? CU_TENSOR_MAP_DATA_TYPE_UINT8 : CU_TENSOR_MAP_DATA_TYPE_UINT16, 3, d, dims,
                   strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  size_t smem = 128 + bw * bh * sizeof(T) + 128;
  cudaFuncSetAttribute(k<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  k<T><<<1, 128, smem>>>(map, bw, bh, x, y, z, o);
  cudaError_t e = cudaDeviceSynchronize();
  std::vector<T> g(bw * bh);
  int bad = 0;
  if (e == cudaSuccess) {
    cudaMemcpy(g.data(), o, g.size() * sizeof(T), cudaMemcpyDeviceToHost);
    for (int j = 0; j < bh; ++j)
      for (int i = 0; i < bw; ++i) {
        int gx = x + i, gy = y + j;
        T exp = (gx < 0 || gy < 0 || gx >= W || gy >= H) ? 0 : h[((size_t)z * H + gy) * W + gx];
        bad += g[j * bw + i] != exp;
      }
  }
  printf("T=%zu W=%d H=%d box %dx%d at (%d,%d,%d): encode=%d kernel=%s bad=%d\n", sizeof(T), W, H, bw, bh, x, y, z, (int)r,
         cudaGetErrorString(e), bad);
  cudaFree(d);
  cudaFree(o);
  return e != cudaSuccess;
}

int main(int argc, char** argv) {
  int which = argc > 1 ? atoi(argv[1]) : 0;
  switch (which) {
    case 0: return run<uint16_t>(128, 128, 2, 48, 48, -8, -8, 0);
    case 1: return run<uint16_t>(128, 128, 2, 48, 48, -7, -7, 0);
    case 2: return run<uint8_t>(128, 128, 2, 48, 48, -8, -8, 0);
    case 3: return run<uint8_t>(128, 128, 2, 48, 48, 8, 8, 1);
    case 4: return run<uint16_t>(128, 128, 2, 48, 48, 9, 9, 1);
    case 5: return run<uint16_t>(128, 128, 2, 48, 46, 8, 8, 1);
  }
  return 0;
}
