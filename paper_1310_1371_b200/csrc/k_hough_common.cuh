// k_hough_common.cuh — small device helpers of the Hough kernel (k_hough2.cu): exact rounding
// of vote offsets, clamped shifts, shared-memory atomics and asynchronous copies.
#pragma once
#include "rd_internal.cuh"

namespace rd {
namespace hk {

// llround of an exactly computed product (|v| < 2^31): copysign(0.5) added toward zero,
// then truncated — the same two roundings as the oracle's llround (R9)
__device__ __forceinline__ int round_half_away_i(double v) {
  return __double2int_rz(__dadd_rz(v, copysign(0.5, v)));
}

// shared-memory atomic add on a 32-bit shared address: returns the old word
// shifts with PTX semantics: amounts >= 32 give 0
__device__ __forceinline__ uint32_t shl_clamp(uint32_t x, uint32_t n) {
  uint32_t r;
  asm("shl.b32 %0, %1, %2;" : "=r"(r) : "r"(x), "r"(n));
  return r;
}
__device__ __forceinline__ uint32_t shr_clamp(uint32_t x, uint32_t n) {
  uint32_t r;
  asm("shr.b32 %0, %1, %2;" : "=r"(r) : "r"(x), "r"(n));
  return r;
}
__device__ __forceinline__ uint32_t atom_add_shared(uint32_t saddr, uint32_t v) {
  uint32_t old;
  asm volatile("atom.shared.add.u32 %0, [%1], %2;" : "=r"(old) : "r"(saddr), "r"(v) : "memory");
  return old;
}

__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async4(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

__device__ __forceinline__ unsigned lanemask_lt() {
  unsigned m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

}  // namespace hk
}  // namespace rd
