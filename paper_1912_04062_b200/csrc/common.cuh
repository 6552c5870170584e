// common.cuh -- shared device helpers for the sm_100a FP64 path (CUDA side only;
// nothing here is shared with the CPU reference checker).
#pragma once
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>

#define SK_IDX(i, j, ld) ((size_t)(i) + (size_t)(j) * (size_t)(ld))

namespace sk {

template <class T>
__host__ __device__ __forceinline__ T smin(T a, T b) { return a < b ? a : b; }
template <class T>
__host__ __device__ __forceinline__ T smax(T a, T b) { return a > b ? a : b; }

// ---- FP64 tensor-core tile op. On sm_100a every mma.sync .f64 shape lowers to
// SASS DMMA.8x8x4 (checked with cuobjdump); we issue m8n8k4 directly.
//   A fragment (8x4 row):  a = A[g][t]      g = lane>>2, t = lane&3
//   B fragment (4x8 col):  b = B[t][g]
//   C fragment (8x8):      c0 = C[g][2t], c1 = C[g][2t+1]
__device__ __forceinline__ void dmma884(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
}

// ---- cp.async (LDGSTS) 16-byte global->shared copy with zero-fill of the tail
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, int src_bytes) {
  unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" :: "r"(s), "l"(gmem), "r"(src_bytes));
}
__device__ __forceinline__ void cp_async8(void* smem, const void* gmem, int src_bytes) {
  unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" :: "r"(s), "l"(gmem), "r"(src_bytes));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" :: "n"(N)); }

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

}  // namespace sk
