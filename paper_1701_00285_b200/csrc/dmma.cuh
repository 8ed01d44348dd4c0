// FP64 tensor-core primitives for sm_100a.  tcgen05 has no f64 kind; ptxas lowers
// mma.sync.m8n8k4 .f64 to DMMA.8x8x4 (SURVEY [M10]).  Fragment layout (lane = 0..31):
//   A (8x4, row):  a  = A[lane/4][lane%4]
//   B (4x8, col):  b  = B[lane%4][lane/4]
//   C/D (8x8):     c0 = C[lane/4][2*(lane%4)], c1 = C[lane/4][2*(lane%4)+1]
#pragma once
#include <cuda_runtime.h>

namespace mlk {

__device__ __forceinline__ void dmma_8x8x4(double& d0, double& d1, double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

__device__ __forceinline__ void cp_async8(void* smem, const void* gmem, bool pred) {
  unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  int sz = pred ? 8 : 0;
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(s), "l"(gmem), "r"(sz));
}

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, bool pred) {
  unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  int sz = pred ? 16 : 0;
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "r"(sz));
}

__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }

template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

}  // namespace mlk
