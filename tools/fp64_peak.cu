// FP64 roofline calibration for B200 (sm_100a): DFMA-only, DMMA.8x8x4-only and mixed loops.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_peak fp64_peak.cu
// Prints one JSON line with TFLOP/s per mode (2 flops per FMA) and the sm clock seen by NVML is sampled
// separately by the caller.
#include <cstdio>
#include <cuda_runtime.h>

#define ITERS 4096

__global__ void k_dfma(double* out, double a, double b) {
  double x[16];
#pragma unroll
  for (int i = 0; i < 16; i++) x[i] = threadIdx.x * 1e-3 + i;
  for (int it = 0; it < ITERS; it++) {
#pragma unroll
    for (int i = 0; i < 16; i++) x[i] = fma(x[i], a, b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 16; i++) s += x[i];
  if (s == 12345.678) out[threadIdx.x] = s;
}

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}

__global__ void k_dmma(double* out, double a, double b) {
  double acc[16];
#pragma unroll
  for (int i = 0; i < 16; i++) acc[i] = 0;
  double av = a + threadIdx.x * 1e-9, bv = b;
  for (int it = 0; it < ITERS; it++) {
#pragma unroll
    for (int i = 0; i < 8; i++) dmma(acc[2 * i], acc[2 * i + 1], av, bv);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 16; i++) s += acc[i];
  if (s == 12345.678) out[threadIdx.x] = s;
}

// mixed: per iteration 8 DMMA (2048 FMA per warp) + 16 DFMA per lane (512 FMA per warp)
template <int nf>
__global__ void k_mixed(double* out, double a, double b) {
  double acc[16];
  double x[16];
#pragma unroll
  for (int i = 0; i < 16; i++) { acc[i] = 0; x[i] = threadIdx.x * 1e-3 + i; }
  double av = a + threadIdx.x * 1e-9, bv = b;
  for (int it = 0; it < ITERS; it++) {
#pragma unroll
    for (int i = 0; i < 8; i++) dmma(acc[2 * i], acc[2 * i + 1], av, bv);
#pragma unroll
    for (int i = 0; i < nf; i++) x[i] = fma(x[i], a, b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 16; i++) s += acc[i] + x[i];
  if (s == 12345.678) out[threadIdx.x] = s;
}

// per 8 iterations: 8 DMMA + 2 exp(-sqrt(x)) per lane (the Matern inner loop shape)
__global__ void k_exp(double* out, double a, double b) {
  double acc[16];
#pragma unroll
  for (int i = 0; i < 16; i++) acc[i] = 0;
  double av = a + threadIdx.x * 1e-9, bv = b;
  double e0 = 0, e1 = 0, z = threadIdx.x * 1e-4;
  for (int it = 0; it < ITERS / 8; it++) {
#pragma unroll
    for (int i = 0; i < 8; i++) dmma(acc[2 * i], acc[2 * i + 1], av, bv);
    e0 += exp(-sqrt(z + it * 1e-6));
    e1 += exp(-sqrt(z + it * 2e-6));
  }
  double s = e0 + e1;
#pragma unroll
  for (int i = 0; i < 16; i++) s += acc[i];
  if (s == 12345.678) out[threadIdx.x] = s;
}

int main() {
  int dev = 0; cudaDeviceProp p; cudaGetDeviceProperties(&p, dev);
  double* out; cudaMalloc(&out, 4096 * sizeof(double));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int threads = 256;
  int blocks_list[3] = {p.multiProcessorCount * 4, p.multiProcessorCount * 8, p.multiProcessorCount * 16};
  printf("{\"sms\": %d, \"results\": [", p.multiProcessorCount);
  bool first = true;
  for (int mode = 0; mode < 6; mode++) {
    for (int bi = 0; bi < 3; bi++) {
      int blocks = blocks_list[bi];
      float best = 1e30f;
      for (int rep = 0; rep < 5; rep++) {
        cudaEventRecord(e0);
        if (mode == 0) k_dfma<<<blocks, threads>>>(out, 0.999999, 1e-7);
        else if (mode == 1) k_dmma<<<blocks, threads>>>(out, 0.999999, 1e-7);
        else if (mode == 2) k_mixed<4><<<blocks, threads>>>(out, 0.999999, 1e-7);
        else if (mode == 3) k_mixed<8><<<blocks, threads>>>(out, 0.999999, 1e-7);
        else if (mode == 4) k_mixed<16><<<blocks, threads>>>(out, 0.999999, 1e-7);
        else k_exp<<<blocks, threads>>>(out, 0.999999, 1e-7);
        cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
      }
      double warps = (double)blocks * threads / 32.0;
      double fma_per_warp;
      if (mode == 0) fma_per_warp = (double)ITERS * 16 * 32;
      else if (mode == 1) fma_per_warp = (double)ITERS * 8 * 256;
      else if (mode < 5) fma_per_warp = (double)ITERS * (8 * 256 + (mode == 2 ? 4 : (mode == 3 ? 8 : 16)) * 32);
      else fma_per_warp = (double)ITERS / 8 * (8 * 256);  // exp mode: DMMA flops only
      double tflops = warps * fma_per_warp * 2.0 / (best * 1e-3) / 1e12;
      const char* name = mode == 0 ? "dfma" : mode == 1 ? "dmma" : mode == 2 ? "mixed_dmma8_dfma4" : mode == 3 ? "mixed_dmma8_dfma8" : mode == 4 ? "mixed_dmma8_dfma16" : "dmma8_plus_2exp_sqrt";
      printf("%s{\"mode\": \"%s\", \"blocks\": %d, \"ms\": %.4f, \"tflops\": %.3f}", first ? "" : ", ", name, blocks, best, tflops);
      first = false;
    }
  }
  printf("]}\n");
  cudaError_t err = cudaGetLastError();
  if (err != cudaSuccess) { fprintf(stderr, "CUDA error %s\n", cudaGetErrorString(err)); return 1; }
  return 0;
}
