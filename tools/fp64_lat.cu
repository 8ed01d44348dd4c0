// FP64 latency / issue microbenchmarks on B200 (sm_100a), one CTA on one SM, clock64 timing.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_lat fp64_lat.cu
// Prints one JSON line: cycles per op for dependent chains and for k independent chains per
// warp with w warps per CTA (w/4 warps per SM sub-partition).
#include <cstdio>
#include <cuda_runtime.h>

#define N 2048

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}

template <int K>
__global__ void k_dfma_chains(double* out, long long* cyc, double a, double b) {
  double x[K];
#pragma unroll
  for (int i = 0; i < K; i++) x[i] = threadIdx.x * 1e-3 + i;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < N; it++) {
#pragma unroll
    for (int i = 0; i < K; i++) x[i] = fma(x[i], a, b);
  }
  long long t1 = clock64();
  double s = 0;
#pragma unroll
  for (int i = 0; i < K; i++) s += x[i];
  if (s == 12345.678) out[threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}

template <int K>
__global__ void k_dmma_chains(double* out, long long* cyc, double a, double b) {
  double acc[2 * K];
#pragma unroll
  for (int i = 0; i < 2 * K; i++) acc[i] = 0;
  double av = a + threadIdx.x * 1e-9, bv = b;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < N; it++) {
#pragma unroll
    for (int i = 0; i < K; i++) dmma(acc[2 * i], acc[2 * i + 1], av, bv);
  }
  long long t1 = clock64();
  double s = 0;
#pragma unroll
  for (int i = 0; i < 2 * K; i++) s += acc[i];
  if (s == 12345.678) out[threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}

// DMMA result feeding the next DMMA's A operand (the fused kernel's C -> A hand-off)
__global__ void k_dmma_feed(double* out, long long* cyc, double a, double b) {
  double d0 = a, d1 = b;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < N; it++) {
    double e0 = 0, e1 = 0;
    dmma(e0, e1, d0, b);
    d0 = e0 * 1e-3;
    d1 = e1;
  }
  long long t1 = clock64();
  if (d0 + d1 == 12345.678) out[threadIdx.x] = d0;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}

__global__ void k_lds_chain(double* out, long long* cyc) {
  __shared__ int idx[1024];
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) idx[i] = (i + 1) & 1023;
  __syncthreads();
  int p = threadIdx.x & 7;
  long long t0 = clock64();
  for (int it = 0; it < N; it++) p = idx[p];
  long long t1 = clock64();
  if (p == 12345) out[threadIdx.x] = p;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}

__global__ void k_rsq_chain(double* out, long long* cyc, double a) {
  double x = a + threadIdx.x;
  long long t0 = clock64();
  for (int it = 0; it < N; it++) {
    double y;
    asm volatile("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
    x = y + 1.0;
  }
  long long t1 = clock64();
  if (x == 12345.678) out[threadIdx.x] = x;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}

__global__ void k_sqrt_chain(double* out, long long* cyc, double a) {
  double x = a + threadIdx.x;
  long long t0 = clock64();
  for (int it = 0; it < N; it++) x = sqrt(x) + 2.0;
  long long t1 = clock64();
  if (x == 12345.678) out[threadIdx.x] = x;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}

__global__ void k_div_chain(double* out, long long* cyc, double a) {
  double x = a + threadIdx.x;
  long long t0 = clock64();
  for (int it = 0; it < N; it++) x = 3.0 / x + 1.0;
  long long t1 = clock64();
  if (x == 12345.678) out[threadIdx.x] = x;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}

__global__ void k_bar(double* out, long long* cyc) {
  long long t0 = clock64();
  for (int it = 0; it < N; it++) __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}

// fixed-latency integer chain for reference
__global__ void k_imad_chain(double* out, long long* cyc, int a) {
  int x = threadIdx.x;
  long long t0 = clock64();
  for (int it = 0; it < N; it++) x = x * a + 7;
  long long t1 = clock64();
  if (x == 12345) out[threadIdx.x] = x;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}

template <typename F>
double run(F launch, long long* dcyc) {
  launch();
  cudaDeviceSynchronize();
  launch();
  long long c = 0;
  cudaMemcpy(&c, dcyc, sizeof(c), cudaMemcpyDeviceToHost);
  return (double)c / N;
}

int main() {
  double* out;
  long long* cyc;
  cudaMalloc(&out, 1024 * sizeof(double));
  cudaMalloc(&cyc, sizeof(long long));
  printf("{");
  const int ws[] = {1, 4, 8, 16};
  for (int w : ws) {
    int t = 32 * w;
    printf("\"dfma_k1_w%d\": %.2f, ", w, run([&] { k_dfma_chains<1><<<1, t>>>(out, cyc, 1.0000001, 1e-9); }, cyc));
    printf("\"dfma_k4_w%d\": %.2f, ", w, run([&] { k_dfma_chains<4><<<1, t>>>(out, cyc, 1.0000001, 1e-9); }, cyc) / 4);
    printf("\"dfma_k8_w%d\": %.2f, ", w, run([&] { k_dfma_chains<8><<<1, t>>>(out, cyc, 1.0000001, 1e-9); }, cyc) / 8);
    printf("\"dmma_k1_w%d\": %.2f, ", w, run([&] { k_dmma_chains<1><<<1, t>>>(out, cyc, 1e-3, 1e-3); }, cyc));
    printf("\"dmma_k2_w%d\": %.2f, ", w, run([&] { k_dmma_chains<2><<<1, t>>>(out, cyc, 1e-3, 1e-3); }, cyc) / 2);
    printf("\"dmma_k4_w%d\": %.2f, ", w, run([&] { k_dmma_chains<4><<<1, t>>>(out, cyc, 1e-3, 1e-3); }, cyc) / 4);
    printf("\"dmma_k8_w%d\": %.2f, ", w, run([&] { k_dmma_chains<8><<<1, t>>>(out, cyc, 1e-3, 1e-3); }, cyc) / 8);
  }
  printf("\"dmma_feed_w1\": %.2f, ", run([&] { k_dmma_feed<<<1, 32>>>(out, cyc, 1e-3, 1e-3); }, cyc));
  printf("\"lds_chain\": %.2f, ", run([&] { k_lds_chain<<<1, 32>>>(out, cyc); }, cyc));
  printf("\"rsq64h_chain\": %.2f, ", run([&] { k_rsq_chain<<<1, 32>>>(out, cyc, 2.0); }, cyc));
  printf("\"dsqrt_chain\": %.2f, ", run([&] { k_sqrt_chain<<<1, 32>>>(out, cyc, 2.0); }, cyc));
  printf("\"ddiv_chain\": %.2f, ", run([&] { k_div_chain<<<1, 32>>>(out, cyc, 2.0); }, cyc));
  printf("\"imad_chain\": %.2f, ", run([&] { k_imad_chain<<<1, 32>>>(out, cyc, 3); }, cyc));
  printf("\"bar_256\": %.2f, ", run([&] { k_bar<<<1, 256>>>(out, cyc); }, cyc));
  printf("\"bar_1024\": %.2f", run([&] { k_bar<<<1, 1024>>>(out, cyc); }, cyc));
  printf("}\n");
  return 0;
}
