// FP64 throughput microbenchmark on sm_100a: DFMA (CUDA cores), DMMA
// (mma.sync m8n8k4 f64, tensor cores) and both concurrently in one kernel.
// Used to decide whether the DG contractions (Ic, Pr, Ps, Lg) should move to
// the FP64 tensor path.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_dfma(double *out, int iters) {
  double a0 = threadIdx.x * 1e-3, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, a4 = a0 + 4, a5 = a0 + 5, a6 = a0 + 6,
         a7 = a0 + 7;
  const double b = 0.999999, c = 1e-9;
  for (int i = 0; i < iters; i++) {
#pragma unroll
    for (int k = 0; k < 8; k++) {
      a0 = fma(a0, b, c); a1 = fma(a1, b, c); a2 = fma(a2, b, c); a3 = fma(a3, b, c);
      a4 = fma(a4, b, c); a5 = fma(a5, b, c); a6 = fma(a6, b, c); a7 = fma(a7, b, c);
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
}

__device__ __forceinline__ void dmma(double &d0, double &d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

__global__ void k_dmma(double *out, int iters) {
  double a = 1e-3 * (threadIdx.x & 31), b = 0.5;
  double d[8][2];
#pragma unroll
  for (int j = 0; j < 8; j++) d[j][0] = d[j][1] = 0.0;
  for (int i = 0; i < iters; i++) {
#pragma unroll
    for (int k = 0; k < 8; k++)
#pragma unroll
      for (int j = 0; j < 8; j++) dmma(d[j][0], d[j][1], a, b);
  }
  double s = 0;
#pragma unroll
  for (int j = 0; j < 8; j++) s += d[j][0] + d[j][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

// even warps DFMA, odd warps DMMA
__global__ void k_mixed(double *out, int iters_f, int iters_m) {
  int w = threadIdx.x >> 5;
  if (w & 1) {
    double a = 1e-3 * (threadIdx.x & 31), b = 0.5;
    double d[8][2];
#pragma unroll
    for (int j = 0; j < 8; j++) d[j][0] = d[j][1] = 0.0;
    for (int i = 0; i < iters_m; i++)
#pragma unroll
      for (int k = 0; k < 8; k++)
#pragma unroll
        for (int j = 0; j < 8; j++) dmma(d[j][0], d[j][1], a, b);
    double s = 0;
#pragma unroll
    for (int j = 0; j < 8; j++) s += d[j][0] + d[j][1];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  } else {
    double a0 = threadIdx.x * 1e-3, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, a4 = a0 + 4, a5 = a0 + 5, a6 = a0 + 6,
           a7 = a0 + 7;
    const double b = 0.999999, c = 1e-9;
    for (int i = 0; i < iters_f; i++)
#pragma unroll
      for (int k = 0; k < 8; k++) {
        a0 = fma(a0, b, c); a1 = fma(a1, b, c); a2 = fma(a2, b, c); a3 = fma(a3, b, c);
        a4 = fma(a4, b, c); a5 = fma(a5, b, c); a6 = fma(a6, b, c); a7 = fma(a7, b, c);
      }
    out[blockIdx.x * blockDim.x + threadIdx.x] = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
  }
}

int main() {
  int nsm = 0;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  const int blocks = nsm * 4, threads = 256;
  double *out;
  cudaMalloc(&out, sizeof(double) * blocks * threads);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float ms;
  const int it = 4096;
  k_dfma<<<blocks, threads>>>(out, 16);
  cudaEventRecord(e0);
  k_dfma<<<blocks, threads>>>(out, it);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  cudaEventElapsedTime(&ms, e0, e1);
  double fl = 2.0 * 64.0 * it * blocks * threads;
  printf("DFMA: %.2f TFLOP/s (%.3f ms)\n", fl / ms / 1e9, ms);
  k_dmma<<<blocks, threads>>>(out, 16);
  cudaEventRecord(e0);
  k_dmma<<<blocks, threads>>>(out, it / 8);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  cudaEventElapsedTime(&ms, e0, e1);
  double flm = 2.0 * 256.0 * 64.0 * (it / 8) * blocks * (threads / 32);
  printf("DMMA m8n8k4: %.2f TFLOP/s (%.3f ms)\n", flm / ms / 1e9, ms);
  cudaEventRecord(e0);
  k_mixed<<<blocks, threads>>>(out, it, it / 8);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  cudaEventElapsedTime(&ms, e0, e1);
  double fmix = fl / 2 + flm / 2;
  printf("mixed (half warps each): %.2f TFLOP/s combined (%.3f ms)\n", fmix / ms / 1e9, ms);
  cudaError_t err = cudaGetLastError();
  printf("status: %s\n", cudaGetErrorString(err));
  return 0;
}
