// Latency microbenchmark on sm_100a: cycles per dependent DFMA / DMUL / MUFU.RSQ64H+correction, one warp, and the
// throughput of DFMA per SMSP with 1, 2, 4, 8 independent chains per warp (1 warp and 2 warps per SMSP).
// Used to read K1's "wait" stalls.
#include <cstdio>
#include <cuda_runtime.h>

template <int CH>
__global__ void k_chain(double *out, long long *cyc, int iters) {
  double a[CH];
#pragma unroll
  for (int c = 0; c < CH; c++) a[c] = threadIdx.x * 1e-3 + c;
  const double b = 0.999999, d = 1e-9;
  __syncwarp();
  long long t0 = clock64();
  for (int i = 0; i < iters; i++) {
#pragma unroll
    for (int k = 0; k < 16; k++)
#pragma unroll
      for (int c = 0; c < CH; c++) a[c] = fma(a[c], b, d);
  }
  long long t1 = clock64();
  double s = 0;
#pragma unroll
  for (int c = 0; c < CH; c++) s += a[c];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

__global__ void k_rsq(double *out, long long *cyc, int iters) {
  double x = 1.0 + threadIdx.x * 1e-3;
  long long t0 = clock64();
  for (int i = 0; i < iters; i++) {
#pragma unroll
    for (int k = 0; k < 16; k++) {
      double y;
      asm volatile("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
      x = y + 1.0;
    }
  }
  long long t1 = clock64();
  out[threadIdx.x] = x;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}

template <int CH>
void run(const char *name, int warps_per_block, double *d, long long *c) {
  const int iters = 4096;
  k_chain<CH><<<1, 32 * warps_per_block>>>(d, c, iters);
  cudaDeviceSynchronize();
  long long cyc;
  cudaMemcpy(&cyc, c, sizeof(cyc), cudaMemcpyDeviceToHost);
  const double ops = (double)iters * 16 * CH;  // dependent-chain ops per thread
  printf("%-28s warps/block %2d: %.2f cycles per op per warp (chain length view: %.2f cycles per dependent op)\n", name,
         warps_per_block, (double)cyc / ops, (double)cyc / (iters * 16.0));
}

int main() {
  double *d;
  long long *c;
  cudaMalloc(&d, 1 << 20);
  cudaMalloc(&c, 1 << 16);
  run<1>("DFMA 1 chain", 1, d, c);
  run<2>("DFMA 2 chains", 1, d, c);
  run<4>("DFMA 4 chains", 1, d, c);
  run<8>("DFMA 8 chains", 1, d, c);
  run<16>("DFMA 16 chains", 1, d, c);
  run<1>("DFMA 1 chain", 4, d, c);
  run<4>("DFMA 4 chains", 4, d, c);
  run<8>("DFMA 8 chains", 8, d, c);
  k_rsq<<<1, 32>>>(d, c, 4096);
  cudaDeviceSynchronize();
  long long cyc;
  cudaMemcpy(&cyc, c, sizeof(cyc), cudaMemcpyDeviceToHost);
  printf("MUFU.RSQ64H + DADD dependent: %.2f cycles per step\n", (double)cyc / (4096.0 * 16));
  return 0;
}
