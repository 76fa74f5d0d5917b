// Accuracy of rsqrt.approx.ftz.f64 (MUFU.RSQ64H) and of one quadratic / cubic correction, against 1/sqrt in double
// (max relative error over 2^24 arguments spread over 40 binades).  Decides the flux's rsqrt polynomial (K1_FASTMATH).
#include <cmath>
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k(double *err) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const double x = exp2(-20.0 + 40.0 * ((double)i / (double)(gridDim.x * blockDim.x)));
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  const double ref = 1.0 / sqrt(x);
  const double e = fma(-x, y * y, 1.0);
  const double q = fma(0.5 * y, e, y);                        // one Newton step (quadratic)
  const double c = fma(y * e, fma(0.375, e, 0.5), y);         // the cubic correction in use
  err[3 * i + 0] = fabs(y - ref) / ref;
  err[3 * i + 1] = fabs(q - ref) / ref;
  err[3 * i + 2] = fabs(c - ref) / ref;
}

int main() {
  const int n = 1 << 24;
  double *d, *h = new double[3 * (size_t)n];
  cudaMalloc(&d, sizeof(double) * 3 * (size_t)n);
  k<<<n / 256, 256>>>(d);
  cudaMemcpy(h, d, sizeof(double) * 3 * (size_t)n, cudaMemcpyDeviceToHost);
  double m[3] = {0, 0, 0};
  for (size_t i = 0; i < (size_t)n; i++)
    for (int j = 0; j < 3; j++) m[j] = fmax(m[j], h[3 * i + j]);
  printf("max rel err: MUFU.RSQ64H %.3e (2^%.1f), + Newton %.3e, + cubic %.3e\n", m[0], log2(m[0]), m[1], m[2]);
  return 0;
}
