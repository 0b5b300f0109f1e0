// Dependent-chain latencies of FP64 ops and shuffles on one warp (dev tool).
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(double* out, long long* cyc, double a, double b) {
  double x = a, y = b;
  long long t0, t1;
  const int N = 512;
  t0 = clock64();
#pragma unroll 16
  for (int i = 0; i < N; ++i) x = fma(x, y, a);
  t1 = clock64(); cyc[0] = (t1 - t0) / N;
  t0 = clock64();
#pragma unroll 16
  for (int i = 0; i < N; ++i) x = x + y;
  t1 = clock64(); cyc[1] = (t1 - t0) / N;
  t0 = clock64();
#pragma unroll 16
  for (int i = 0; i < N; ++i) x = __shfl_xor_sync(0xffffffffu, x, 1) ;
  t1 = clock64(); cyc[2] = (t1 - t0) / N;
  t0 = clock64();
#pragma unroll 4
  for (int i = 0; i < N; ++i) x = a / x;
  t1 = clock64(); cyc[3] = (t1 - t0) / N;
  t0 = clock64();
#pragma unroll 4
  for (int i = 0; i < N; ++i) x = sqrt(x + a);
  t1 = clock64(); cyc[4] = (t1 - t0) / N;
  float f = float(x);
  t0 = clock64();
#pragma unroll 16
  for (int i = 0; i < N; ++i) f = fmaf(f, float(b), float(a));
  t1 = clock64(); cyc[5] = (t1 - t0) / N;
  out[threadIdx.x] = x + f;
}
int main() {
  double* o; long long* c; cudaMalloc(&o, 256); cudaMalloc(&c, 64);
  k<<<1, 32>>>(o, c, 0.5, 0.999);
  k<<<1, 32>>>(o, c, 0.5, 0.999);
  long long h[6]; cudaMemcpy(h, c, 48, cudaMemcpyDeviceToHost);
  printf("latency cycles: DFMA %lld DADD %lld SHFL(f64) %lld DDIV %lld DSQRT %lld FFMA %lld\n", h[0], h[1], h[2], h[3], h[4], h[5]);
}
