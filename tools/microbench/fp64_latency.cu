// Dependent-chain latency (cycles) of FP64 ops and barrier cost on sm_100a.
#include <cstdio>
__global__ void lat(double* out, long long* cyc, double x0, int n) {
  double x = x0 + threadIdx.x * 1e-9;
  long long t0, t1;
  // DFMA chain
  t0 = clock64();
  for (int i = 0; i < n; ++i) x = fma(x, 0.9999999, 1e-7);
  t1 = clock64(); if (threadIdx.x == 0) cyc[0] = (t1 - t0);
  // DMUL chain
  t0 = clock64();
  for (int i = 0; i < n; ++i) x = x * 1.0000001;
  t1 = clock64(); if (threadIdx.x == 0) cyc[1] = (t1 - t0);
  // DIV chain
  t0 = clock64();
  for (int i = 0; i < n; ++i) x = 1.0 / (x + 1.0);
  t1 = clock64(); if (threadIdx.x == 0) cyc[2] = (t1 - t0);
  // SQRT chain
  t0 = clock64();
  for (int i = 0; i < n; ++i) x = sqrt(x + 1.0);
  t1 = clock64(); if (threadIdx.x == 0) cyc[3] = (t1 - t0);
  // barrier
  t0 = clock64();
  for (int i = 0; i < n; ++i) __syncthreads();
  t1 = clock64(); if (threadIdx.x == 0) cyc[4] = (t1 - t0);
  // FFMA chain (reference)
  float f = (float)x;
  t0 = clock64();
  for (int i = 0; i < n; ++i) f = fmaf(f, 0.9999f, 1e-4f);
  t1 = clock64(); if (threadIdx.x == 0) cyc[5] = (t1 - t0);
  // smem round trip chain
  __shared__ double sm[256];
  sm[threadIdx.x] = x;
  __syncthreads();
  int idx = threadIdx.x;
  t0 = clock64();
  for (int i = 0; i < n; ++i) { double y = sm[idx]; idx = (int)(y * 0.0) + ((idx + 1) & 255); }
  t1 = clock64(); if (threadIdx.x == 0) cyc[6] = (t1 - t0);
  out[threadIdx.x] = x + f + idx;
}
int main() {
  double* out; long long* cyc; cudaMalloc(&out, 4096); cudaMallocManaged(&cyc, 64 * 8);
  int n = 1000;
  for (int threads : {32, 160, 256}) {
    lat<<<1, threads>>>(out, cyc, 1.0, n); cudaDeviceSynchronize();
    lat<<<1, threads>>>(out, cyc, 1.0, n); cudaDeviceSynchronize();
    printf("threads %d: DFMA %.1f  DMUL %.1f  DDIV %.1f  DSQRT %.1f  BAR %.1f  FFMA %.1f  LDS-chain %.1f cycles/op\n", threads,
           cyc[0] / (double)n, cyc[1] / (double)n, cyc[2] / (double)n, cyc[3] / (double)n, cyc[4] / (double)n, cyc[5] / (double)n, cyc[6] / (double)n);
  }
  return 0;
}
