// FP64 issue-rate microbenchmark for sm_100a: DMMA shapes vs DFMA.
// Each warp runs ITERS iterations of NACC independent MMA chains.
#include <cstdio>
#include <cuda_runtime.h>

#define ITERS 4096
#define NACC 8

__global__ void k_m8n8k4(double* out, double seed) {
  double a = seed + threadIdx.x, b = seed * 0.5;
  double c[NACC][2];
  for (int i = 0; i < NACC; i++) c[i][0] = c[i][1] = 0.0;
  for (int it = 0; it < ITERS; it++) {
#pragma unroll
    for (int i = 0; i < NACC; i++)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
  }
  double s = 0; for (int i = 0; i < NACC; i++) s += c[i][0] + c[i][1];
  if (s == 1.2345) out[0] = s;
}
__global__ void k_m16n8k4(double* out, double seed) {
  double a0 = seed + threadIdx.x, a1 = seed, b = seed * 0.5;
  double c[NACC][4];
  for (int i = 0; i < NACC; i++) c[i][0] = c[i][1] = c[i][2] = c[i][3] = 0.0;
  for (int it = 0; it < ITERS; it++) {
#pragma unroll
    for (int i = 0; i < NACC; i++)
      asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};"
                   : "+d"(c[i][0]), "+d"(c[i][1]), "+d"(c[i][2]), "+d"(c[i][3]) : "d"(a0), "d"(a1), "d"(b));
  }
  double s = 0; for (int i = 0; i < NACC; i++) s += c[i][0] + c[i][1] + c[i][2] + c[i][3];
  if (s == 1.2345) out[0] = s;
}
__global__ void k_m16n8k16(double* out, double seed) {
  double a[8], b[4];
  for (int i = 0; i < 8; i++) a[i] = seed + i + threadIdx.x;
  for (int i = 0; i < 4; i++) b[i] = seed * 0.5 + i;
  double c[NACC / 2][4];
  for (int i = 0; i < NACC / 2; i++) c[i][0] = c[i][1] = c[i][2] = c[i][3] = 0.0;
  for (int it = 0; it < ITERS; it++) {
#pragma unroll
    for (int i = 0; i < NACC / 2; i++)
      asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};"
                   : "+d"(c[i][0]), "+d"(c[i][1]), "+d"(c[i][2]), "+d"(c[i][3])
                   : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]),
                     "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
  }
  double s = 0; for (int i = 0; i < NACC / 2; i++) s += c[i][0] + c[i][1] + c[i][2] + c[i][3];
  if (s == 1.2345) out[0] = s;
}
__global__ void k_dfma(double* out, double seed) {
  double a = seed + threadIdx.x, b = seed * 0.999;
  double c[NACC];
  for (int i = 0; i < NACC; i++) c[i] = i;
  for (int it = 0; it < ITERS; it++) {
#pragma unroll
    for (int i = 0; i < NACC; i++) c[i] = fma(a, c[i], b);
  }
  double s = 0; for (int i = 0; i < NACC; i++) s += c[i];
  if (s == 1.2345) out[0] = s;
}

template <typename F>
void run(const char* name, F kern, double flops_per_warp_iter, int threads, int blocks_per_sm) {
  double* d; cudaMalloc(&d, 8);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int blocks = sms * blocks_per_sm;
  kern<<<blocks, threads>>>(d, 1.0);
  cudaDeviceSynchronize();
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  float best = 1e30f;
  for (int rep = 0; rep < 5; rep++) {
    cudaEventRecord(e0);
    kern<<<blocks, threads>>>(d, 1.0);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
  }
  double warps = (double)blocks * threads / 32;
  double flops = warps * ITERS * flops_per_warp_iter;
  printf("%-12s threads=%4d blk/sm=%d  %.3f ms  %.2f TFLOP/s\n", name, threads, blocks_per_sm, best, flops / best / 1e9);
  cudaFree(d);
}

int main() {
  cudaDeviceProp p; cudaGetDeviceProperties(&p, 0);
  printf("%s SMs=%d clock=%d kHz\n", p.name, p.multiProcessorCount, p.clockRate);
  for (int bps : {1, 2, 4}) {
    run("m8n8k4", k_m8n8k4, NACC * 2.0 * 8 * 8 * 4, 256, bps);
    run("m16n8k4", k_m16n8k4, NACC * 2.0 * 16 * 8 * 4, 256, bps);
    run("m16n8k16", k_m16n8k16, NACC / 2 * 2.0 * 16 * 8 * 16, 256, bps);
    run("dfma", k_dfma, NACC * 2.0 * 32, 256, bps);
  }
  return 0;
}
