// Shared device helpers for the H²-ULV B200 kernels (sm_100a).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/h2ulv_b200.h"

namespace h2g {

// 8-byte asynchronous global->shared copy; src_bytes = 0 zero-fills.
__device__ __forceinline__ void cp_async8(void* smem, const void* gmem, bool valid) {
  unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  int n = valid ? 8 : 0;
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(s), "l"(gmem), "r"(n) : "memory");
}
// 16 bytes, L2 only (.cg): for data another CTA of the same launch published
__device__ __forceinline__ void cp_async16_cg(void* smem, const void* gmem) {
  unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory"); }

// D(8x8) += A(8x4, row) * B(4x8, col): FP64 tensor core (SASS DMMA.8x8x4).
__device__ __forceinline__ void dmma884(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c[0]), "+d"(c[1])
               : "d"(a), "d"(b));
}

// D(16x8) += A(16x16, row) * B(16x8, col): FP64 tensor core, 8x the work of m8n8k4 per instruction.
// Fragments (g = lane >> 2, t = lane & 3): a[i] = A[g + 8*(i&1)][t + 4*(i>>1)], b[i] = B[t + 4*i][g],
// c[0..1] = C[g][2t..2t+1], c[2..3] = C[g+8][2t..2t+1].
__device__ __forceinline__ void dmma16816(double (&c)[4], const double (&a)[8], const double (&b)[4]) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, "
      "{%12,%13,%14,%15}, {%0,%1,%2,%3};\n"
      : "+d"(c[0]), "+d"(c[1]), "+d"(c[2]), "+d"(c[3])
      : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]), "d"(b[0]),
        "d"(b[1]), "d"(b[2]), "d"(b[3]));
}

// Row of lower-triangular tile t (t = i(i+1)/2 + j, j <= i) without FP64 math.
__device__ __forceinline__ int tri_row(int t) {
  int i = (int)((sqrtf(8.0f * (float)t + 1.0f) - 1.0f) * 0.5f);
  while ((i + 1) * (i + 2) / 2 <= t) ++i;
  while (i * (i + 1) / 2 > t) --i;
  return i;
}

// Sign flip of a double on the integer pipe (keeps the FP64 pipe free for DMMA).
__device__ __forceinline__ double neg_int(double x) {
  return __longlong_as_double(__double_as_longlong(x) ^ (long long)0x8000000000000000ULL);
}

// Largest index p in [0, n) with starts[p] <= x (starts ascending).
__device__ __forceinline__ int upper_index(const int32_t* starts_strided, int stride_ints, int n, int x) {
  int lo = 0, hi = n - 1;
  while (lo < hi) {
    int mid = (lo + hi + 1) >> 1;
    if (starts_strided[(size_t)mid * stride_ints] <= x) lo = mid; else hi = mid - 1;
  }
  return lo;
}

}  // namespace h2g

int h2g_set_error(int code, const char* fmt, ...);
int h2g_check_launch(const char* what);
