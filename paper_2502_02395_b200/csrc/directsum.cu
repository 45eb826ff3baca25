// Direct-sum product with the EXACT kernel matrix, never formed:
// y = A x with A_ij = K(|p_i - p_j|) (i != j), A_ii = shift — the dense
// operator of oracle.dense_assemble / kernels.gen_block (oracle.py:34-40,
// kernels.py:46-64) at sizes where N^2 entries do not fit anywhere
// (‖A_exact x − b‖ at 1M-8M, iterative refinement).
//
// FP64-pipe bound (no reuse to put on tensor cores: every entry is used
// once per right-hand side): one thread per target row, the sources staged
// in shared memory 256 at a time, the source range split across blockIdx.y
// so small N still fills 148 SMs.  The partial sums land in a workspace and
// a second kernel adds them in split order, so the result is deterministic.
// 1/r is rsqrt (≤ 1 ulp), not the correctly rounded division of the
// kernel-block generator: the sum order differs from a dense GEMV anyway.
#include <algorithm>

#include "common.cuh"

namespace h2g {

constexpr int DS_THREADS = 256;

template <int R, int F>
__global__ void __launch_bounds__(DS_THREADS) direct_matvec_kernel(const double* __restrict__ pts,
                                                                   const double* __restrict__ x, int ldx,
                                                                   double* __restrict__ work, long long n,
                                                                   long long chunk, double decay,
                                                                   long long* __restrict__ coincident) {
  __shared__ double sp[3][DS_THREADS];
  __shared__ double sx[R][DS_THREADS];
  const long long i = (long long)blockIdx.x * DS_THREADS + threadIdx.x;
  const long long j0 = (long long)blockIdx.y * chunk;
  const long long j1 = min(n, j0 + chunk);
  double xi = 0.0, yi = 0.0, zi = 0.0;
  if (i < n) xi = pts[3 * i], yi = pts[3 * i + 1], zi = pts[3 * i + 2];
  double acc[R];
#pragma unroll
  for (int r = 0; r < R; ++r) acc[r] = 0.0;
  int zeros = 0;
  for (long long t0 = j0; t0 < j1; t0 += DS_THREADS) {
    const long long j = t0 + threadIdx.x;
    __syncthreads();
    if (j < j1) {
      sp[0][threadIdx.x] = pts[3 * j];
      sp[1][threadIdx.x] = pts[3 * j + 1];
      sp[2][threadIdx.x] = pts[3 * j + 2];
#pragma unroll
      for (int r = 0; r < R; ++r) sx[r][threadIdx.x] = x[j * ldx + r];
    } else {  // far away, zero weight: contributes exactly 0
      sp[0][threadIdx.x] = sp[1][threadIdx.x] = sp[2][threadIdx.x] = 1.0e100;
#pragma unroll
      for (int r = 0; r < R; ++r) sx[r][threadIdx.x] = 0.0;
    }
    __syncthreads();
#pragma unroll 4
    for (int q = 0; q < DS_THREADS; ++q) {
      const double dx = xi - sp[0][q], dy = yi - sp[1][q], dz = zi - sp[2][q];
      const double s = fma(dz, dz, fma(dy, dy, dx * dx));
      const bool z = !(s > 0.0);   // the diagonal (or a coincident pair): added / flagged below
      zeros += z;
      double v;
      if (F == 2) {
        v = z ? 0.0 : exp(-s * decay);
      } else {
        const double inv = z ? 0.0 : rsqrt(s);
        v = F == 0 ? inv : exp(-decay * (s * inv)) * inv;
      }
#pragma unroll
      for (int r = 0; r < R; ++r) acc[r] = fma(v, sx[r][q], acc[r]);
    }
  }
  if (i >= n) return;
  // the target itself is the one expected zero distance inside its own source range
  const int expected = (i >= j0 && i < j1) ? 1 : 0;
  if (zeros > expected) atomicExch((unsigned long long*)coincident, 1ULL);
  double* w = work + ((long long)blockIdx.y * n + i) * R;
#pragma unroll
  for (int r = 0; r < R; ++r) w[r] = acc[r];
}

template <int R>
__global__ void __launch_bounds__(DS_THREADS) direct_reduce_kernel(const double* __restrict__ work, int nsplit,
                                                                   const double* __restrict__ x, int ldx,
                                                                   double* __restrict__ y, int ldy, long long n,
                                                                   double shift) {
  const long long i = (long long)blockIdx.x * DS_THREADS + threadIdx.x;
  if (i >= n) return;
#pragma unroll
  for (int r = 0; r < R; ++r) {
    double s = 0.0;
    for (int k = 0; k < nsplit; ++k) s += work[((long long)k * n + i) * R + r];
    y[i * ldy + r] = fma(shift, x[i * ldx + r], s);
  }
}

// source-range splits for the current device: >= 8 CTAs per SM in total
static int direct_splits(long long n) {
  int dev = 0, sms = 148;
  if (cudaGetDevice(&dev) != cudaSuccess || cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess)
    sms = 148;
  const long long rows = (n + DS_THREADS - 1) / DS_THREADS;
  const long long want = 8LL * sms;
  long long s = (want + rows - 1) / rows;
  s = std::min(s, rows);
  return (int)std::max(1LL, std::min(s, 64LL));
}

template <int R>
static void launch(const double* pts, const double* x, int ldx, double* y, int ldy, long long n, int nsplit,
                   int family, double shift, double decay, double* work, long long* flag, cudaStream_t st) {
  const long long rows = (n + DS_THREADS - 1) / DS_THREADS;
  long long chunk = (n + nsplit - 1) / nsplit;
  chunk = (chunk + DS_THREADS - 1) / DS_THREADS * DS_THREADS;
  const dim3 grid((unsigned)rows, (unsigned)nsplit);
  if (family == 0)
    direct_matvec_kernel<R, 0><<<grid, DS_THREADS, 0, st>>>(pts, x, ldx, work, n, chunk, decay, flag);
  else if (family == 1)
    direct_matvec_kernel<R, 1><<<grid, DS_THREADS, 0, st>>>(pts, x, ldx, work, n, chunk, decay, flag);
  else
    direct_matvec_kernel<R, 2><<<grid, DS_THREADS, 0, st>>>(pts, x, ldx, work, n, chunk, decay, flag);
  direct_reduce_kernel<R><<<(unsigned)rows, DS_THREADS, 0, st>>>(work, nsplit, x, ldx, y, ldy, n, shift);
}

}  // namespace h2g

extern "C" int64_t h2g_direct_matvec_workspace(int64_t n) {
  if (n <= 0) return 0;
  return (int64_t)h2g::direct_splits(n) * n * 4;
}

extern "C" int h2g_direct_matvec(const double* d_points, const double* d_x, double* d_y, int64_t n, int nrhs,
                                 int family, double shift, double decay, double* d_work, int64_t work_elems,
                                 int64_t* d_coincident, void* stream) {
  if (n <= 0 || nrhs <= 0) return H2G_OK;
  if (!d_points || !d_x || !d_y || !d_work || !d_coincident)
    return h2g_set_error(H2G_EINVAL, "h2g_direct_matvec: null argument");
  if (family < 0 || family > 2) return h2g_set_error(H2G_EINVAL, "h2g_direct_matvec: unknown family %d", family);
  const int nsplit = h2g::direct_splits(n);
  if (work_elems < (int64_t)nsplit * n * std::min(nrhs, 4))
    return h2g_set_error(H2G_EINVAL, "h2g_direct_matvec: workspace %lld < %lld", (long long)work_elems,
                         (long long)nsplit * n * std::min(nrhs, 4));
  cudaStream_t st = (cudaStream_t)stream;
  long long* flag = (long long*)d_coincident;
  for (int c = 0; c < nrhs; c += 4) {
    const int w = std::min(4, nrhs - c);
    const double* x = d_x + c;
    double* y = d_y + c;
    switch (w) {
      case 1: h2g::launch<1>(d_points, x, nrhs, y, nrhs, n, nsplit, family, shift, decay, d_work, flag, st); break;
      case 2: h2g::launch<2>(d_points, x, nrhs, y, nrhs, n, nsplit, family, shift, decay, d_work, flag, st); break;
      case 3: h2g::launch<3>(d_points, x, nrhs, y, nrhs, n, nsplit, family, shift, decay, d_work, flag, st); break;
      default: h2g::launch<4>(d_points, x, nrhs, y, nrhs, n, nsplit, family, shift, decay, d_work, flag, st); break;
    }
    int rc = h2g_check_launch("direct_matvec");
    if (rc != H2G_OK) return rc;
  }
  return H2G_OK;
}
