// Diagonal-block step of the batched partial (ULV) Cholesky.
//
// One CTA per box with r_i > p: D = H[p:p+b, p:p+b] (b <= 64) is factored in
// shared memory and written back as L_pp, and W = L_pp^-1 is written to a
// 64x64 scratch block.  Cholesky and inverse advance together, one column per
// step and ONE barrier per step: in step j every thread owns one row i and a
// quarter of its columns, and applies
//     L[i][j] = D[i][j] / sqrt(d_jj)
//     D[i][k] -= L[i][j] L[k][j]      (j < k <= i)   trailing update
//     W[i][c] -= L[i][j] W[j][c]      (c <= j)       inverse, row elimination
// using the still-unscaled column j / row j (scaled lazily after the
// barrier, where nothing reads them any more).  All per-thread updates of a
// step are independent, so they issue back to back (16-way unrolled).
// A pivot that is not > 0 (or NaN) records atomicMin(npd[slot], p+j):
// dpotrf's info-1 (dense_core.py:60-63).
//
// The rest of the panel step is tensor-pipe GEMM work issued by the host
// program (ulv_factor.FactorPlan): TRSM X <- X Linv^T in place for the rows
// below the panel of H and for the q_red rows of R, then the trailing update.
// Over all panels: L(r)_ii = chol(RR), L(s)_ii = SR L^-T, V_i = q_red L^-T and
// SS_ii - L(s) L(s)^T (ulv_factor.py:217-241).
#include "common.cuh"

namespace h2g {

constexpr int PB = 64;        // max panel width
constexpr int PS = PB + 1;    // odd stride: conflict-free row and column walks
constexpr int DIAG_THREADS = 256;

__global__ void __launch_bounds__(DIAG_THREADS) potrf_diag_kernel(const h2g_panel_desc* __restrict__ descs,
                                                                  int32_t* __restrict__ npd) {
  extern __shared__ double dsm[];
  double* Ds = dsm;              // D, becomes L (lower)
  double* Ws = dsm + PB * PS;    // W, becomes L^-1 (lower)
  const h2g_panel_desc P = descs[blockIdx.x];
  const int tid = threadIdx.x;
  const int p = P.p, b = P.b;
  double* H = P.H;
  const int ldh = P.ldh;

  // load D (lower, identity padded) and W = I; 16 independent loads per thread
#pragma unroll
  for (int t = 0; t < (PB * PB) / DIAG_THREADS; ++t) {
    const int e = tid + t * DIAG_THREADS;
    const int r = e >> 6, c = e & 63;
    double v;
    if (r < b && c < b) v = (c <= r) ? H[(size_t)(p + r) * ldh + p + c] : 0.0;
    else v = (r == c) ? 1.0 : 0.0;
    Ds[r * PS + c] = v;
    Ws[r * PS + c] = (r == c) ? 1.0 : 0.0;
  }
  __syncthreads();

  const int i = tid >> 2, cq = tid & 3;
  for (int j = 0; j < PB; ++j) {
    const double djj = Ds[j * PS + j];
    const double rinv = 1.0 / sqrt(djj);
    if (i > j) {
      const double lij = Ds[i * PS + j] * rinv;
#pragma unroll
      for (int t = 0; t < PB / 4; ++t) {
        const int c = cq + 4 * t;
        if (c <= j) {
          Ws[i * PS + c] -= lij * (Ws[j * PS + c] * rinv);
        } else if (c <= i) {
          Ds[i * PS + c] -= lij * (Ds[c * PS + j] * rinv);
        }
      }
    }
    __syncthreads();
    // finalize column j of L and row j of W (no thread reads them in step j+1)
    if (tid == 0 && !(djj > 0.0) && j < b) atomicMin(&npd[P.npd_slot], p + j);
    if (tid > j && tid < PB) Ds[tid * PS + j] *= rinv;
    if (tid == j) Ds[j * PS + j] = djj * rinv;   // sqrt(djj)
    if (tid >= PB && tid - PB <= j) Ws[j * PS + (tid - PB)] *= rinv;
  }
  __syncthreads();

  double* __restrict__ out = P.Linv;  // 64 x 64 scratch, ld = ldl
#pragma unroll
  for (int t = 0; t < (PB * PB) / DIAG_THREADS; ++t) {
    const int e = tid + t * DIAG_THREADS;
    const int r = e >> 6, c = e & 63;
    out[(size_t)r * P.ldl + c] = (r < b && c < b && c <= r) ? Ws[r * PS + c] : 0.0;
    if (r < b && c <= r) H[(size_t)(p + r) * ldh + p + c] = Ds[r * PS + c];
  }
}

}  // namespace h2g

extern "C" int h2g_panel_potrf(const h2g_panel_desc* d_descs, int count, int32_t* d_npd, void* stream) {
  if (count <= 0) return H2G_OK;
  if (!d_descs || !d_npd) return h2g_set_error(H2G_EINVAL, "h2g_panel_potrf: null argument");
  const int smem = 2 * h2g::PB * h2g::PS * 8;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(h2g::potrf_diag_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    attr = true;
  }
  h2g::potrf_diag_kernel<<<count, h2g::DIAG_THREADS, smem, (cudaStream_t)stream>>>(d_descs, d_npd);
  return h2g_check_launch("potrf_diag");
}
