// Diagonal-block step of the batched partial (ULV) Cholesky.
//
// One CTA per box with r_i > p: D = H[p:p+b, p:p+b] (b <= 64) is factored in
// shared memory (right-looking, one barrier per column), written back as
// L_pp, and its inverse L_pp^-1 is written to a 64x64 scratch block.  A pivot
// that is not > 0 (or NaN) records atomicMin(npd[slot], p+j): dpotrf's
// info-1 (dense_core.py:60-63).
//
// The rest of the panel step is GEMM work on the tensor pipe, issued by the
// host program right after this kernel:
//   TRSM   X <- X * Linv^T  for X = H[p+b:n, p:p+b] (L(r) rows and the SR rows
//          = L(s)_ii) and X = R[0:n, p:p+b] (q_red rows = V_i), in place
//          (each 64-row GEMM tile owns complete rows: N = b <= 64);
//   TRAIL  H[p+b:, p+b:] -= X X^T (lower tiles), R[:, p+b:r] -= V_P L[p+b:r, P]^T.
// Over all panels this is L(r)_ii = chol(RR), L(s)_ii = SR L^-T,
// V_i = q_red L^-T and SS_ii - L(s) L(s)^T (ulv_factor.py:217-241).
#include "common.cuh"

namespace h2g {

constexpr int PB = 64;        // max panel width
constexpr int PS = PB + 1;    // odd stride: conflict-free row and column walks
constexpr int DIAG_THREADS = 256;

__global__ void __launch_bounds__(DIAG_THREADS) potrf_diag_kernel(const h2g_panel_desc* __restrict__ descs,
                                                                  int32_t* __restrict__ npd) {
  extern __shared__ double dsm[];
  double* Ds = dsm;
  double* Li = dsm + PB * PS;
  const h2g_panel_desc P = descs[blockIdx.x];
  const int tid = threadIdx.x;
  const int p = P.p, b = P.b;
  double* H = P.H;
  const int ldh = P.ldh;

  for (int e = tid; e < PB * PB; e += DIAG_THREADS) {
    int r = e / PB, c = e % PB;
    double v;
    if (r < b && c < b) v = (c <= r) ? H[(size_t)(p + r) * ldh + p + c] : 0.0;
    else v = (r == c) ? 1.0 : 0.0;
    Ds[r * PS + c] = v;
  }
  __syncthreads();

  // right-looking Cholesky: thread -> row i = tid/4, columns k = j+1+cq (step 4)
  {
    const int i = tid >> 2, cq = tid & 3;
    for (int j = 0; j < PB; ++j) {
      const double djj = Ds[j * PS + j];
      if (i > j) {
        const double lij = Ds[i * PS + j] / djj;
        for (int k = j + 1 + cq; k <= i; k += 4) Ds[i * PS + k] -= lij * Ds[k * PS + j];
      }
      __syncthreads();
      if (tid == 0 && !(djj > 0.0) && j < b) atomicMin(&npd[P.npd_slot], p + j);
      const double sq = sqrt(djj);
      if (tid > j && tid < PB) Ds[tid * PS + j] /= sq;
      if (tid == j) Ds[j * PS + j] = sq;
      // column j is not read again before the next barrier
    }
    __syncthreads();
  }

  for (int e = tid; e < b * b; e += DIAG_THREADS) {
    int r = e / b, c = e % b;
    if (c <= r) H[(size_t)(p + r) * ldh + p + c] = Ds[r * PS + c];
  }

  // Linv: 4 lanes per column c, rows i >= c in order
  {
    const int c = tid >> 2, q = tid & 3;
    for (int i = 0; i < PB; ++i) {
      double s = 0.0;
      if (i > c)
        for (int m = c + q; m < i; m += 4) s += Ds[i * PS + m] * Li[m * PS + c];
      s += __shfl_xor_sync(0xffffffffu, s, 1);
      s += __shfl_xor_sync(0xffffffffu, s, 2);
      if (q == 0) {
        double v;
        if (i < c) v = 0.0;
        else if (i == c) v = 1.0 / Ds[i * PS + i];
        else v = -s / Ds[i * PS + i];
        Li[i * PS + c] = v;
      }
      __syncwarp();
    }
  }
  __syncthreads();
  double* __restrict__ out = P.Linv;  // 64 x 64 scratch, ld = ldl
  for (int e = tid; e < PB * PB; e += DIAG_THREADS) {
    int r = e / PB, c = e % PB;
    out[(size_t)r * P.ldl + c] = (r < b && c < b) ? Li[r * PS + c] : 0.0;
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
