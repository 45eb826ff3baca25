// Diagonal-block step of the batched partial (ULV) Cholesky.
//
// One CTA per box with r_i > p: D = H[p:p+b, p:p+b] (b <= 64, identity
// padded to 64) is factored in shared memory, written back as L_pp, and
// W = L_pp^-1 is written to a 64x64 scratch block (used by the TRSM GEMM and
// later by the substitution).  The 64x64 factorization is blocked by 16:
//   for each 16-column block K:
//     warp 0   : unblocked Cholesky of the 16x16 diagonal block (warp-synchronous,
//                no CTA barrier) and its 16x16 inverse
//     all warps: TRSM of the rows below with that inverse, SYRK of the trailing part
//   all warps  : block forward substitution W_IJ = -W_II sum_K L_IK W_KJ
// so the serial chain is 4 x 16 cheap warp steps instead of 64 CTA-wide
// steps.  A pivot that is not > 0 (or NaN) records atomicMin(npd[slot], p+j):
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
constexpr int SB = 16;        // inner block
constexpr int DIAG_THREADS = 256;

__global__ void __launch_bounds__(DIAG_THREADS) potrf_diag_kernel(const h2g_panel_desc* __restrict__ descs,
                                                                  int32_t* __restrict__ npd) {
  extern __shared__ double dsm[];
  double* Ds = dsm;              // D, becomes L (lower)
  double* Ws = dsm + PB * PS;    // becomes L^-1 (lower)
  __shared__ double Xt[48 * SB];  // TRSM results staging
  const h2g_panel_desc P = descs[blockIdx.x];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int p = P.p, b = P.b;
  double* H = P.H;
  const int ldh = P.ldh;

#pragma unroll
  for (int t = 0; t < (PB * PB) / DIAG_THREADS; ++t) {
    const int e = tid + t * DIAG_THREADS;
    const int r = e >> 6, c = e & 63;
    double v;
    if (r < b && c < b) v = (c <= r) ? H[(size_t)(p + r) * ldh + p + c] : 0.0;
    else v = (r == c) ? 1.0 : 0.0;
    Ds[r * PS + c] = v;
    Ws[r * PS + c] = 0.0;
  }
  __syncthreads();

  for (int kb = 0; kb < PB; kb += SB) {
    // ---- (a) warp 0: 16x16 Cholesky + inverse of the diagonal block
    if (warp == 0) {
      double* Dk = Ds + kb * PS + kb;
      for (int j = 0; j < SB; ++j) {
        const double djj = Dk[j * PS + j];
        const double rinv = 1.0 / sqrt(djj);
        if (lane == 0 && !(djj > 0.0) && kb + j < b) atomicMin(&npd[P.npd_slot], p + kb + j);
        // trailing update inside the block with the unscaled column j
        for (int e = lane; e < SB * SB; e += 32) {
          const int i = e >> 4, k = e & 15;
          if (k > j && k <= i) Dk[i * PS + k] -= Dk[i * PS + j] * Dk[k * PS + j] * (rinv * rinv);
        }
        __syncwarp();
        if (lane > j && lane < SB) Dk[lane * PS + j] *= rinv;
        if (lane == j) Dk[j * PS + j] = djj * rinv;
        __syncwarp();
      }
      // inverse of the 16x16 lower block: lane c < 16 solves column c
      if (lane < SB) {
        const int c = lane;
        double* Wk = Ws + kb * PS + kb;
        for (int i = 0; i < SB; ++i) {
          double s = (i == c) ? 1.0 : 0.0;
          for (int m = c; m < i; ++m) s -= Dk[i * PS + m] * Wk[m * PS + c];
          Wk[i * PS + c] = (i >= c) ? s / Dk[i * PS + i] : 0.0;
        }
      }
    }
    __syncthreads();
    const int below = PB - kb - SB;  // rows under the block
    if (below > 0) {
      // ---- (b) TRSM: X[r][c] = sum_{m<=c} D[kb+16+r][kb+m] * W_kk[c][m]
      for (int e = tid; e < below * SB; e += DIAG_THREADS) {
        const int r = e >> 4, c = e & 15;
        const double* xr = Ds + (kb + SB + r) * PS + kb;
        const double* wc = Ws + (kb + c) * PS + kb;
        double s = 0.0;
#pragma unroll
        for (int m = 0; m < SB; ++m)
          if (m <= c) s += xr[m] * wc[m];
        Xt[r * SB + c] = s;
      }
      __syncthreads();
      for (int e = tid; e < below * SB; e += DIAG_THREADS) {
        const int r = e >> 4, c = e & 15;
        Ds[(kb + SB + r) * PS + kb + c] = Xt[r * SB + c];
      }
      // ---- (c) SYRK: D[i][k] -= sum_m X[i][m] X[k][m]   (kb+16 <= k <= i)
      for (int e = tid; e < below * below; e += DIAG_THREADS) {
        const int ii = e / below, kk = e % below;
        if (kk > ii) continue;
        const double* xi = Xt + ii * SB;
        const double* xk = Xt + kk * SB;
        double s = 0.0;
#pragma unroll
        for (int m = 0; m < SB; ++m) s += xi[m] * xk[m];
        Ds[(kb + SB + ii) * PS + kb + SB + kk] -= s;
      }
      __syncthreads();
    }
  }

  // ---- block forward substitution for the off-diagonal blocks of W = L^-1
  for (int I = 1; I < PB / SB; ++I) {
    // T_J[r][c] = sum_{K=J}^{I-1} L[I][K] W[K][J]  for J < I  (into Xt, I*256 <= 768 entries)
    for (int e = tid; e < I * SB * SB; e += DIAG_THREADS) {
      const int J = e >> 8, r = (e >> 4) & 15, c = e & 15;
      const double* lrow = Ds + (I * SB + r) * PS;
      double s = 0.0;
      for (int m = J * SB + c; m < I * SB; ++m) s += lrow[m] * Ws[m * PS + J * SB + c];
      Xt[e] = s;
    }
    __syncthreads();
    // W[I][J] = -W_II T_J
    for (int e = tid; e < I * SB * SB; e += DIAG_THREADS) {
      const int J = e >> 8, r = (e >> 4) & 15, c = e & 15;
      const double* wrow = Ws + (I * SB + r) * PS + I * SB;
      double s = 0.0;
#pragma unroll
      for (int m = 0; m < SB; ++m)
        if (m <= r) s += wrow[m] * Xt[(J << 8) + (m << 4) + c];
      Ws[(I * SB + r) * PS + J * SB + c] = -s;
    }
    __syncthreads();
  }

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
