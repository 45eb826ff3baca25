// Panel step of the batched partial (ULV) Cholesky.
//
// For every box with r_i > p (one or more CTAs per box):
//   1. D = H[p:p+b, p:p+b] -> smem, identity-padded to 64x64
//   2. in-smem right-looking Cholesky of D (one barrier per column);
//      a pivot that is not > 0 (or NaN) records atomicMin(npd[slot], p+j)
//      exactly like dpotrf's info (dense_core.py:60-63)
//   3. Linv = L^-1 in smem (4 lanes per column, shuffle-reduced)
//   4. the CTA's slice of the rows below the panel — H[p+b:n, p:p+b]
//      (the L(r) rows still below the panel and the SR rows = L(s)_ii) and
//      R[0:nr, p:p+b] (q_red rows = V_i) — is overwritten by X * Linv^T on
//      the FP64 tensor pipe (64x64x64 DMMA tile per 64-row chunk).
// The trailing update that completes the right-looking step is a grouped
// GEMM launch (NT, alpha=-1, beta=1).  Over all panels this computes
// L(r)_ii = chol(RR), L(s)_ii = SR L^-T, V_i = q_red L^-T and
// SS_ii - L(s) L(s)^T  (ulv_factor.py:217-241) in one pass over H.
#include "common.cuh"

namespace h2g {

constexpr int PB = 64;        // max panel width
constexpr int PS = PB + 4;    // smem row stride (4 mod 16 doubles: conflict-free fragments)
constexpr int PANEL_THREADS = 256;
constexpr int PANEL_SMEM = 3 * PB * PS * 8;

__global__ void __launch_bounds__(PANEL_THREADS) panel_potrf_kernel(const h2g_panel_desc* __restrict__ descs,
                                                                    const int32_t* __restrict__ cta_map,
                                                                    int32_t* __restrict__ npd) {
  extern __shared__ __align__(16) double psm[];
  double* Ds = psm;               // L (lower), identity padded
  double* Li = psm + PB * PS;     // L^-1
  double* Xs = psm + 2 * PB * PS; // row chunk

  const int di = cta_map[blockIdx.x];
  const h2g_panel_desc P = descs[di];
  const int local = blockIdx.x - P.cta_start;
  const int tid = threadIdx.x;
  const int p = P.p, b = P.b;
  double* __restrict__ H = P.H;
  const int ldh = P.ldh;

  // 1. load D (lower part), identity padding
  for (int e = tid; e < PB * PB; e += PANEL_THREADS) {
    int r = e / PB, c = e % PB;
    double v;
    if (r < b && c < b) v = (c <= r) ? H[(size_t)(p + r) * ldh + p + c] : 0.0;
    else v = (r == c) ? 1.0 : 0.0;
    Ds[r * PS + c] = v;
  }
  __syncthreads();

  // 2. Cholesky: thread -> row i = tid/4, columns k = j+1+cq (step 4)
  {
    const int i = tid >> 2, cq = tid & 3;
    for (int j = 0; j < PB; ++j) {
      const double djj = Ds[j * PS + j];
      if (i > j) {
        const double lij = Ds[i * PS + j] / djj;
        for (int k = j + 1 + cq; k <= i; k += 4) Ds[i * PS + k] -= lij * Ds[k * PS + j];
      }
      __syncthreads();
      // finalize column j (no other thread touches column j in step j+1's update phase)
      if (tid == 0) {
        if (!(djj > 0.0) && j < b && local == 0) atomicMin(&npd[P.npd_slot], p + j);
      }
      const double sq = sqrt(djj);
      if (tid > j && tid < PB) Ds[tid * PS + j] /= sq;
      if (tid == j) Ds[j * PS + j] = sq;
      // entries in column j are read again only after the next barrier
    }
    __syncthreads();
  }

  // write the factored diagonal block back (once per box)
  if (local == 0) {
    for (int e = tid; e < b * b; e += PANEL_THREADS) {
      int r = e / b, c = e % b;
      if (c <= r) H[(size_t)(p + r) * ldh + p + c] = Ds[r * PS + c];
    }
  }

  const int rows_h = P.n - p - b;           // H rows below the panel
  const int rows_total = rows_h + P.nr;
  const int row_begin = local * P.rows_per_cta;
  const int row_end = min(rows_total, row_begin + P.rows_per_cta);
  if (row_begin >= row_end) return;

  // 3. Linv: 4 lanes per column c, rows i >= c sequentially
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

  // 4. Y = X * Linv^T over 64-row chunks on DMMA; warp w -> rows (w&3)*16.., cols (w>>2)*32..
  const int lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, tq = lane & 3;
  const int wr = (warp & 3) * 16, wc = (warp >> 2) * 32;
  double* __restrict__ R = P.R;
  const int ldr = P.ldr;
  for (int c0 = row_begin; c0 < row_end; c0 += PB) {
    const int nrows = min(PB, row_end - c0);
    for (int e = tid; e < PB * PB; e += PANEL_THREADS) {
      int r = e / PB, c = e % PB;
      double v = 0.0;
      if (r < nrows && c < b) {
        int vr = c0 + r;
        v = (vr < rows_h) ? H[(size_t)(p + b + vr) * ldh + p + c] : R[(size_t)(vr - rows_h) * ldr + p + c];
      }
      Xs[r * PS + c] = v;
    }
    __syncthreads();
    double acc[2][4][2];
#pragma unroll
    for (int a = 0; a < 2; ++a)
#pragma unroll
      for (int bq = 0; bq < 4; ++bq) acc[a][bq][0] = acc[a][bq][1] = 0.0;
#pragma unroll 4
    for (int kk = 0; kk < PB; kk += 4) {
      double af[2], bf[4];
#pragma unroll
      for (int a = 0; a < 2; ++a) af[a] = Xs[(wr + a * 8 + g) * PS + kk + tq];
#pragma unroll
      for (int bq = 0; bq < 4; ++bq) bf[bq] = Li[(wc + bq * 8 + g) * PS + kk + tq];  // Linv^T[k][n] = Li[n][k]
#pragma unroll
      for (int a = 0; a < 2; ++a)
#pragma unroll
        for (int bq = 0; bq < 4; ++bq) dmma884(acc[a][bq], af[a], bf[bq]);
    }
#pragma unroll
    for (int a = 0; a < 2; ++a) {
      int r = wr + a * 8 + g;
      if (r >= nrows) continue;
      int vr = c0 + r;
      double* dst = (vr < rows_h) ? H + (size_t)(p + b + vr) * ldh + p : R + (size_t)(vr - rows_h) * ldr + p;
#pragma unroll
      for (int bq = 0; bq < 4; ++bq) {
        int c = wc + bq * 8 + 2 * tq;
        if (c < b) dst[c] = acc[a][bq][0];
        if (c + 1 < b) dst[c + 1] = acc[a][bq][1];
      }
    }
    __syncthreads();
  }
}

}  // namespace h2g

extern "C" int h2g_panel_potrf(const h2g_panel_desc* d_descs, const int32_t* d_cta_map, int total_ctas,
                               int32_t* d_npd, void* stream) {
  if (total_ctas <= 0) return H2G_OK;
  if (!d_descs || !d_cta_map || !d_npd) return h2g_set_error(H2G_EINVAL, "h2g_panel_potrf: null argument");
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(h2g::panel_potrf_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, h2g::PANEL_SMEM);
    attr = true;
  }
  h2g::panel_potrf_kernel<<<total_ctas, h2g::PANEL_THREADS, h2g::PANEL_SMEM, (cudaStream_t)stream>>>(
      d_descs, d_cta_map, d_npd);
  return h2g_check_launch("panel_potrf");
}
