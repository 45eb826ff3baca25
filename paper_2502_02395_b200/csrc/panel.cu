// Diagonal-block step of the batched partial (ULV) Cholesky.
//
// One CTA per box with r_i > p: D = H[p:p+b, p:p+b] (b <= 64, identity
// padded to 64) is factored and written back as L_pp, and W = L_pp^-1 is
// written to a 64x64 scratch block (used by the TRSM GEMM and later by the
// substitution).
//
// Latency is what matters here (one small block per box, all boxes in one
// wave), so the factorization is a square-root-free LDL^T elimination with
// the 64x64 matrix distributed over the CTA in 2x2 register blocks (thread
// (br, bc) owns rows 2br.., columns 2bc..): in step j every thread updates
// its 4 entries with the pivot column j and the finished row j of
// V = U^-1 (U unit lower), then the owners of column j+1 / row j+1 publish
// them to shared memory and ONE barrier ends the step.  No entry moves
// between threads; the chain per step is barrier + 1 broadcast load + one
// reciprocal + one FMA.  At the end L = U diag(sqrt d), L^-1 = diag(1/sqrt d) V.
// A pivot that is not > 0 (or NaN) records atomicMin(npd[slot], p+j): the
// pivot dpotrf reports as info-1 (dense_core.py:60-63).
//
// The rest of the panel step is tensor-pipe GEMM work issued by the host
// program (ulv_factor.FactorPlan): TRSM X <- X Linv^T in place for the rows
// below the panel of H and for the q_red rows of R, then the trailing update.
// Over all panels: L(r)_ii = chol(RR), L(s)_ii = SR L^-T, V_i = q_red L^-T and
// SS_ii - L(s) L(s)^T (ulv_factor.py:217-241).
#include <climits>

#include "common.cuh"

namespace h2g {

constexpr int PB = 64;        // max panel width
constexpr int BS = 2;                 // register block per thread
constexpr int NBLK = (PB / BS) * (PB / BS + 1) / 2;   // 528 lower blocks
constexpr int DIAG_THREADS = 544;

#ifdef H2G_DIAG_TRACE
__device__ long long g_diag_trace[64];
#define TRACE(k) do { if (blockIdx.x == 0 && threadIdx.x == 0) g_diag_trace[k] = clock64(); } while (0)
#else
#define TRACE(k) do { } while (0)
#endif

__global__ void __launch_bounds__(DIAG_THREADS) potrf_diag_kernel(const h2g_panel_desc* __restrict__ descs,
                                                                  int32_t* __restrict__ npd) {
  // colD[buf][r]: column j of the working matrix for rows r > j, ZERO for rows <= j
  // (so the multiplier of a finished row is 0 without a branch); rowV[buf][x]:
  // row j of V = U^-1, zero for x > j.  pv / rpv: pivots and their reciprocals.
  __shared__ __align__(16) double colD[2][PB];
  __shared__ __align__(16) double rowV[2][PB];
  __shared__ double pv[PB], rpv[PB];
  const h2g_panel_desc P = descs[blockIdx.x];
  const int tid = threadIdx.x;
  // the NBLK lower 2x2 blocks are enumerated row by row over threads 0..NBLK-1
  int br = (int)((sqrtf(8.0f * tid + 1.0f) - 1.0f) * 0.5f);
  while ((br + 1) * (br + 2) / 2 <= tid) ++br;
  while (br * (br + 1) / 2 > tid) --br;
  int bc = tid - br * (br + 1) / 2;
  const bool active = tid < NBLK;
  if (!active) br = bc = 0;          // idle threads shadow block (0,0) but never publish
  const int r0 = BS * br, c0 = BS * bc;
  const int p = P.p, b = P.b;
  double* H = P.H;
  const int ldh = P.ldh;
  TRACE(0);

  double d[BS][BS], v[BS][BS];
#pragma unroll
  for (int a = 0; a < BS; ++a)
#pragma unroll
    for (int e = 0; e < BS; ++e) {
      const int i = r0 + a, x = c0 + e;
      double val = 0.0;
      if (active && x <= i) {
        if (i < b && x < b) val = H[(size_t)(p + i) * ldh + p + x];
        else val = (i == x) ? 1.0 : 0.0;
      }
      d[a][e] = val;
      v[a][e] = (i == x) ? 1.0 : 0.0;
    }
  if (tid < PB) {
    rowV[0][tid] = (tid == 0) ? 1.0 : 0.0;
    rowV[1][tid] = 0.0;
    colD[1][tid] = 0.0;
  }
  if (active && bc == 0) {
    colD[0][r0] = (r0 == 0) ? 0.0 : d[0][0];
    colD[0][r0 + 1] = d[1][0];
    if (r0 == 0) {
      pv[0] = d[0][0];
      rpv[0] = 1.0 / d[0][0];
    }
  }
  __syncthreads();
  TRACE(1);

#pragma unroll 1
  for (int j = 0; j < PB; ++j) {
    const int cur = j & 1;
    const double rj = rpv[j];
    const double2 cr = reinterpret_cast<const double2*>(&colD[cur][0])[br];
    const double2 cc = reinterpret_cast<const double2*>(&colD[cur][0])[bc];
    const double2 rv = reinterpret_cast<const double2*>(&rowV[cur][0])[bc];
    const double li0 = cr.x * rj, li1 = cr.y * rj;          // 0 for rows <= j
    d[0][0] = fma(-li0, cc.x, d[0][0]);                      // cc: 0 for columns <= j
    d[0][1] = fma(-li0, cc.y, d[0][1]);
    d[1][0] = fma(-li1, cc.x, d[1][0]);
    d[1][1] = fma(-li1, cc.y, d[1][1]);
    v[0][0] = fma(-li0, rv.x, v[0][0]);                      // rv: 0 for columns > j
    v[0][1] = fma(-li0, rv.y, v[0][1]);
    v[1][0] = fma(-li1, rv.x, v[1][0]);
    v[1][1] = fma(-li1, rv.y, v[1][1]);
    // publish column / row jn = j+1 (final after this update) into the other buffer
    const int jn = j + 1;
    if (active && jn < PB) {
      const bool hi = jn & 1;
      if ((jn >> 1) == bc) {
        const double c_0 = hi ? d[0][1] : d[0][0], c_1 = hi ? d[1][1] : d[1][0];
        double* cn = colD[cur ^ 1];
        cn[r0] = (r0 > jn) ? c_0 : 0.0;
        cn[r0 + 1] = (r0 + 1 > jn) ? c_1 : 0.0;
        if (br == bc) {                                      // owner of the pivot d_jn
          const double dn = hi ? d[1][1] : d[0][0];
          pv[jn] = dn;
          rpv[jn] = 1.0 / dn;
          if (jn >= 2) cn[jn - 2] = 0.0;                     // rows that finished since
          cn[jn - 1] = 0.0;                                  //   this buffer was last filled
        }
      }
      if ((jn >> 1) == br) {
        double* rn = rowV[cur ^ 1];
        rn[c0] = hi ? v[1][0] : v[0][0];
        rn[c0 + 1] = hi ? v[1][1] : v[0][1];
      }
    }
    __syncthreads();
  }
  TRACE(2);
  if (tid == 0) {
    for (int j = 0; j < b; ++j)
      if (!(pv[j] > 0.0)) {
        atomicMin(&npd[P.npd_slot], p + j);
        break;
      }
  }

  // L[i][x] = D[i][x] / sqrt(d_x) (x < i), L[x][x] = sqrt(d_x);  Linv[i][x] = V[i][x] / sqrt(d_i)
  double* __restrict__ out = P.Linv;  // 64 x 64 scratch, ld = ldl
  if (active) {
#pragma unroll
    for (int a = 0; a < BS; ++a)
#pragma unroll
      for (int e = 0; e < BS; ++e) {
        const int i = r0 + a, x = c0 + e;
        double wv = 0.0;
        if (x <= i && i < b) {
          const double sx = sqrt(pv[x]);
          wv = v[a][e] / sqrt(pv[i]);
          H[(size_t)(p + i) * ldh + p + x] = (x == i) ? sx : d[a][e] / sx;
        }
        out[(size_t)i * P.ldl + x] = wv;
        if (bc < br) out[(size_t)x * P.ldl + i] = 0.0;   // mirror block above the diagonal
      }
  }
  TRACE(3);
}

}  // namespace h2g

extern "C" int h2g_panel_potrf(const h2g_panel_desc* d_descs, int count, int32_t* d_npd, void* stream) {
  if (count <= 0) return H2G_OK;
  if (!d_descs || !d_npd) return h2g_set_error(H2G_EINVAL, "h2g_panel_potrf: null argument");
  h2g::potrf_diag_kernel<<<count, h2g::DIAG_THREADS, 0, (cudaStream_t)stream>>>(d_descs, d_npd);
  return h2g_check_launch("potrf_diag");
}
