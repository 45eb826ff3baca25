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

// 2x2 pivot block [[a, .], [b, c]]: a, b, c, 1/a, u = b/a, 1/d1, d1 = c - b^2/a
__device__ __forceinline__ void pivot_block(double* s, double a, double b, double c) {
  const double ra = 1.0 / a;
  const double det = fma(a, c, -b * b);
  const double rdet = 1.0 / det;
  s[0] = a;
  s[1] = b;
  s[2] = c;
  s[3] = ra;
  s[4] = b * ra;
  s[5] = a * rdet;
  s[6] = det * ra;
}

__global__ void __launch_bounds__(DIAG_THREADS) potrf_diag_kernel(const h2g_panel_desc* __restrict__ descs,
                                                                  int32_t* __restrict__ npd) {
  // Step q eliminates the 2x2 pivot block {2q, 2q+1} (two scalar LDL^T steps
  // fused, so 32 barriers instead of 64).  Published per step, double buffered:
  //   colX / colY : columns 2q and 2q+1 of the working matrix for rows > 2q+1,
  //                 zero for rows <= 2q+1 (multipliers of finished rows are 0)
  //   rowA / rowB : rows 2q and 2q+1 of V = U^-1 (rowB before its in-block step)
  //   scal        : the pivot block a = D[2q][2q], b = D[2q+1][2q], c = D[2q+1][2q+1]
  __shared__ __align__(16) double colX[2][PB], colY[2][PB], rowA[2][PB], rowB[2][PB];
  __shared__ __align__(16) double scal[2][8];
  __shared__ double pv[PB];
  const h2g_panel_desc P = descs[blockIdx.x];
  const int tid = threadIdx.x;
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
    colX[1][tid] = colY[1][tid] = 0.0;
    rowA[0][tid] = (tid == 0) ? 1.0 : 0.0;
    rowB[0][tid] = (tid == 1) ? 1.0 : 0.0;
    rowA[1][tid] = rowB[1][tid] = 0.0;
  }
  if (active && bc == 0) {
    colX[0][r0] = (br > 0) ? d[0][0] : 0.0;
    colX[0][r0 + 1] = (br > 0) ? d[1][0] : 0.0;
    colY[0][r0] = (br > 0) ? d[0][1] : 0.0;
    colY[0][r0 + 1] = (br > 0) ? d[1][1] : 0.0;
    if (br == 0) pivot_block(scal[0], d[0][0], d[1][0], d[1][1]);
  }
  __syncthreads();
  TRACE(1);

#pragma unroll 1
  for (int q = 0; q < PB / 2; ++q) {
    const int cur = q & 1, nxt = cur ^ 1;
    const double ra = scal[cur][3], u = scal[cur][4], rd1 = scal[cur][5];
    if (tid == 0) {
      pv[2 * q] = scal[cur][0];
      pv[2 * q + 1] = scal[cur][6];
    }
    if (br > q) {
      const double2 xr = reinterpret_cast<const double2*>(&colX[cur][0])[br];
      const double2 yr = reinterpret_cast<const double2*>(&colY[cur][0])[br];
      const double2 xc = reinterpret_cast<const double2*>(&colX[cur][0])[bc];
      const double2 yc = reinterpret_cast<const double2*>(&colY[cur][0])[bc];
      const double2 ac = reinterpret_cast<const double2*>(&rowA[cur][0])[bc];
      const double2 bcv = reinterpret_cast<const double2*>(&rowB[cur][0])[bc];
      const double xrs[2] = {xr.x, xr.y}, yrs[2] = {yr.x, yr.y};
      const double xcs[2] = {xc.x, xc.y}, ycs[2] = {fma(-u, xc.x, yc.x), fma(-u, xc.y, yc.y)};
      const double acs[2] = {ac.x, ac.y}, bcs[2] = {bcv.x, bcv.y};
#pragma unroll
      for (int a = 0; a < BS; ++a) {
        const double al = xrs[a] * ra;                    // X_i / a
        const double be = fma(-u, xrs[a], yrs[a]) * rd1;  // Y'_i / d1
        const double ga = fma(-be, u, al);                // coefficient of row 2q of V
#pragma unroll
        for (int e = 0; e < BS; ++e) {
          d[a][e] = fma(-al, xcs[e], fma(-be, ycs[e], d[a][e]));
          v[a][e] = fma(-ga, acs[e], fma(-be, bcs[e], v[a][e]));
        }
      }
    }
    if (active && bc == q) {              // column 2q+1 of L uses Y' = Y - u X
      d[0][1] = fma(-u, d[0][0], d[0][1]);
      d[1][1] = fma(-u, d[1][0], d[1][1]);
    }
    if (active && br == q) {              // row 2q+1 of V after its in-block step
      v[1][0] = fma(-u, v[0][0], v[1][0]);
      v[1][1] = fma(-u, v[0][1], v[1][1]);
    }
    // publish pivot block q+1 (final after this step) into the other buffer
    const int qn = q + 1;
    if (active && qn < PB / 2) {
      if (bc == qn) {
        const bool below = br > qn;
        colX[nxt][r0] = below ? d[0][0] : 0.0;
        colX[nxt][r0 + 1] = below ? d[1][0] : 0.0;
        colY[nxt][r0] = below ? d[0][1] : 0.0;
        colY[nxt][r0 + 1] = below ? d[1][1] : 0.0;
        if (br == qn) {
          pivot_block(scal[nxt], d[0][0], d[1][0], d[1][1]);
          colX[nxt][2 * q] = colX[nxt][2 * q + 1] = 0.0;   // stale rows of this buffer
          colY[nxt][2 * q] = colY[nxt][2 * q + 1] = 0.0;
        }
      }
      if (br == qn) {
        rowA[nxt][c0] = v[0][0];
        rowA[nxt][c0 + 1] = v[0][1];
        rowB[nxt][c0] = v[1][0];
        rowB[nxt][c0 + 1] = v[1][1];
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
