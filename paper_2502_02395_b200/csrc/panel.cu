// Cholesky panels of the batched partial (ULV) Cholesky.
//
// The ULV step of a box is a right-looking Cholesky of H_i = Q_i^T A_ii Q_i
// that stops after r_i pivots: the 64-wide panels factor RR, their rows
// below become L(s)_ii = SR L^-T and the trailing updates of the SS corner
// are the single Schur update SS - L(s) L(s)^T (ulv_factor.py:217-241).
//
// Kernels, all built on one 64x64 factorization routine (diag_ldlt):
//
//  potrf_diag_kernel     (h2g_panel_potrf) one CTA per box: factor the
//                        diagonal block H[p:p+b, p:p+b] in place and write
//                        its inverse.  Kept as a stand-alone ABI entry.
//  chol_diag_kernel +    (h2g_chol_panel) the panel step used by the
//  chol_rows_kernel      factorization, see the section below: together
//                        they apply the previous panel to block column q,
//                        factor its diagonal block and TRSM the rows below,
//                        so the critical lane issues two kernels per panel;
//                        the update of the columns right of the next panel
//                        (REST) is a grouped GEMM on a side lane.
//
// diag_ldlt: square-root-free LDL^T elimination of a 64x64 block distributed
// over the CTA in BSxBS register blocks (thread (br, bc) owns rows
// BS*br.., columns BS*bc.., br >= bc), two pivots per step (a 2x2 pivot
// block), one barrier per step; the inverse V = U^-1 (U unit lower) is
// eliminated alongside.  At the end L = U diag(sqrt d), L^-1 = diag(1/sqrt d) V.
// A pivot that is not > 0 (or NaN) records atomicMin(npd[slot], p+j): the
// pivot dpotrf reports as info-1 (dense_core.py:60-63).
#include <climits>

#include "common.cuh"

namespace h2g {

#ifdef H2G_PANEL_TRACE
__device__ long long g_panel_trace[16];
#define PTRACE(k) do { if (blockIdx.x == 0 && threadIdx.x == 0) g_panel_trace[k] = clock64(); } while (0)
#else
#define PTRACE(k) do { } while (0)
#endif

constexpr int PB = 64;   // panel width
constexpr int SD = 68;   // smem stride (doubles) of the 64-wide blocks: 68 = 4 mod 16 -> conflict-free fragments

template <int BS>
struct Ldlt {
  static constexpr int NBLK = PB / BS;
  static constexpr int NT = NBLK * (NBLK + 1) / 2;   // active threads
};

struct LdltShared {
  double colX[2][PB], colY[2][PB], rowA[2][PB], rowB[2][PB];
  double scal[2][8];
  double pv[PB];
};

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

__device__ __forceinline__ void tri_index(int t, int& br, int& bc) {
  int i = (int)((sqrtf(8.0f * t + 1.0f) - 1.0f) * 0.5f);
  while ((i + 1) * (i + 2) / 2 <= t) ++i;
  while (i * (i + 1) / 2 > t) --i;
  br = i;
  bc = t - i * (i + 1) / 2;
}

// Factor the 64x64 block D (smem, stride SD; only the lower triangle is
// read; rows/cols >= b are treated as identity).  On return
//   L (lower, incl. diagonal) is in D, Li (stride SD) holds L^-1 with zeros
//   above the diagonal, sh.pv[j] holds the pivots d_j.
// Must be called by every thread of the CTA (nthreads >= Ldlt<BS>::NT).
template <int BS>
__device__ void diag_ldlt(double* D, double* Li, int b, LdltShared& sh) {
  const int tid = threadIdx.x;
  const bool active = tid < Ldlt<BS>::NT;
  int br = 0, bc = 0;
  if (active) tri_index(tid, br, bc);
  const int r0 = BS * br, c0 = BS * bc;

  double d[BS][BS], v[BS][BS];
#pragma unroll
  for (int a = 0; a < BS; ++a)
#pragma unroll
    for (int e = 0; e < BS; ++e) {
      const int i = r0 + a, x = c0 + e;
      double val = 0.0;
      if (active && x <= i) val = (i < b && x < b) ? D[i * SD + x] : (i == x ? 1.0 : 0.0);
      d[a][e] = val;
      v[a][e] = (i == x) ? 1.0 : 0.0;
    }
  if (tid < PB) {
    sh.colX[1][tid] = sh.colY[1][tid] = 0.0;
    sh.rowA[0][tid] = (tid == 0) ? 1.0 : 0.0;
    sh.rowB[0][tid] = (tid == 1) ? 1.0 : 0.0;
    sh.rowA[1][tid] = sh.rowB[1][tid] = 0.0;
  }
  __syncthreads();   // D reads above may alias nothing, but sh init must precede the publish below
  if (active && bc == 0) {   // publish pivot pair 0 (columns 0, 1)
#pragma unroll
    for (int a = 0; a < BS; ++a) {
      const int row = r0 + a;
      sh.colX[0][row] = row > 1 ? d[a][0] : 0.0;
      sh.colY[0][row] = row > 1 ? d[a][1] : 0.0;
    }
    if (br == 0) pivot_block(sh.scal[0], d[0][0], d[1][0], d[1][1]);
  }
  __syncthreads();

#pragma unroll 1
  for (int q = 0; q < PB / 2; ++q) {
    const int cur = q & 1, nxt = cur ^ 1;
    const int qb = (2 * q) / BS, o = (2 * q) % BS;
    const double ra = sh.scal[cur][3], u = sh.scal[cur][4], rd1 = sh.scal[cur][5];
    if (tid == 0) {
      sh.pv[2 * q] = sh.scal[cur][0];
      sh.pv[2 * q + 1] = sh.scal[cur][6];
    }
    if (active && br >= qb) {
      double xr[BS], yr[BS], xc[BS], yc[BS], ac[BS], bv[BS];
#pragma unroll
      for (int a = 0; a < BS; a += 2) {
        const double2 t0 = *reinterpret_cast<const double2*>(&sh.colX[cur][r0 + a]);
        const double2 t1 = *reinterpret_cast<const double2*>(&sh.colY[cur][r0 + a]);
        const double2 t2 = *reinterpret_cast<const double2*>(&sh.colX[cur][c0 + a]);
        const double2 t3 = *reinterpret_cast<const double2*>(&sh.colY[cur][c0 + a]);
        const double2 t4 = *reinterpret_cast<const double2*>(&sh.rowA[cur][c0 + a]);
        const double2 t5 = *reinterpret_cast<const double2*>(&sh.rowB[cur][c0 + a]);
        xr[a] = t0.x; xr[a + 1] = t0.y;
        yr[a] = t1.x; yr[a + 1] = t1.y;
        xc[a] = t2.x; xc[a + 1] = t2.y;
        yc[a] = fma(-u, t2.x, t3.x); yc[a + 1] = fma(-u, t2.y, t3.y);   // Y' = Y - u X
        ac[a] = t4.x; ac[a + 1] = t4.y;
        bv[a] = t5.x; bv[a + 1] = t5.y;
      }
#pragma unroll
      for (int a = 0; a < BS; ++a) {
        const double al = xr[a] * ra;                    // X_i / a
        const double be = fma(-u, xr[a], yr[a]) * rd1;  // Y'_i / d1
        const double ga = fma(-be, u, al);                // coefficient of row 2q of V
#pragma unroll
        for (int e = 0; e < BS; ++e) {
          d[a][e] = fma(-al, xc[e], fma(-be, yc[e], d[a][e]));
          v[a][e] = fma(-ga, ac[e], fma(-be, bv[e], v[a][e]));
        }
      }
    }
    if (active && bc == qb) {           // column 2q+1 of L uses Y' = Y - u X
#pragma unroll
      for (int a = 0; a < BS; ++a)
#pragma unroll
        for (int oo = 0; oo < BS; oo += 2)
          if (oo == o) d[a][oo + 1] = fma(-u, d[a][oo], d[a][oo + 1]);
    }
    if (active && br == qb) {           // row 2q+1 of V after its in-block step
#pragma unroll
      for (int e = 0; e < BS; ++e)
#pragma unroll
        for (int oo = 0; oo < BS; oo += 2)
          if (oo == o) v[oo + 1][e] = fma(-u, v[oo][e], v[oo + 1][e]);
    }
    // publish pivot pair q+1 (final after this step) into the other buffer
    const int qn = q + 1;
    if (active && qn < PB / 2) {
      const int qbn = (2 * qn) / BS, on = (2 * qn) % BS;
      if (bc == qbn) {
#pragma unroll
        for (int a = 0; a < BS; ++a) {
          const int row = r0 + a;
          const bool below = row > 2 * qn + 1;
#pragma unroll
          for (int oo = 0; oo < BS; oo += 2)
            if (oo == on) {
              sh.colX[nxt][row] = below ? d[a][oo] : 0.0;
              sh.colY[nxt][row] = below ? d[a][oo + 1] : 0.0;
            }
        }
        if (br == qbn) {
#pragma unroll
          for (int oo = 0; oo < BS; oo += 2)
            if (oo == on) pivot_block(sh.scal[nxt], d[oo][oo], d[oo + 1][oo], d[oo + 1][oo + 1]);
          sh.colX[nxt][2 * q] = sh.colX[nxt][2 * q + 1] = 0.0;   // stale rows of this buffer
          sh.colY[nxt][2 * q] = sh.colY[nxt][2 * q + 1] = 0.0;
        }
      }
      if (br == qbn) {
#pragma unroll
        for (int e = 0; e < BS; ++e)
#pragma unroll
          for (int oo = 0; oo < BS; oo += 2)
            if (oo == on) {
              sh.rowA[nxt][c0 + e] = v[oo][e];
              sh.rowB[nxt][c0 + e] = v[oo + 1][e];
            }
      }
    }
    __syncthreads();
  }

  // L[i][x] = D[i][x] / sqrt(d_x) (x < i), L[x][x] = sqrt(d_x);  Linv[i][x] = V[i][x] / sqrt(d_i)
  if (tid < PB) {
    const double sq = sqrt(sh.pv[tid]);
    sh.colX[0][tid] = sq;
    sh.colY[0][tid] = 1.0 / sq;
  }
  __syncthreads();
  if (active) {
#pragma unroll
    for (int a = 0; a < BS; ++a)
#pragma unroll
      for (int e = 0; e < BS; ++e) {
        const int i = r0 + a, x = c0 + e;
        if (x <= i) {
          D[i * SD + x] = (x == i) ? sh.colX[0][x] : d[a][e] * sh.colY[0][x];
          Li[i * SD + x] = v[a][e] * sh.colY[0][i];
        } else {
          Li[i * SD + x] = 0.0;
        }
        if (bc < br) Li[x * SD + i] = 0.0;   // mirror block above the diagonal
      }
  }
  __syncthreads();
}

// First pivot j < b that is not > 0 (or NaN) -> atomicMin(npd[slot], p + j).  Called by warp 0.
__device__ __forceinline__ void record_npd(const LdltShared& sh, int b, int p, int32_t* npd, int slot) {
  const int lane = threadIdx.x & 31;
  const unsigned lo = __ballot_sync(0xffffffffu, lane < b && !(sh.pv[lane] > 0.0));
  const unsigned hi = __ballot_sync(0xffffffffu, lane + 32 < b && !(sh.pv[lane + 32] > 0.0));
  if (lane == 0 && (lo | hi)) atomicMin(&npd[slot], p + (lo ? __ffs(lo) - 1 : 32 + __ffs(hi) - 1));
}

// ------------------------------------------------------------------ stand-alone DIAG
#ifndef H2G_DIAG_BS
#define H2G_DIAG_BS 2
#endif
constexpr int DIAG_BS = H2G_DIAG_BS;
constexpr int DIAG_THREADS = (Ldlt<DIAG_BS>::NT + 31) / 32 * 32;

__global__ void __launch_bounds__(DIAG_THREADS) potrf_diag_kernel(const h2g_panel_desc* __restrict__ descs,
                                                                  int32_t* __restrict__ npd) {
  extern __shared__ __align__(16) double dsm[];
  double* D = dsm;
  double* Li = dsm + PB * SD;
  LdltShared& sh = *reinterpret_cast<LdltShared*>(dsm + 2 * PB * SD);
  const h2g_panel_desc P = descs[blockIdx.x];
  const int p = P.p, b = P.b, ldh = P.ldh;
  double* H = P.H;
#pragma unroll 4
  for (int t = threadIdx.x; t < PB * PB; t += DIAG_THREADS) {
    const int i = t / PB, x = t % PB;
    const bool v = x <= i && i < b;
    cp_async8(D + i * SD + x, v ? H + (size_t)(p + i) * ldh + p + x : H, v);
  }
  cp_async_commit();
  cp_async_wait<0>();
  __syncthreads();
  diag_ldlt<DIAG_BS>(D, Li, b, sh);
  if (threadIdx.x < 32) record_npd(sh, b, p, npd, P.npd_slot);
  for (int t = threadIdx.x; t < PB * PB; t += blockDim.x) {
    const int i = t / PB, x = t % PB;
    if (x <= i && i < b) H[(size_t)(p + i) * ldh + p + x] = D[i * SD + x];
    P.Linv[(size_t)i * P.ldl + x] = Li[i * SD + x];
  }
}

// ------------------------------------------------------------------ panel step (two kernels)
// Both kernels first apply the previous panel q-1 (columns p-64 .. p-1, final
// L) to their part of block column q:  acc = H[rows, p:p+b] - X[rows] X[p:p+b]^T
// with X = H[:, p-64:p] (K = 64, DMMA; nothing when p == 0).
//   chol_diag_kernel  one CTA per box: rows p .. p+b-1 (the diagonal block),
//                     then factor it: L_pp -> H, L_pp^-1 -> Linv, pivot status.
//   chol_rows_kernel  one CTA per 64-row chunk of the rows below the panel:
//                     its chunk rows, then X_c <- X_c L_pp^-T (DMMA, Linv from
//                     the diag kernel) written back to H.
// Neither reads what the other writes in the same step, so there is no
// intra-launch dependency and no redundant factorization.
constexpr int RW_THREADS = 256;   // 8 warps: 64x64 output, warp tile 32x16

// acc (64x64 block rows `rows(s)`, cols p..p+b) = -H + X[rows] X[p:p+b]^T
// A rows: smem rows arow0 .. arow0+63 of S; B rows: smem rows 0..63 of S.
__device__ __forceinline__ void panel_update_64(double (&acc)[4][2][2], const double* S, int arow0, int warp, int g,
                                                int tq) {
  const int wm = (warp >> 2) & 1, wn = warp & 3;
#pragma unroll 4
  for (int kk = 0; kk < PB; kk += 4) {
    double af[4], bf[2];
#pragma unroll
    for (int i = 0; i < 4; ++i) af[i] = S[(arow0 + wm * 32 + i * 8 + g) * SD + kk + tq];
#pragma unroll
    for (int j = 0; j < 2; ++j) bf[j] = S[(wn * 16 + j * 8 + g) * SD + kk + tq];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 2; ++j) dmma884(acc[i][j], af[i], bf[j]);
  }
}

__global__ void __launch_bounds__(DIAG_THREADS) chol_diag_kernel(const h2g_chol_panel_desc* __restrict__ descs,
                                                                 int32_t* __restrict__ npd) {
  extern __shared__ __align__(16) double csm[];
  double* S = csm;                  // PB x SD: X_{q-1}[p:p+b], then D
  double* Li = csm + PB * SD;       // PB x SD
  LdltShared& sh = *reinterpret_cast<LdltShared*>(csm + 2 * PB * SD);
  const h2g_chol_panel_desc P = descs[blockIdx.x];
  const int p = P.p, b = P.b, ldh = P.ldh;
  double* __restrict__ H = P.H;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, tq = lane & 3;
  const bool gw = warp < 8;
  if (p > 0) {
    const double* src = H + (size_t)p * ldh + (p - PB);
#pragma unroll 4
    for (int t = tid; t < PB * PB; t += DIAG_THREADS) {
      const int s = t / PB, c = t % PB;
      cp_async8(S + s * SD + c, s < b ? src + (size_t)s * ldh + c : H, s < b);
    }
    cp_async_commit();
  }
  double acc[4][2][2];
  const int wm = (warp >> 2) & 1, wn = warp & 3;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int s = wm * 32 + i * 8 + g;
#pragma unroll
    for (int j = 0; j < 2; ++j)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int col = wn * 16 + j * 8 + 2 * tq + e;
        acc[i][j][e] = (gw && s < b && col <= s) ? -H[(size_t)(p + s) * ldh + p + col] : 0.0;
      }
  }
  if (p > 0) {
    cp_async_wait<0>();
    __syncthreads();
    if (gw) panel_update_64(acc, S, 0, warp, g, tq);
    __syncthreads();   // S becomes D
  }
  if (gw) {
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        const int s = wm * 32 + i * 8 + g, col = wn * 16 + j * 8 + 2 * tq;
        S[s * SD + col] = -acc[i][j][0];
        S[s * SD + col + 1] = -acc[i][j][1];
      }
  }
  __syncthreads();
  diag_ldlt<DIAG_BS>(S, Li, b, sh);
  if (tid < 32) record_npd(sh, b, p, npd, P.npd_slot);
  for (int t = tid; t < PB * PB; t += DIAG_THREADS) {
    const int i = t / PB, x = t % PB;
    if (x <= i && i < b) H[(size_t)(p + i) * ldh + p + x] = S[i * SD + x];
    P.Linv[(size_t)i * P.ldl + x] = Li[i * SD + x];
  }
}

__global__ void __launch_bounds__(RW_THREADS, 2) chol_rows_kernel(const h2g_chol_panel_desc* __restrict__ descs,
                                                                  const int32_t* __restrict__ tile_map) {
  extern __shared__ __align__(16) double csm[];
  double* S = csm;                  // 2PB x SD: X_{q-1}[p:p+b] (B), X_{q-1}[chunk] (A), then C
  double* Li = csm + 2 * PB * SD;   // PB x SD: L_pp^-1
  const int pi = tile_map[blockIdx.x];
  const h2g_chol_panel_desc P = descs[pi];
  const int chunk = blockIdx.x - P.tile_start;
  const int p = P.p, b = P.b, n = P.n, ldh = P.ldh;
  double* __restrict__ H = P.H;
  const int row0 = p + b + PB * chunk;
  const int nrows = max(0, min(PB, n - row0));
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, tq = lane & 3;
  PTRACE(0);
  // L_pp^-1 and (p > 0) the previous panel's rows, all copies in flight at once
#pragma unroll 4
  for (int t = tid; t < PB * PB; t += RW_THREADS) {
    const int i = t / PB, x = t % PB;
    cp_async8(Li + i * SD + x, P.Linv + (size_t)i * P.ldl + x, true);
  }
  if (p > 0) {
    const int k0 = p - PB;
#pragma unroll 4
    for (int t = tid; t < 2 * PB * PB; t += RW_THREADS) {
      const int s = t / PB, c = t % PB;
      const int gr = s < PB ? (s < b ? p + s : -1) : (s - PB < nrows ? row0 + s - PB : -1);
      cp_async8(S + s * SD + c, gr >= 0 ? H + (size_t)gr * ldh + k0 + c : H, gr >= 0);
    }
  }
  cp_async_commit();
  double acc[4][2][2];
  const int wm = (warp >> 2) & 1, wn = warp & 3;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int c = wm * 32 + i * 8 + g;
#pragma unroll
    for (int j = 0; j < 2; ++j)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int col = wn * 16 + j * 8 + 2 * tq + e;
        acc[i][j][e] = (c < nrows && col < b) ? -H[(size_t)(row0 + c) * ldh + p + col] : 0.0;
      }
  }
  PTRACE(1);
  cp_async_wait<0>();
  __syncthreads();
  PTRACE(2);
  if (p > 0) panel_update_64(acc, S, PB, warp, g, tq);
  PTRACE(3);
  __syncthreads();   // chunk rows of S become C
  double* C = S + PB * SD;
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      const int c = wm * 32 + i * 8 + g, col = wn * 16 + j * 8 + 2 * tq;
      C[c * SD + col] = -acc[i][j][0];
      C[c * SD + col + 1] = -acc[i][j][1];
    }
  __syncthreads();
  // X_c <- C L_pp^-T
  double out[4][2][2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 2; ++j) out[i][j][0] = out[i][j][1] = 0.0;
#pragma unroll 4
  for (int kk = 0; kk < PB; kk += 4) {
    double af[4], bf[2];
#pragma unroll
    for (int i = 0; i < 4; ++i) af[i] = C[(wm * 32 + i * 8 + g) * SD + kk + tq];
#pragma unroll
    for (int j = 0; j < 2; ++j) bf[j] = Li[(wn * 16 + j * 8 + g) * SD + kk + tq];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 2; ++j) dmma884(out[i][j], af[i], bf[j]);
  }
  PTRACE(4);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int c = wm * 32 + i * 8 + g;
    if (c >= nrows) continue;
    double* dst = H + (size_t)(row0 + c) * ldh + p;
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      const int col = wn * 16 + j * 8 + 2 * tq;
      if (col < b) dst[col] = out[i][j][0];
      if (col + 1 < b) dst[col + 1] = out[i][j][1];
    }
  }
  PTRACE(5);
}

constexpr size_t DIAG_SMEM = (2 * PB * SD) * sizeof(double) + sizeof(LdltShared);
constexpr size_t RW_SMEM = (3 * PB * SD) * sizeof(double);

}  // namespace h2g

extern "C" int h2g_panel_potrf(const h2g_panel_desc* d_descs, int count, int32_t* d_npd, void* stream) {
  if (count <= 0) return H2G_OK;
  if (!d_descs || !d_npd) return h2g_set_error(H2G_EINVAL, "h2g_panel_potrf: null argument");
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(h2g::potrf_diag_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)h2g::DIAG_SMEM);
    attr = true;
  }
  h2g::potrf_diag_kernel<<<count, h2g::DIAG_THREADS, h2g::DIAG_SMEM, (cudaStream_t)stream>>>(d_descs, d_npd);
  return h2g_check_launch("potrf_diag");
}

extern "C" int h2g_chol_panel_tiles(int n, int p, int b) {
  if (b <= 0) return 0;
  const int below = n - p - b;
  return below > 0 ? (below + h2g::PB - 1) / h2g::PB : 0;
}

extern "C" int h2g_chol_panel(const h2g_chol_panel_desc* d_descs, int count, const int32_t* d_tile_map,
                              int total_tiles, int32_t* d_npd, void* stream) {
  if (count <= 0) return H2G_OK;
  if (!d_descs || !d_npd || (total_tiles > 0 && !d_tile_map))
    return h2g_set_error(H2G_EINVAL, "h2g_chol_panel: null argument");
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(h2g::chol_diag_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)h2g::DIAG_SMEM);
    cudaFuncSetAttribute(h2g::chol_rows_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)h2g::RW_SMEM);
    attr = true;
  }
  cudaStream_t st = (cudaStream_t)stream;
  h2g::chol_diag_kernel<<<count, h2g::DIAG_THREADS, h2g::DIAG_SMEM, st>>>(d_descs, d_npd);
  int rc = h2g_check_launch("chol_diag");
  if (rc || total_tiles <= 0) return rc;
  h2g::chol_rows_kernel<<<total_tiles, h2g::RW_THREADS, h2g::RW_SMEM, st>>>(d_descs, d_tile_map);
  return h2g_check_launch("chol_rows");
}
