// Cholesky panels of the batched partial (ULV) Cholesky.
//
// The ULV step of a box is a right-looking Cholesky of H_i = Q_i^T A_ii Q_i
// that stops after r_i pivots: the 64-wide panels factor RR, their rows
// below become L(s)_ii = SR L^-T and the trailing updates of the SS corner
// are the single Schur update SS - L(s) L(s)^T (ulv_factor.py:217-241).
//
// Kernels, all built on one 64x64 factorization routine (diag_blocked):
//
//  chol_diag_kernel +    (h2g_chol_panel) the panel step used by the
//  chol_rows_kernel      factorization, see the section below: together
//                        they apply the previous panel to block column q,
//                        factor its diagonal block and TRSM the rows below,
//                        so the critical lane issues two kernels per panel;
//                        the update of the columns right of the next panel
//                        (REST) is a grouped GEMM on a side lane.
//
//  chol_box_kernel       (h2g_chol_box) the whole partial Cholesky of one box
//                        per CTA, for levels with many boxes.
//  trsm_rows_kernel      (h2g_trsm_rows) V = q_red L^-T, left-looking rows.
//
// A pivot that is not > 0 (or NaN) records atomicMin(npd[slot], p+j): the
// pivot dpotrf reports as info-1 (dense_core.py:60-63).
#include <climits>

#include "common.cuh"

namespace h2g {

#ifdef H2G_PANEL_TRACE
__device__ long long g_panel_trace[32];
#define PTRACE(k) do { if (blockIdx.x == 0 && threadIdx.x == 0) g_panel_trace[k] = clock64(); } while (0)
#else
#define PTRACE(k) do { } while (0)
#endif

constexpr int PB = 64;   // panel width
constexpr int SD = 68;   // smem stride (doubles) of the 64-wide blocks: 68 = 4 mod 16 -> conflict-free fragments

// (DiagShared: scratch of the diagonal factorization, defined after Chol16Shared)

// ------------------------------------------------------------------ blocked 64x64 factorization
// diag_blocked: L in D, L^-1 in Li, pivots in pv, on a short critical path
// (an LDL^T variant with 2x2 pivot steps measured 2x slower; round 1).  The block is split into 16x16
// blocks; each diagonal block is factored by ONE warp entirely in registers
// (lane i owns row i of the block and row i of its inverse; the pivot row is
// broadcast with shuffles, so a pivot step is a shuffle + reciprocal + FMA
// chain with no CTA barrier), and the TRSM of the rows below, the trailing
// update and the off-diagonal blocks of L^-1 are DMMA work spread over the
// CTA's 8 warps.  Rows/cols >= b must already hold the identity.
constexpr int DB = 16;

// 1/d to full double precision without the IEEE division subroutine:
// MUFU.RCP64H seed + two Newton steps.
__device__ __forceinline__ double fast_rcp(double d) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(d));
  // r(1 + e)(1 + e^2) with e = 1 - d r: the second Newton step's residual is
  // e^2, formed beside the first step -> three dependent FP64 ops after the seed
  const double e = fma(-d, r, 1.0);
  const double e2 = e * e;
  r = fma(r, e, r);
  return fma(r, e2, r);
}

// Factor the 16x16 block at blk (lower part read, stride SD) with one warp:
// L -> blk (zeros above the diagonal), L^-1 -> lblk, pivots -> piv[0..15].
// Lanes 0..15 hold row i = lane of the working matrix, lanes 16..31 row
// i = lane - 16 of the inverse V = U^-1 (U unit lower).  Step j broadcasts
// row j of both through a double-buffered shared-memory row (the owners
// store it, __syncwarp, every lane reads it with 128-bit broadcast loads):
// ~20 shared-memory ops per pivot instead of 2 x 34 shuffles.
struct Chol16Shared {
  double row[2][2][DB];   // [buffer][half][column]
  double col[2][DB];      // [buffer][row]: column j of the working matrix
};

struct DiagShared {
  Chol16Shared cs;   // the 16x16 pivot rows / columns
  double pv[PB];     // pivots d_j of the 64x64 block
};

__device__ __forceinline__ void chol16_warp(double* blk, double* lblk, double* piv, Chol16Shared& cs) {
  const int lane = threadIdx.x & 31;
  const int i = lane & 15, half = lane >> 4;
  double x[DB];
#pragma unroll
  for (int k = 0; k < DB; ++k) {
    const double m = k <= i ? blk[i * SD + k] : blk[k * SD + i];   // full symmetric row i
    x[k] = half ? (k == i ? 1.0 : 0.0) : m;
  }
#pragma unroll
  for (int j = 0; j < DB; ++j) {
    const int buf = j & 1;
    if (i == j) {
#pragma unroll
      for (int k = 0; k < DB; k += 2)
        *reinterpret_cast<double2*>(&cs.row[buf][half][k]) = make_double2(x[k], x[k + 1]);
    }
    if (!half) cs.col[buf][i] = x[j];
    __syncwarp();
    const double d = cs.row[buf][0][j];
    const double lj = cs.col[buf][i] * fast_rcp(d);
    const bool act = i > j;
#pragma unroll
    for (int k = 0; k < DB; k += 2) {
      const double2 t = *reinterpret_cast<const double2*>(&cs.row[buf][half][k]);
      if (act && (half ? (k <= j) : (k > j))) x[k] = fma(-lj, t.x, x[k]);
      if (act && (half ? (k + 1 <= j) : (k + 1 > j))) x[k + 1] = fma(-lj, t.y, x[k + 1]);
    }
    if (act && !half) x[j] = lj;           // multiplier l_ij; lane j keeps its pivot d_j in x[j]
  }
  double di = x[0];
#pragma unroll
  for (int k = 1; k < DB; ++k)
    if (k == i) di = x[k];
  if (!half) cs.col[0][i] = di;
  __syncwarp();
  di = cs.col[0][i];
  const double sqi = sqrt(di), rsqi = fast_rcp(sqi);
  if (!half) cs.col[1][i] = sqi;
  __syncwarp();
#pragma unroll
  for (int k = 0; k < DB; ++k) {
    if (!half) blk[i * SD + k] = k < i ? x[k] * cs.col[1][k] : (k == i ? sqi : 0.0);
    else lblk[i * SD + k] = k <= i ? x[k] * rsqi : 0.0;
  }
  if (!half) piv[i] = di;
  __syncwarp();
}

// out(8x8 tile at rows m0, cols n0) = sum_k A[m0+.][k] * B[n0+.][k], k < 16 (A, B smem, stride SD)
__device__ __forceinline__ void tile8_nt16(double (&c)[2], const double* A, const double* B, int g, int tq) {
  c[0] = c[1] = 0.0;
#pragma unroll
  for (int kk = 0; kk < DB; kk += 4) dmma884(c, A[g * SD + kk + tq], B[g * SD + kk + tq]);
}

// NW warps (4 or 8).  D, Li: 64 x SD smem; pv: 64 doubles smem.
// b < 64 (a partial last panel): rows / cols >= b hold the identity, so the 16x16 blocks
// past ceil(b/16) are skipped — they would factor to the identity with zero coupling
// (their Li diagonal blocks are set to I, the off-diagonal blocks stay 0).
template <int NW>
__device__ void diag_blocked(double* D, double* Li, double* pv, Chol16Shared& cs, int b = PB) {
  constexpr int NU = (16 + NW - 1) / NW;   // 8x8 output tiles per warp (<= 12 / 16 tiles per phase)
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, tq = lane & 3;
  const int nb = b >= PB ? PB / DB : max(1, (b + DB - 1) / DB);   // 16x16 blocks with real pivots
  for (int t = tid; t < PB * PB; t += blockDim.x) {
    const int i = t / PB, x = t % PB;
    Li[i * SD + x] = (i == x && i >= nb * DB) ? 1.0 : 0.0;
  }
  __syncthreads();
  PTRACE(16);
#pragma unroll 1
  for (int kb = 0; kb < nb; ++kb) {
    const int c = kb * DB;
    if (warp == 0) chol16_warp(D + c * SD + c, Li + c * SD + c, pv + c, cs);
    __syncthreads();
    PTRACE(17 + 2 * kb);
    const int R = nb * DB - c - DB;            // rows below the block (padding rows stay the identity)
    if (R == 0) break;
    // TRSM: X = D[c+16:, c:c+16] <- X Linv_kk^T; 8x8 output tiles (R/8) x 2
    const int nt = (R / 8) * 2;
    double x[NU][2];
    int tt[NU];
#pragma unroll
    for (int u = 0; u < NU; ++u) {
      tt[u] = warp + NW * u;
      if (tt[u] < nt) {
        const int tm = tt[u] >> 1, tn = tt[u] & 1;
        tile8_nt16(x[u], D + (c + DB + 8 * tm) * SD + c, Li + (c + 8 * tn) * SD + c, g, tq);
      }
    }
    __syncthreads();
#pragma unroll
    for (int u = 0; u < NU; ++u)
      if (tt[u] < nt) {
        const int tm = tt[u] >> 1, tn = tt[u] & 1;
        double* dst = D + (c + DB + 8 * tm + g) * SD + c + 8 * tn + 2 * tq;
        dst[0] = x[u][0];
        dst[1] = x[u][1];
      }
    __syncthreads();
    // trailing update of the lower 8x8 tiles of D[c+16:, c+16:] (K = 16)
    const int T = R / 8, ntile = T * (T + 1) / 2;
    for (int t = warp; t < ntile; t += NW) {
      int tm = 0;
      while ((tm + 1) * (tm + 2) / 2 <= t) ++tm;
      const int tn = t - tm * (tm + 1) / 2;
      double cc[2];
      tile8_nt16(cc, D + (c + DB + 8 * tm) * SD + c, D + (c + DB + 8 * tn) * SD + c, g, tq);
      double* dst = D + (c + DB + 8 * tm + g) * SD + c + DB + 8 * tn + 2 * tq;
      dst[0] -= cc[0];
      dst[1] -= cc[1];
    }
    __syncthreads();
    PTRACE(18 + 2 * kb);
  }
  PTRACE(25);
  // off-diagonal 16x16 blocks of L^-1, by block diagonals dd = 1..3:
  //   Linv_IJ = -Linv_II * (sum_{K=J}^{I-1} L_IK Linv_KJ),  I = J + dd
#pragma unroll 1
  for (int dd = 1; dd < nb; ++dd) {
    const int nblk = nb - dd;                  // blocks on this block diagonal
    // phase 1: W_J = sum_K L_IK Linv_KJ (16x16 each, 4 8x8 tiles) -> registers, then smem scratch
    double w[NU][2];
    int tt[NU];
#pragma unroll
    for (int u = 0; u < NU; ++u) {
      tt[u] = warp + NW * u;
      w[u][0] = w[u][1] = 0.0;
      if (tt[u] < nblk * 4) {
        const int J = tt[u] >> 2, I = J + dd, tm = (tt[u] >> 1) & 1, tn = tt[u] & 1;
        // sum over K = J .. I-1 of L[I,K] (16x16 from D) * Linv[K,J] (16x16 from Li); k runs over K's 16 columns
        for (int K = J; K < I; ++K) {
#pragma unroll
          for (int kk = 0; kk < DB; kk += 4) {
            const double av = D[(I * DB + 8 * tm + g) * SD + K * DB + kk + tq];
            const double bv = Li[(K * DB + kk + tq) * SD + J * DB + 8 * tn + g];
            dmma884(w[u], av, bv);
          }
        }
      }
    }
    __syncthreads();
    // stash W in the (zero) upper part of Li: block (J, I) position holds W_J for pair (I, J)
#pragma unroll
    for (int u = 0; u < NU; ++u)
      if (tt[u] < nblk * 4) {
        const int J = tt[u] >> 2, I = J + dd, tm = (tt[u] >> 1) & 1, tn = tt[u] & 1;
        double* dst = Li + (J * DB + 8 * tm + g) * SD + I * DB + 8 * tn + 2 * tq;
        dst[0] = w[u][0];
        dst[1] = w[u][1];
      }
    __syncthreads();
    // phase 2: Linv_IJ = -Linv_II W
#pragma unroll
    for (int u = 0; u < NU; ++u) {
      w[u][0] = w[u][1] = 0.0;
      if (tt[u] < nblk * 4) {
        const int J = tt[u] >> 2, I = J + dd, tm = (tt[u] >> 1) & 1, tn = tt[u] & 1;
#pragma unroll
        for (int kk = 0; kk < DB; kk += 4) {
          const double av = Li[(I * DB + 8 * tm + g) * SD + I * DB + kk + tq];
          const double bv = Li[(J * DB + kk + tq) * SD + I * DB + 8 * tn + g];
          dmma884(w[u], av, bv);
        }
      }
    }
    __syncthreads();
#pragma unroll
    for (int u = 0; u < NU; ++u)
      if (tt[u] < nblk * 4) {
        const int J = tt[u] >> 2, I = J + dd, tm = (tt[u] >> 1) & 1, tn = tt[u] & 1;
        double* dst = Li + (I * DB + 8 * tm + g) * SD + J * DB + 8 * tn + 2 * tq;
        dst[0] = -w[u][0];
        dst[1] = -w[u][1];
        double* scr = Li + (J * DB + 8 * tm + g) * SD + I * DB + 8 * tn + 2 * tq;   // clear the stash
        scr[0] = scr[1] = 0.0;
      }
    __syncthreads();
  }
  PTRACE(26);
}

// First pivot j < b that is not > 0 (or NaN) -> atomicMin(npd[slot], p + j).  Called by warp 0.
__device__ __forceinline__ void record_npd(const DiagShared& sh, int b, int p, int32_t* npd, int slot) {
  const int lane = threadIdx.x & 31;
  const unsigned lo = __ballot_sync(0xffffffffu, lane < b && !(sh.pv[lane] > 0.0));
  const unsigned hi = __ballot_sync(0xffffffffu, lane + 32 < b && !(sh.pv[lane + 32] > 0.0));
  if (lane == 0 && (lo | hi)) atomicMin(&npd[slot], p + (lo ? __ffs(lo) - 1 : 32 + __ffs(hi) - 1));
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

// NW = 8: latency variant (few boxes); NW = 4: throughput variant (many boxes, more CTAs per SM).
template <int NW>
__device__ __forceinline__ void chol_diag_body(const h2g_chol_panel_desc& P, double* csm, int32_t* __restrict__ npd) {
  constexpr int NT = NW * 32, NV = 8 / NW;   // NV virtual 32x16 warp tiles per warp
  double* S = csm;                  // PB x SD: X_{q-1}[p:p+b], then D
  double* Li = csm + PB * SD;       // PB x SD
  DiagShared& sh = *reinterpret_cast<DiagShared*>(csm + 2 * PB * SD);
  const int p = P.p, b = P.b, ldh = P.ldh;
  double* __restrict__ H = P.H;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, tq = lane & 3;
  if (p > 0) {
    const double* src = H + (size_t)p * ldh + (p - PB);
#pragma unroll 4
    for (int t = tid; t < PB * PB; t += NT) {
      const int s = t / PB, c = t % PB;
      cp_async8(S + s * SD + c, s < b ? src + (size_t)s * ldh + c : H, s < b);
    }
    cp_async_commit();
  }
  double acc[NV][4][2][2];
#pragma unroll
  for (int v = 0; v < NV; ++v) {
    const int vw = warp + NW * v, wm = vw >> 2, wn = vw & 3;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int s = wm * 32 + i * 8 + g;
#pragma unroll
      for (int j = 0; j < 2; ++j)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int col = wn * 16 + j * 8 + 2 * tq + e;
          acc[v][i][j][e] = (s < b && col <= s) ? neg_int(H[(size_t)(p + s) * ldh + p + col]) : 0.0;
        }
    }
  }
  if (p > 0) {
    cp_async_wait<0>();
    __syncthreads();
#pragma unroll
    for (int v = 0; v < NV; ++v) panel_update_64(acc[v], S, 0, warp + NW * v, g, tq);
    __syncthreads();   // S becomes D
  }
#pragma unroll
  for (int v = 0; v < NV; ++v) {
    const int vw = warp + NW * v, wm = vw >> 2, wn = vw & 3;
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        const int s = wm * 32 + i * 8 + g, col = wn * 16 + j * 8 + 2 * tq;
        S[s * SD + col] = neg_int(acc[v][i][j][0]);
        S[s * SD + col + 1] = neg_int(acc[v][i][j][1]);
      }
  }
  __syncthreads();
  if (tid < PB && tid >= b) {   // identity padding beyond the panel width
    for (int x = 0; x < PB; ++x) S[tid * SD + x] = (x == tid) ? 1.0 : 0.0;
  }
  if (NT < PB && tid + NT < PB && tid + NT >= b) {
    const int r = tid + NT;
    for (int x = 0; x < PB; ++x) S[r * SD + x] = (x == r) ? 1.0 : 0.0;
  }
  __syncthreads();
  diag_blocked<NW>(S, Li, sh.pv, sh.cs, b);
  if (tid < 32) record_npd(sh, b, p, npd, P.npd_slot);
  for (int t = tid; t < PB * PB; t += NT) {
    const int i = t / PB, x = t % PB;
    if (x <= i && i < b) H[(size_t)(p + i) * ldh + p + x] = S[i * SD + x];
    P.Linv[(size_t)i * P.ldl + x] = Li[i * SD + x];
  }
}

template <int NW>
__global__ void __launch_bounds__(NW * 32, NW == 8 ? 2 : 3) chol_diag_kernel(const h2g_chol_panel_desc* __restrict__ descs,
                                                                    int32_t* __restrict__ npd) {
  extern __shared__ __align__(16) double csm[];
  const h2g_chol_panel_desc P = descs[blockIdx.x];
  chol_diag_body<NW>(P, csm, npd);
}

__device__ __forceinline__ int chol_row_chunks(const h2g_chol_panel_desc& P) {
  const int below = P.n - P.p - P.b;
  return below > 0 ? (below + PB - 1) / PB : 0;
}

__device__ __forceinline__ int ld_acquire(const int32_t* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release(int32_t* p, int v) {
  asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// FUSED: the diag CTA of the same launch publishes L_pp^-1 through *flag; the
// chunk loads and applies the previous panel first, then waits for it.  The
// last chunk of the box to pass the flag resets flag and counter for the next launch.
template <bool FUSED>
__device__ __forceinline__ void chol_rows_body(const h2g_chol_panel_desc& P, int chunk, double* csm,
                                               int32_t* flag = nullptr, int32_t* cnt = nullptr) {
  double* S = csm;                  // 2PB x SD: X_{q-1}[p:p+b] (B), X_{q-1}[chunk] (A), then C
  double* Li = csm + 2 * PB * SD;   // PB x SD: L_pp^-1
  const int p = P.p, b = P.b, n = P.n, ldh = P.ldh;
  double* __restrict__ H = P.H;
  const int row0 = p + b + PB * chunk;
  const int nrows = max(0, min(PB, n - row0));
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, tq = lane & 3;
  PTRACE(0);
  auto load_li = [&]() {
    if (FUSED) {   // published by the diag CTA during this launch: bypass L1
#pragma unroll 4
      for (int t = tid; t < PB * PB / 2; t += RW_THREADS) {
        const int i = t / (PB / 2), x = 2 * (t % (PB / 2));
        cp_async16_cg(Li + i * SD + x, P.Linv + (size_t)i * P.ldl + x);
      }
    } else {
#pragma unroll 4
      for (int t = tid; t < PB * PB; t += RW_THREADS) {
        const int i = t / PB, x = t % PB;
        cp_async8(Li + i * SD + x, P.Linv + (size_t)i * P.ldl + x, true);
      }
    }
  };
  // L_pp^-1 and (p > 0) the previous panel's rows, all copies in flight at once
  if (!FUSED) load_li();
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
        acc[i][j][e] = (c < nrows && col < b) ? neg_int(H[(size_t)(row0 + c) * ldh + p + col]) : 0.0;
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
      C[c * SD + col] = neg_int(acc[i][j][0]);
      C[c * SD + col + 1] = neg_int(acc[i][j][1]);
    }
  if (FUSED) {
    if (tid == 0) {
      while (ld_acquire(flag) == 0) __nanosleep(64);
      __threadfence();
    }
    __syncthreads();
    load_li();
    cp_async_commit();
    cp_async_wait<0>();
    __syncthreads();
    if (tid == 0 && atomicAdd(cnt, 1) == chol_row_chunks(P) - 1) {
      *cnt = 0;
      *flag = 0;
    }
  } else {
    __syncthreads();
  }
  // X_c <- C L_pp^-T
  double out[4][2][2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 2; ++j) out[i][j][0] = out[i][j][1] = 0.0;
  const int kend = wn * 16 < b ? min(16 * (wn + 1), (b + 3) & ~3) : 0;   // Linv[n][k] = 0 for k > n, k >= b
#pragma unroll 4
  for (int kk = 0; kk < kend; kk += 4) {
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

__global__ void __launch_bounds__(RW_THREADS, 2) chol_rows_kernel(const h2g_chol_panel_desc* __restrict__ descs,
                                                                  const int32_t* __restrict__ tile_map) {
  extern __shared__ __align__(16) double csm[];
  const int pi = tile_map[blockIdx.x];
  const h2g_chol_panel_desc P = descs[pi];
  chol_rows_body<false>(P, blockIdx.x - P.tile_start, csm);
}

// One launch for the whole panel step (few boxes: the step is latency-bound).
// Each CTA takes a ticket: tickets < count factor box `ticket`'s diagonal
// block, the rest are row chunks.  A chunk only waits for diag CTAs that
// already hold their ticket (they are running and wait for nothing), so
// there is no dependence on the hardware's CTA dispatch order.
// sync: [0] ticket counter, [1] finished CTAs, [2, 2+count) flags,
// [2+count, 2+2count) per-box chunk counters; all zero between launches.
__global__ void __launch_bounds__(RW_THREADS, 2) chol_panel_fused_kernel(const h2g_chol_panel_desc* __restrict__ descs,
                                                                         const int32_t* __restrict__ tile_map,
                                                                         int32_t* __restrict__ npd,
                                                                         int32_t* __restrict__ sync, int count,
                                                                         int total) {
  extern __shared__ __align__(16) double csm[];
  __shared__ int ticket;
  if (threadIdx.x == 0) ticket = atomicAdd(&sync[0], 1);
  __syncthreads();
  const int t = ticket;
  int32_t* flag = sync + 2;
  int32_t* cnt = sync + 2 + count;
  if (t < count) {
    const h2g_chol_panel_desc P = descs[t];
    chol_diag_body<8>(P, csm, npd);
    __syncthreads();
    if (threadIdx.x == 0 && chol_row_chunks(P) > 0) {
      __threadfence();
      st_release(flag + t, 1);
    }
  } else {
    const int pi = tile_map[t - count];
    const h2g_chol_panel_desc P = descs[pi];
    chol_rows_body<true>(P, t - count - P.tile_start, csm, flag + pi, cnt + pi);
  }
  if (threadIdx.x == 0 && atomicAdd(&sync[1], 1) == total - 1) {
    sync[0] = 0;
    sync[1] = 0;
  }
}

// ------------------------------------------------------------------ left-looking row solve
// trsm_rows_kernel (h2g_trsm_rows): X = B L^-T, block column by block column,
// for one 64-row chunk of a descriptor.  For panel q in [q_begin, q_end)
// (p = 64q, b = min(64, cols - p)):
//   Xout[rows, p:p+b] = (Xin[rows, p:p+b] - Xout[rows, 0:p] L[p:p+b, 0:p]^T) Linv_q^T
// (A = the already solved columns of the same rows, read back from Xout).
// Xin == NULL stands for the identity (X = L^-T itself, upper triangular:
// only rows < p + b are formed).  The K loop streams 64x32 slices of A and
// of L's row block through a 2-stage cp.async pipeline; the TRSM with the
// panel's 64x64 inverse runs on the accumulators.  One CTA walks all panels
// of its rows, so a whole level's V = q_red L^-T is ONE launch.
constexpr int TS_BK = 32;
constexpr int TS_S = TS_BK + 4;   // 36 = 4 mod 16 doubles: conflict-free fragments

// Shared memory: two stage regions of 2 x (64 x TS_S) doubles each.  The K loop
// ping-pongs between them; the panel's 64x64 inverse is prefetched into the
// region the loop no longer needs (that of tile KT) during the last tile, and
// the accumulators go to the other region after the loop — 74 KB per CTA,
// 3 CTAs per SM.
constexpr int TS_REGION = 2 * PB * TS_S;   // doubles per stage region (>= PB * SD)
static_assert(TS_REGION >= PB * SD, "a stage region must hold a 64 x SD block");

__global__ void __launch_bounds__(RW_THREADS, 3) trsm_rows_kernel(const h2g_rows_desc* __restrict__ descs,
                                                                  const int32_t* __restrict__ tile_map) {
  extern __shared__ __align__(16) double tsm[];
  const int pi = tile_map[blockIdx.x];
  const h2g_rows_desc P = descs[pi];
  const int chunk = blockIdx.x - P.tile_start;
  const int r0 = PB * chunk;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, tq = lane & 3;
  const int wm = warp >> 2, wn = warp & 3;       // warp tile 32 x 16
  const bool ident = P.Xin == nullptr;

#pragma unroll 1
  for (int q = P.q_begin; q < P.q_end; ++q) {
    const int p = PB * q, b = min(PB, P.cols - p), K = p;
    const int nrows = min(PB, (ident ? min(P.rows, p + b) : P.rows) - r0);
    if (b <= 0) break;
    if (nrows <= 0) continue;   // identity: these rows of L^-T start at a later block column
    const double* __restrict__ Lb = P.Lb + (size_t)p * P.ldlb;
    const double* __restrict__ Lq = P.Linv + (size_t)q * PB * PB;
    const int KT = (K + TS_BK - 1) / TS_BK;
    const bool wact = wn * 16 < b;
    double* Li = tsm + (KT & 1) * TS_REGION;          // the region tile KT would use
    double* Cs = tsm + ((KT + 1) & 1) * TS_REGION;    // the region of the last tile
    auto load_li = [&]() {
#pragma unroll 4
      for (int t = tid; t < PB * PB; t += RW_THREADS) {
        const int i = t / PB, x = t % PB;
        cp_async8(Li + i * SD + x, Lq + (size_t)i * PB + x, true);
      }
    };
    auto load_stage = [&](int st, int k0) {
      double* as = tsm + st * TS_REGION;
      double* bs = as + PB * TS_S;
#pragma unroll
      for (int u = 0; u < (PB * TS_BK) / RW_THREADS; ++u) {
        const int idx = tid + u * RW_THREADS;
        const int m = idx / TS_BK, k = idx % TS_BK;
        const bool va = m < nrows && k0 + k < K;
        cp_async8(as + m * TS_S + k, va ? P.Xout + (size_t)(r0 + m) * P.ldx + k0 + k : P.Xout, va);
        const bool vb = m < b && k0 + k < K;
        cp_async8(bs + m * TS_S + k, vb ? Lb + (size_t)m * P.ldlb + k0 + k : Lb, vb);
      }
    };
    if (KT > 0) load_stage(0, 0);
    else load_li();
    cp_async_commit();

    double acc[4][2][2];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 2; ++j)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int m = wm * 32 + i * 8 + g, c = wn * 16 + j * 8 + 2 * tq + e;
          double v = 0.0;
          if (m < nrows && c < b)
            v = ident ? ((r0 + m == p + c) ? 1.0 : 0.0) : P.Xin[(size_t)(r0 + m) * P.ldx + p + c];
          acc[i][j][e] = neg_int(v);
        }
    for (int kt = 0; kt < KT; ++kt) {
      if (kt + 1 < KT) load_stage((kt + 1) & 1, (kt + 1) * TS_BK);
      else load_li();                                  // overlaps the last tile's math
      cp_async_commit();
      cp_async_wait<1>();
      __syncthreads();
      const double* as = tsm + (kt & 1) * TS_REGION;
      const double* bs = as + PB * TS_S;
#pragma unroll
      for (int kk = 0; kk < (wact ? TS_BK : 0); kk += 4) {   // columns >= b of a partial panel: no math
        double af[4], bf[2];
#pragma unroll
        for (int i = 0; i < 4; ++i) af[i] = as[(wm * 32 + i * 8 + g) * TS_S + kk + tq];
#pragma unroll
        for (int j = 0; j < 2; ++j) bf[j] = bs[(wn * 16 + j * 8 + g) * TS_S + kk + tq];
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int j = 0; j < 2; ++j) dmma884(acc[i][j], af[i], bf[j]);
      }
      __syncthreads();
    }
    cp_async_wait<0>();
    __syncthreads();
    // C = Xin - A Lb^T = -acc  ->  smem, then Xout = C Linv^T
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        const int m = wm * 32 + i * 8 + g, c = wn * 16 + j * 8 + 2 * tq;
        Cs[m * SD + c] = neg_int(acc[i][j][0]);
        Cs[m * SD + c + 1] = neg_int(acc[i][j][1]);
      }
    __syncthreads();
    double out[4][2][2];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 2; ++j) out[i][j][0] = out[i][j][1] = 0.0;
    const int kend = wact ? min(16 * (wn + 1), (b + 3) & ~3) : 0;   // Linv[n][k] = 0 for k > n and k >= b
#pragma unroll 4
    for (int kk = 0; kk < kend; kk += 4) {
      double af[4], bf[2];
#pragma unroll
      for (int i = 0; i < 4; ++i) af[i] = Cs[(wm * 32 + i * 8 + g) * SD + kk + tq];
#pragma unroll
      for (int j = 0; j < 2; ++j) bf[j] = Li[(wn * 16 + j * 8 + g) * SD + kk + tq];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 2; ++j) dmma884(out[i][j], af[i], bf[j]);
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int m = wm * 32 + i * 8 + g;
      if (m >= nrows) continue;
      double* dst = P.Xout + (size_t)(r0 + m) * P.ldx + p;
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        const int c = wn * 16 + j * 8 + 2 * tq;
        if (c < b) dst[c] = out[i][j][0];
        if (c + 1 < b) dst[c + 1] = out[i][j][1];
      }
    }
    __syncthreads();   // the next panel reads these columns back (and reuses the regions)
  }
}


// ------------------------------------------------------------------ fused per-box partial Cholesky
// chol_box_kernel (h2g_chol_box): ONE CTA factors one box's H completely —
// the whole ULV elimination of the box (ulv_factor.py:217-241) in one
// kernel: for every 64-column panel q of RR, left-looking,
//   diag:   D = H[p:p+b, p:p+b] - L[p:p+b, 0:p] L[p:p+b, 0:p]^T  (DMMA)
//           -> L_qq (blocked 64x64 factorization, diag_blocked) and L_qq^-1,
//              pivot status (NotPositiveDefiniteError contract)
//   rows:   for every 64-row chunk below (the rest of RR and all SR rows)
//           L[c, p:p+b] = (H[c, p:p+b] - L[c, 0:p] L[p:p+b, 0:p]^T) L_qq^-T
// then the single Schur update SS -= L(s) L(s)^T (lower 64x64 tiles, K = r).
// No trailing matrix is ever written back (left-looking), so a box costs one
// read of its block columns per panel and no inter-CTA synchronisation; the
// latency of the 64-pivot chains is hidden by the other boxes' CTAs on the
// SM (3 per SM).  Used for levels with many boxes (the leaf of N = 1M has
// 4096), where a launch per panel step leaves the SMs waiting on the chain.
// Shared memory: the two stage regions of trsm_rows (74 KB); the diagonal
// factorization puts D in region 0 (+ its pivots / 16x16 scratch in the
// region's spare tail) and L_qq^-1 in region 1.
constexpr int CB_PV = PB * SD;                  // pivots after D in region 0
constexpr int CB_CS = CB_PV + PB;               // Chol16Shared after the pivots
static_assert(CB_CS + (int)(sizeof(Chol16Shared) / sizeof(double)) <= TS_REGION, "diag scratch must fit region 0");

// acc (64 x 64, warp tile 32 x 16 at (wm, wn)) += A[0:arows, 0:K] B[0:brows, 0:K]^T, operands row-major in
// global memory (lda / ldb), streamed through the two stage regions in 64 x 32 slices.  Leaves both
// regions free (ends with a barrier).
__device__ __forceinline__ void cb_gemm_nt(double (&acc)[4][2][2], const double* __restrict__ A, int lda, int arows,
                                           const double* __restrict__ B, int ldb, int brows, int K, double* tsm,
                                           bool wact) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, tq = lane & 3;
  const int wm = warp >> 2, wn = warp & 3;
  const int KT = (K + TS_BK - 1) / TS_BK;
  auto load_stage = [&](int st, int k0) {
    double* as = tsm + st * TS_REGION;
    double* bs = as + PB * TS_S;
#pragma unroll
    for (int u = 0; u < (PB * TS_BK) / RW_THREADS; ++u) {
      const int idx = tid + u * RW_THREADS;
      const int m = idx / TS_BK, k = idx % TS_BK;
      const bool va = m < arows && k0 + k < K;
      cp_async8(as + m * TS_S + k, va ? A + (size_t)m * lda + k0 + k : A, va);
      const bool vb = m < brows && k0 + k < K;
      cp_async8(bs + m * TS_S + k, vb ? B + (size_t)m * ldb + k0 + k : B, vb);
    }
  };
  if (KT > 0) load_stage(0, 0);
  cp_async_commit();
  for (int kt = 0; kt < KT; ++kt) {
    if (kt + 1 < KT) load_stage((kt + 1) & 1, (kt + 1) * TS_BK);
    cp_async_commit();
    cp_async_wait<1>();
    __syncthreads();
    const double* as = tsm + (kt & 1) * TS_REGION;
    const double* bs = as + PB * TS_S;
#pragma unroll
    for (int kk = 0; kk < (wact ? TS_BK : 0); kk += 4) {
      double af[4], bf[2];
#pragma unroll
      for (int i = 0; i < 4; ++i) af[i] = as[(wm * 32 + i * 8 + g) * TS_S + kk + tq];
#pragma unroll
      for (int j = 0; j < 2; ++j) bf[j] = bs[(wn * 16 + j * 8 + g) * TS_S + kk + tq];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 2; ++j) dmma884(acc[i][j], af[i], bf[j]);
    }
    __syncthreads();
  }
  cp_async_wait<0>();
  __syncthreads();
}

// acc = -X[0:rows, 0:cols] (ld ldx): the K loop then accumulates +A B^T, the result is -acc
__device__ __forceinline__ void cb_load_neg(double (&acc)[4][2][2], const double* X, int ldx, int rows, int cols) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = lane >> 2, tq = lane & 3, wm = warp >> 2, wn = warp & 3;
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 2; ++j)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int m = wm * 32 + i * 8 + g, c = wn * 16 + j * 8 + 2 * tq + e;
        acc[i][j][e] = (m < rows && c < cols) ? neg_int(X[(size_t)m * ldx + c]) : 0.0;
      }
}

__device__ __forceinline__ void cb_store_neg(const double (&acc)[4][2][2], double* S, int lds) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = lane >> 2, tq = lane & 3, wm = warp >> 2, wn = warp & 3;
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      const int m = wm * 32 + i * 8 + g, c = wn * 16 + j * 8 + 2 * tq;
      S[m * lds + c] = neg_int(acc[i][j][0]);
      S[m * lds + c + 1] = neg_int(acc[i][j][1]);
    }
}

__global__ void __launch_bounds__(RW_THREADS, 3) chol_box_kernel(const h2g_cholbox_desc* __restrict__ descs,
                                                                 int32_t* __restrict__ npd) {
  extern __shared__ __align__(16) double tsm[];
  const h2g_cholbox_desc P = descs[blockIdx.x];
  const int n = P.n, r = P.r, ld = P.ldh;
  double* __restrict__ H = P.H;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, tq = lane & 3, wm = warp >> 2, wn = warp & 3;
  double* R0 = tsm;
  double* R1 = tsm + TS_REGION;
  bool bad = false;
  const int nq = (r + PB - 1) / PB;
#pragma unroll 1
  for (int q = 0; q < nq; ++q) {
    const int p = PB * q, b = min(PB, r - p);
    double* Hp = H + (size_t)p * ld;          // rows p.., column 0
    double acc[4][2][2];
    // ---- diagonal block: D = H[p:p+b, p:p+b] - L[p:p+b, 0:p] L[p:p+b, 0:p]^T
    cb_load_neg(acc, Hp + p, ld, b, b);
    cb_gemm_nt(acc, Hp, ld, b, Hp, ld, b, p, tsm, true);
    cb_store_neg(acc, R0, SD);
    __syncthreads();
    if (tid < PB && tid >= b) {
      for (int x = 0; x < PB; ++x) R0[tid * SD + x] = (x == tid) ? 1.0 : 0.0;   // identity padding
    }
    __syncthreads();
    double* pv = R0 + CB_PV;
    diag_blocked<8>(R0, R1, pv, *reinterpret_cast<Chol16Shared*>(R0 + CB_CS), b);
    if (warp == 0) {
      const unsigned lo = __ballot_sync(0xffffffffu, lane < b && !(pv[lane] > 0.0));
      const unsigned hi = __ballot_sync(0xffffffffu, lane + 32 < b && !(pv[lane + 32] > 0.0));
      if (lane == 0 && (lo | hi) && !bad) atomicMin(&npd[P.npd_slot], p + (lo ? __ffs(lo) - 1 : 32 + __ffs(hi) - 1));
      bad = bad || (lo | hi);
    }
    double* Lq = P.Linv + (size_t)q * PB * PB;
    for (int t = tid; t < PB * PB; t += RW_THREADS) {
      const int i = t / PB, x = t % PB;
      if (x <= i && i < b) Hp[(size_t)i * ld + p + x] = R0[i * SD + x];
      Lq[(size_t)i * PB + x] = R1[i * SD + x];
    }
    __syncthreads();
    // ---- row chunks below the diagonal block (rest of RR, then all SR rows) and, with P.Q, the rows
    // of V = q_red L^-T (diag_trsm, ulv_factor.py:223-234): the same left-looking step
    //   out[c, p:p+b] = (X[c, p:p+b] - Y[c, 0:p] L[p:p+b, 0:p]^T) L_qq^-T
    // with (X, Y, out) = (H, L, L) for the rows of H and (Q, V, V) for the rows of V
    const bool wact = wn * 16 < b;
    const int kend = wact ? min(16 * (wn + 1), (b + 3) & ~3) : 0;   // Linv[n][k] = 0 for k > n, k >= b
    const int nv = P.Q ? n : 0;                   // rows of V formed by this CTA
    const int c_begin = p + b, n_chunks = (n - c_begin + PB - 1) / PB + (nv + PB - 1) / PB;
#pragma unroll 1
    for (int t = 0; t < n_chunks; ++t) {
      const int th = (n - c_begin + PB - 1) / PB;
      const bool vrow = t >= th;
      const int c0 = vrow ? PB * (t - th) : c_begin + PB * t;
      const int rows = min(PB, (vrow ? nv : n) - c0);
      double* Y = (vrow ? P.R : H) + (size_t)c0 * ld;                 // solved columns 0..p of these rows
      const double* X = (vrow ? P.Q : H) + (size_t)c0 * ld + p;       // right-hand side block
      cb_load_neg(acc, X, ld, rows, b);
      cb_gemm_nt(acc, Y, ld, rows, Hp, ld, b, p, tsm, wact);
      // L_qq^-1 (written above by this CTA; .cg reads it from L2) -> R1, C = -acc -> R0
#pragma unroll 4
      for (int e = tid; e < PB * PB / 2; e += RW_THREADS) {
        const int i = e / (PB / 2), x = 2 * (e % (PB / 2));
        cp_async16_cg(R1 + i * SD + x, Lq + (size_t)i * PB + x);
      }
      cp_async_commit();
      cb_store_neg(acc, R0, SD);
      cp_async_wait<0>();
      __syncthreads();
      double out[4][2][2];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 2; ++j) out[i][j][0] = out[i][j][1] = 0.0;
#pragma unroll 4
      for (int kk = 0; kk < kend; kk += 4) {
        double af[4], bf[2];
#pragma unroll
        for (int i = 0; i < 4; ++i) af[i] = R0[(wm * 32 + i * 8 + g) * SD + kk + tq];
#pragma unroll
        for (int j = 0; j < 2; ++j) bf[j] = R1[(wn * 16 + j * 8 + g) * SD + kk + tq];
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int j = 0; j < 2; ++j) dmma884(out[i][j], af[i], bf[j]);
      }
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int m = wm * 32 + i * 8 + g;
        if (m >= rows) continue;
        double* dst = Y + (size_t)m * ld + p;
#pragma unroll
        for (int j = 0; j < 2; ++j) {
          const int c = wn * 16 + j * 8 + 2 * tq;
          if (c < b) dst[c] = out[i][j][0];
          if (c + 1 < b) dst[c + 1] = out[i][j][1];
        }
      }
      __syncthreads();   // R0 / R1 are reused by the next chunk
    }
  }
  // ---- the single Schur update SS -= L(s) L(s)^T (lower 64 x 64 tiles of the k x k corner, K = r)
  const int k = n - r;
  if (r > 0 && k > 0) {
    const int T = (k + PB - 1) / PB;
#pragma unroll 1
    for (int t = 0; t < T * (T + 1) / 2; ++t) {
      const int ti = tri_row(t), tj = t - ti * (ti + 1) / 2;
      const int rows = min(PB, k - PB * ti), cols = min(PB, k - PB * tj);
      double* A = H + (size_t)(r + PB * ti) * ld;
      double* B = H + (size_t)(r + PB * tj) * ld;
      double* C = A + r + PB * tj;
      double acc[4][2][2];
      cb_load_neg(acc, C, ld, rows, cols);
      cb_gemm_nt(acc, A, ld, rows, B, ld, cols, r, tsm, true);
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int m = wm * 32 + i * 8 + g;
        if (m >= rows) continue;
#pragma unroll
        for (int j = 0; j < 2; ++j) {
          const int c = wn * 16 + j * 8 + 2 * tq;
          if (c < cols) C[(size_t)m * ld + c] = neg_int(acc[i][j][0]);
          if (c + 1 < cols) C[(size_t)m * ld + c + 1] = neg_int(acc[i][j][1]);
        }
      }
    }
  }
}

constexpr size_t TS_SMEM = (2 * TS_REGION) * sizeof(double);

constexpr size_t DIAG_SMEM = (2 * PB * SD) * sizeof(double) + sizeof(DiagShared);
constexpr size_t RW_SMEM = (3 * PB * SD) * sizeof(double);
constexpr size_t FUSED_SMEM = RW_SMEM > DIAG_SMEM ? RW_SMEM : DIAG_SMEM;

}  // namespace h2g

extern "C" int h2g_chol_panel_tiles(int n, int p, int b) {
  if (b <= 0) return 0;
  const int below = n - p - b;
  return below > 0 ? (below + h2g::PB - 1) / h2g::PB : 0;
}

extern "C" int h2g_chol_panel_fused_max(void) {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("H2G_PANEL_FUSED_MAX");
    v = e ? atoi(e) : 128;
  }
  return v;
}

extern "C" int h2g_chol_panel(const h2g_chol_panel_desc* d_descs, int count, const int32_t* d_tile_map,
                              int total_tiles, int32_t* d_npd, void* stream) {
  return h2g_chol_panel_sync(d_descs, count, d_tile_map, total_tiles, d_npd, nullptr, stream);
}

extern "C" int h2g_chol_panel_sync(const h2g_chol_panel_desc* d_descs, int count, const int32_t* d_tile_map,
                                   int total_tiles, int32_t* d_npd, int32_t* d_sync, void* stream) {
  if (count <= 0) return H2G_OK;
  if (!d_descs || !d_npd || (total_tiles > 0 && !d_tile_map))
    return h2g_set_error(H2G_EINVAL, "h2g_chol_panel: null argument");
  // function attributes are per device; so is the SM count (the current device, not device 0)
  static int attr_dev = -1, sms = 0;
  int dev = 0;
  cudaGetDevice(&dev);
  if (attr_dev != dev) {
    cudaFuncSetAttribute(h2g::chol_diag_kernel<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)h2g::DIAG_SMEM);
    cudaFuncSetAttribute(h2g::chol_diag_kernel<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)h2g::DIAG_SMEM);
    cudaFuncSetAttribute(h2g::chol_rows_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)h2g::RW_SMEM);
    cudaFuncSetAttribute(h2g::chol_panel_fused_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)h2g::FUSED_SMEM);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    attr_dev = dev;
  }
  cudaStream_t st = (cudaStream_t)stream;
  if (d_sync && total_tiles > 0 && count <= h2g_chol_panel_fused_max()) {
    h2g::chol_panel_fused_kernel<<<count + total_tiles, h2g::RW_THREADS, h2g::FUSED_SMEM, st>>>(
        d_descs, d_tile_map, d_npd, d_sync, count, count + total_tiles);
    return h2g_check_launch("chol_panel_fused");
  }
  // many boxes: the 4-warp variant fits 3 CTAs per SM (throughput); few boxes: 8 warps (latency)
  if (count >= 2 * sms) h2g::chol_diag_kernel<4><<<count, 128, h2g::DIAG_SMEM, st>>>(d_descs, d_npd);
  else h2g::chol_diag_kernel<8><<<count, 256, h2g::DIAG_SMEM, st>>>(d_descs, d_npd);
  int rc = h2g_check_launch("chol_diag");
  if (rc || total_tiles <= 0) return rc;
  h2g::chol_rows_kernel<<<total_tiles, h2g::RW_THREADS, h2g::RW_SMEM, st>>>(d_descs, d_tile_map);
  return h2g_check_launch("chol_rows");
}

extern "C" int h2g_chol_box(const h2g_cholbox_desc* d_descs, int count, int32_t* d_npd, void* stream) {
  if (count <= 0) return H2G_OK;
  if (!d_descs || !d_npd) return h2g_set_error(H2G_EINVAL, "h2g_chol_box: null argument");
  static int attr_dev = -1;
  int dev = 0;
  cudaGetDevice(&dev);
  if (attr_dev != dev) {
    cudaFuncSetAttribute(h2g::chol_box_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)h2g::TS_SMEM);
    attr_dev = dev;
  }
  h2g::chol_box_kernel<<<count, h2g::RW_THREADS, h2g::TS_SMEM, (cudaStream_t)stream>>>(d_descs, d_npd);
  return h2g_check_launch("chol_box");
}

extern "C" int h2g_trsm_rows(const h2g_rows_desc* d_descs, const int32_t* d_tile_map, int total_tiles, void* stream) {
  if (total_tiles <= 0) return H2G_OK;
  if (!d_descs || !d_tile_map) return h2g_set_error(H2G_EINVAL, "h2g_trsm_rows: null argument");
  static int attr_dev = -1;
  int dev = 0;
  cudaGetDevice(&dev);
  if (attr_dev != dev) {
    cudaFuncSetAttribute(h2g::trsm_rows_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)h2g::TS_SMEM);
    attr_dev = dev;
  }
  h2g::trsm_rows_kernel<<<total_tiles, h2g::RW_THREADS, h2g::TS_SMEM, (cudaStream_t)stream>>>(d_descs, d_tile_map);
  return h2g_check_launch("trsm_rows");
}
