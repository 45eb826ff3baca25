// Grouped FP64 GEMM on the sm_100a FP64 tensor pipe (DMMA.8x8x4).
//
// One CTA computes one 64x64 tile of one problem; the tile -> problem map
// is precomputed on the host so a level's whole phase (every box or every
// near pair, all different sizes) is ONE launch with no padding beyond the
// tile edge.  Operands are staged global -> shared with 3-stage cp.async;
// the smem layout per operand depends on its transpose so both the global
// reads (coalesced along the contiguous axis) and the fragment reads (bank
// conflict free: stride = 4 mod 16 doubles) are clean.
//
// Reference phases this serves: diag_mul1/2, off_mul1/2, the Schur update
// and the TRSM trailing updates (ulv_factor.py:189-259; the flop model is
// dense_core.flop_count, dense_core.py:166-181).
#include "common.cuh"

namespace h2g {

constexpr int BM = 64, BN = 64, BK = 16, STAGES = 3, THREADS = 128;
constexpr int S_MK = BK + 4;   // row stride when the m (or n) index is outer
constexpr int S_KM = BM + 4;   // row stride when the k index is outer
constexpr int TILE_DBL = (BM * S_MK > BK * S_KM) ? BM * S_MK : BK * S_KM;  // 1280
constexpr int GEMM_SMEM = 2 * STAGES * TILE_DBL * 8;

template <bool TA, bool TB>
__global__ void __launch_bounds__(THREADS) gemm_grouped_kernel(const h2g_gemm_problem* __restrict__ probs,
                                                               const int32_t* __restrict__ tile_map) {
  extern __shared__ __align__(16) double smem[];
  double* As = smem;
  double* Bs = smem + STAGES * TILE_DBL;

  const int tile = blockIdx.x;
  const int pi = tile_map[tile];
  const h2g_gemm_problem P = probs[pi];
  int t = tile - P.tile_start;
  int tm, tn;
  if (P.flags & H2G_GEMM_LOWER) {
    // lower-triangular tile enumeration: t -> (tm, tn), tn <= tm
    int i = (int)((sqrt(8.0 * t + 1.0) - 1.0) * 0.5);
    while ((i + 1) * (i + 2) / 2 <= t) ++i;
    while (i * (i + 1) / 2 > t) --i;
    tm = i;
    tn = t - i * (i + 1) / 2;
  } else {
    int ntn = (P.N + BN - 1) / BN;
    tm = t / ntn;
    tn = t - tm * ntn;
  }
  const int m0 = tm * BM, n0 = tn * BN;
  const int M = P.M, N = P.N, K = P.K;
  const double* __restrict__ A = P.A;
  const double* __restrict__ B = P.B;
  const int lda = P.lda, ldb = P.ldb;

  const int tid = threadIdx.x;
  const int lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, tq = lane & 3;
  const int wm = warp & 1, wn = warp >> 1;

  auto load_stage = [&](int stage, int k0) {
    double* as = As + stage * TILE_DBL;
    double* bs = Bs + stage * TILE_DBL;
#pragma unroll
    for (int j = 0; j < (BM * BK) / THREADS; ++j) {
      int idx = tid + j * THREADS;
      if (!TA) {  // A[m][k] contiguous in k -> As[m][k]
        int m = idx / BK, k = idx % BK;
        int gm = m0 + m, gk = k0 + k;
        bool v = gm < M && gk < K;
        cp_async8(as + m * S_MK + k, v ? A + (size_t)gm * lda + gk : A, v);
      } else {    // A stored K x M, contiguous in m -> As[k][m]
        int k = idx / BM, m = idx % BM;
        int gm = m0 + m, gk = k0 + k;
        bool v = gm < M && gk < K;
        cp_async8(as + k * S_KM + m, v ? A + (size_t)gk * lda + gm : A, v);
      }
      if (!TB) {  // B[k][n] contiguous in n -> Bs[k][n]
        int k = idx / BN, n = idx % BN;
        int gn = n0 + n, gk = k0 + k;
        bool v = gn < N && gk < K;
        cp_async8(bs + k * S_KM + n, v ? B + (size_t)gk * ldb + gn : B, v);
      } else {    // B stored N x K, contiguous in k -> Bs[n][k]
        int n = idx / BK, k = idx % BK;
        int gn = n0 + n, gk = k0 + k;
        bool v = gn < N && gk < K;
        cp_async8(bs + n * S_MK + k, v ? B + (size_t)gn * ldb + gk : B, v);
      }
    }
  };

  double acc[4][4][2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

  const int KT = (K + BK - 1) / BK;
#pragma unroll
  for (int s = 0; s < STAGES - 1; ++s) {
    if (s < KT) load_stage(s, s * BK);
    cp_async_commit();
  }

  for (int kt = 0; kt < KT; ++kt) {
    cp_async_wait<STAGES - 2>();
    __syncthreads();
    {
      int nk = kt + STAGES - 1;
      if (nk < KT) load_stage(nk % STAGES, nk * BK);
      cp_async_commit();
    }
    const double* as = As + (kt % STAGES) * TILE_DBL;
    const double* bs = Bs + (kt % STAGES) * TILE_DBL;
#pragma unroll
    for (int kk = 0; kk < BK; kk += 4) {
      double af[4], bf[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        int m = wm * 32 + i * 8 + g, k = kk + tq;
        af[i] = TA ? as[k * S_KM + m] : as[m * S_MK + k];
      }
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        int n = wn * 32 + j * 8 + g, k = kk + tq;
        bf[j] = TB ? bs[n * S_MK + k] : bs[k * S_KM + n];
      }
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) dmma884(acc[i][j], af[i], bf[j]);
    }
  }
  cp_async_wait<0>();

  // epilogue: C = alpha*acc + beta*C
  double* C = P.C;  // may alias A (in-place TRSM with N <= 64)
  const int ldc = P.ldc;
  const double alpha = P.alpha, beta = P.beta;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    int row = m0 + wm * 32 + i * 8 + g;
    if (row >= M) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      int col = n0 + wn * 32 + j * 8 + 2 * tq;
      double* cp = C + (size_t)row * ldc + col;
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        if (col + e < N) {
          double v = alpha * acc[i][j][e];
          if (beta != 0.0) v += beta * cp[e];
          cp[e] = v;
        }
      }
    }
  }
}

template <bool TA, bool TB>
static int launch_gemm(const h2g_gemm_problem* d_probs, const int32_t* d_map, int tiles, cudaStream_t s) {
  static bool attr_set = false;
  if (!attr_set) {
    cudaFuncSetAttribute(gemm_grouped_kernel<TA, TB>, cudaFuncAttributeMaxDynamicSharedMemorySize, GEMM_SMEM);
    attr_set = true;
  }
  gemm_grouped_kernel<TA, TB><<<tiles, THREADS, GEMM_SMEM, s>>>(d_probs, d_map);
  return h2g_check_launch("gemm_grouped");
}

}  // namespace h2g

extern "C" int h2g_gemm_tiles(int M, int N, int flags) {
  if (M <= 0 || N <= 0) return 0;
  if (flags & H2G_GEMM_LOWER) {
    int t = (M + h2g::BM - 1) / h2g::BM;
    return t * (t + 1) / 2;
  }
  return ((M + h2g::BM - 1) / h2g::BM) * ((N + h2g::BN - 1) / h2g::BN);
}

extern "C" int h2g_gemm_grouped(int trans_a, int trans_b, const h2g_gemm_problem* d_probs,
                                const int32_t* d_tile_map, int total_tiles, void* stream) {
  if (total_tiles <= 0) return H2G_OK;
  if (!d_probs || !d_tile_map) return h2g_set_error(H2G_EINVAL, "h2g_gemm_grouped: null descriptor");
  cudaStream_t s = (cudaStream_t)stream;
  if (!trans_a && !trans_b) return h2g::launch_gemm<false, false>(d_probs, d_tile_map, total_tiles, s);
  if (!trans_a && trans_b) return h2g::launch_gemm<false, true>(d_probs, d_tile_map, total_tiles, s);
  if (trans_a && !trans_b) return h2g::launch_gemm<true, false>(d_probs, d_tile_map, total_tiles, s);
  return h2g::launch_gemm<true, true>(d_probs, d_tile_map, total_tiles, s);
}
