// Grouped FP64 GEMM on the sm_100a FP64 tensor pipe (DMMA.8x8x4).
//
// One CTA computes one BMxBN tile of one problem; the tile -> problem map is
// precomputed on the host so a level's whole phase (every box or every near
// pair, all different sizes) is ONE launch with no padding beyond the tile
// edge.  Tile shapes: 64x64 with 4 warps (32x32 warp tiles; cfg 2 at 4 CTAs/SM,
// cfg 7 at 3 CTAs/SM) and 32x32 (cfg 9) for ragged small problems.
// Operands are staged global -> shared with 2-stage cp.async; the smem layout
// per operand follows its transpose so both the global reads (coalesced
// along the contiguous axis) and the fragment reads (stride = 4 mod 16
// doubles: bank-conflict free) are clean.  With beta != 0 the C tile is read
// into the accumulators before the main loop (its latency overlaps the
// operand prologue), which matters for the K = 64 Cholesky updates.
//
// Reference phases this serves: diag_mul1/2, off_mul1/2, the Schur update
// and the TRSM/trailing updates (ulv_factor.py:189-259; the flop model is
// dense_core.flop_count, dense_core.py:166-181).
#include "common.cuh"

namespace h2g {

constexpr int BK = 16;

template <int BM, int BN, int WARPS_M, int WARPS_N, int MIN_CTAS, int NSTAGE>
struct GemmCfg {
  static constexpr int TBM = BM, TBN = BN, NWARP_N = WARPS_N, MIN_BLOCKS = MIN_CTAS, STAGES = NSTAGE;
  static constexpr int THREADS = WARPS_M * WARPS_N * 32;
  static constexpr int WM = BM / WARPS_M, WN = BN / WARPS_N;   // warp tile
  static constexpr int MI = WM / 8, NI = WN / 8;                // 8x8 sub-tiles per warp
  static constexpr int S_MK = BK + 4;                           // stride, m/n outer
  static constexpr int SA_KM = BM + 4, SB_KN = BN + 4;          // stride, k outer
  static constexpr int A_DBL = (BM * S_MK > BK * SA_KM) ? BM * S_MK : BK * SA_KM;
  static constexpr int B_DBL = (BN * S_MK > BK * SB_KN) ? BN * S_MK : BK * SB_KN;
  static constexpr int SMEM = STAGES * (A_DBL + B_DBL) * 8;
};

// The three configurations the planner chooses from (program.choose_tile_cfg; tile shapes,
// stage counts and the m16n8k16 variant measured in profiles/r01_gemm_tile_configs*.jsonl):
#ifndef H2G_GEMM_STAGES
#define H2G_GEMM_STAGES 2
#endif
using Cfg64b = GemmCfg<64, 64, 2, 2, 4, H2G_GEMM_STAGES>;   // cfg 2: 4 CTAs/SM, <= 128 registers (transforms)
using Cfg64m3 = GemmCfg<64, 64, 2, 2, 3, 2>;    // cfg 7: 3 CTAs/SM (170 registers), 2 stages (K <= 64 updates)
using Cfg32 = GemmCfg<32, 32, 2, 2, 6, 2>;      // cfg 9: small / ragged problems, 32x32 tiles, 6 CTAs/SM
using Cfg64w8 = GemmCfg<64, 64, 2, 4, 3, 2>;    // cfg 11: 8 warps (32x16 warp tiles), EXT launches only (A/B)

// EXT: per-problem extension (h2g_gemm_ext): the beta term read from a separate Cin and, with
// remap_k >= 0, the compact-WY relabel epilogue of the diag transform (see h2g_gemm_grouped_ext).
// SPLIT: deterministic split-K for launches under one wave (few-box upper levels): every tile
// is nsplit consecutive CTAs, CTA s of a tile accumulates K range s (BK-aligned), writes its
// partial tile to ws, and the last CTA to arrive (per-tile counter) sums the partials in the
// fixed order 0..nsplit-1, adds the beta term and stores C — the same result whatever the
// arrival order.  ws = [tiles int32 counters, zero between launches | 256 B align | partials].
template <class C, bool TA, bool TB, bool EXT = false, bool SPLIT = false>
__global__ void __launch_bounds__(C::THREADS, C::MIN_BLOCKS) gemm_grouped_kernel(const h2g_gemm_problem* __restrict__ probs,
                                                                  const int32_t* __restrict__ tile_map,
                                                                  const h2g_gemm_ext* __restrict__ ext = nullptr,
                                                                  double* __restrict__ ws = nullptr,
                                                                  int nsplit = 1, int ntiles = 0) {
  extern __shared__ __align__(16) double smem[];
  double* As = smem;
  double* Bs = smem + C::STAGES * C::A_DBL;
  constexpr int tBM = C::TBM, tBN = C::TBN, wn_count = C::NWARP_N;

  const int tile = blockIdx.x;
  const int pi = tile_map[tile];
  const h2g_gemm_problem P = probs[pi];
  int t = tile - P.tile_start;
  int split = 0;
  if constexpr (SPLIT) {
    split = t % nsplit;
    t /= nsplit;
  }
  int tm, tn;
  if (P.flags & H2G_GEMM_LOWER) {
    const int i = tri_row(t);
    tm = i;
    tn = t - i * (i + 1) / 2;
  } else {
    int ntn = (P.N + tBN - 1) / tBN;
    tm = t / ntn;
    tn = t - tm * ntn;
  }
  const int m0 = tm * tBM, n0 = tn * tBN;
  const int M = P.M, N = P.N, K = P.K;
  int kbeg = 0, kend = K;
  if constexpr (SPLIT) {
    const int ks = ((K + nsplit - 1) / nsplit + BK - 1) / BK * BK;
    kbeg = min(K, split * ks);
    kend = min(K, kbeg + ks);
  }
  const double* __restrict__ A = P.A;
  const double* __restrict__ B = P.B;
  const int lda = P.lda, ldb = P.ldb;

  const int tid = threadIdx.x;
  const int lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, tq = lane & 3;
  const int wm = warp / wn_count, wn = warp % wn_count;
  // a warp tile strictly above the diagonal of a LOWER diagonal tile is never read: skip its math
  const bool upper_warp = (P.flags & H2G_GEMM_LOWER) && tm == tn && wm * C::WM + C::WM <= wn * C::WN;
  // a warp tile entirely outside M x N (ragged edge tile of a variable-size problem) has no math
  // either.  (Per-8x8 predication of the DMMAs was measured slower: M1 27.0 -> 29.5 ms.)
  const bool idle_warp = upper_warp || m0 + wm * C::WM >= P.M || n0 + wn * C::WN >= P.N;
  double acc[C::MI][C::NI][2];
  double* Cp = P.C;  // may alias A (in-place TRSM with N <= 64)
  const int ldc = P.ldc;
  const double alpha = P.alpha, beta = P.beta;
  const double* Cin = Cp;   // the beta term's source
  int ldcin = ldc;
  if constexpr (EXT) {
    if (ext[pi].Cin) {
      Cin = ext[pi].Cin;
      ldcin = ext[pi].ldcin;
    }
  }
  // preload beta/alpha * C so the epilogue is a pure store
  // C preload scale beta/alpha: the common +-1 cases stay off the FP64 pipe (it is the DMMA pipe)
  const int cmode = (beta == 0.0 || alpha == 0.0) ? 0 : beta == alpha ? 1 : beta == -alpha ? 2 : 3;
  const double cscale = cmode == 3 ? beta / alpha : 1.0;
#pragma unroll
  for (int i = 0; i < C::MI; ++i)
#pragma unroll
    for (int j = 0; j < C::NI; ++j) {
      const int row = m0 + wm * C::WM + i * 8 + g;
      const int col = n0 + wn * C::WN + j * 8 + 2 * tq;
#pragma unroll
      for (int e = 0; e < 2; ++e)
        acc[i][j][e] = (!SPLIT && cmode && row < M && col + e < N) ? Cin[(size_t)row * ldcin + col + e] : 0.0;
    }
  if (!SPLIT && cmode == 2) {
#pragma unroll
    for (int i = 0; i < C::MI; ++i)
#pragma unroll
      for (int j = 0; j < C::NI; ++j) {
        acc[i][j][0] = neg_int(acc[i][j][0]);
        acc[i][j][1] = neg_int(acc[i][j][1]);
      }
  } else if (!SPLIT && cmode == 3) {
#pragma unroll
    for (int i = 0; i < C::MI; ++i)
#pragma unroll
      for (int j = 0; j < C::NI; ++j) {
        acc[i][j][0] *= cscale;
        acc[i][j][1] *= cscale;
      }
  }

  auto load_stage = [&](int stage, int k0) {
    double* as = As + stage * C::A_DBL;
    double* bs = Bs + stage * C::B_DBL;
#pragma unroll
    for (int jj = 0; jj < (tBM * BK) / C::THREADS; ++jj) {
      int idx = tid + jj * C::THREADS;
      if (!TA) {  // A[m][k] contiguous in k -> As[m][k]
        int m = idx / BK, k = idx % BK;
        int gm = m0 + m, gk = kbeg + k0 + k;
        bool v = gm < M && gk < kend;
        cp_async8(as + m * C::S_MK + k, v ? A + (size_t)gm * lda + gk : A, v);
      } else {    // A stored K x M, contiguous in m -> As[k][m]
        int k = idx / tBM, m = idx % tBM;
        int gm = m0 + m, gk = kbeg + k0 + k;
        bool v = gm < M && gk < kend;
        cp_async8(as + k * C::SA_KM + m, v ? A + (size_t)gk * lda + gm : A, v);
      }
    }
#pragma unroll
    for (int jj = 0; jj < (tBN * BK) / C::THREADS; ++jj) {
      int idx = tid + jj * C::THREADS;
      if (!TB) {  // B[k][n] contiguous in n -> Bs[k][n]
        int k = idx / tBN, n = idx % tBN;
        int gn = n0 + n, gk = kbeg + k0 + k;
        bool v = gn < N && gk < kend;
        cp_async8(bs + k * C::SB_KN + n, v ? B + (size_t)gk * ldb + gn : B, v);
      } else {    // B stored N x K, contiguous in k -> Bs[n][k]
        int n = idx / BK, k = idx % BK;
        int gn = n0 + n, gk = kbeg + k0 + k;
        bool v = gn < N && gk < kend;
        cp_async8(bs + n * C::S_MK + k, v ? B + (size_t)gn * ldb + gk : B, v);
      }
    }
  };

  const int KT = (kend - kbeg + BK - 1) / BK;
#pragma unroll
  for (int s = 0; s < C::STAGES - 1; ++s) {
    if (s < KT) load_stage(s, s * BK);
    cp_async_commit();
  }

  for (int kt = 0; kt < KT; ++kt) {
    cp_async_wait<C::STAGES - 2>();
    __syncthreads();
    {
      int nk = kt + C::STAGES - 1;
      if (nk < KT) load_stage(nk % C::STAGES, nk * BK);
      cp_async_commit();
    }
    const double* as = As + (kt % C::STAGES) * C::A_DBL;
    const double* bs = Bs + (kt % C::STAGES) * C::B_DBL;
    if (idle_warp) continue;    // still takes part in the loads and barriers
#pragma unroll
    for (int kk = 0; kk < BK; kk += 4) {
      double af[C::MI], bf[C::NI];
#pragma unroll
      for (int i = 0; i < C::MI; ++i) {
        int m = wm * C::WM + i * 8 + g, k = kk + tq;
        af[i] = TA ? as[k * C::SA_KM + m] : as[m * C::S_MK + k];
      }
#pragma unroll
      for (int j = 0; j < C::NI; ++j) {
        int n = wn * C::WN + j * 8 + g, k = kk + tq;
        bf[j] = TB ? bs[n * C::S_MK + k] : bs[k * C::SB_KN + n];
      }
#pragma unroll
      for (int i = 0; i < C::MI; ++i)
#pragma unroll
        for (int j = 0; j < C::NI; ++j)
          dmma884(acc[i][j], af[i], bf[j]);
    }
  }
  cp_async_wait<0>();

  if constexpr (SPLIT) {
    // partial tile -> ws (thread-private fragment order), the last CTA of the tile reduces
    constexpr int FR = C::MI * C::NI * 2;
    const int gtile = tile / nsplit;
    int32_t* counters = reinterpret_cast<int32_t*>(ws);
    double* parts = ws + ((size_t)ntiles * 4 + 255) / 256 * 32;   // 256-byte aligned after the counters
    double2* mine = reinterpret_cast<double2*>(parts + ((size_t)tile * C::THREADS + tid) * FR);
#pragma unroll
    for (int i = 0; i < C::MI; ++i)
#pragma unroll
      for (int j = 0; j < C::NI; ++j) mine[i * C::NI + j] = make_double2(acc[i][j][0], acc[i][j][1]);
    __threadfence();
    __syncthreads();
    __shared__ int last;
    if (tid == 0) last = atomicAdd(&counters[gtile], 1) == nsplit - 1;
    __syncthreads();
    if (!last) return;
    __threadfence();
#pragma unroll
    for (int i = 0; i < C::MI; ++i)
#pragma unroll
      for (int j = 0; j < C::NI; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
    for (int s2 = 0; s2 < nsplit; ++s2) {
      const double2* src =
          reinterpret_cast<const double2*>(parts + ((size_t)(gtile * nsplit + s2) * C::THREADS + tid) * FR);
#pragma unroll
      for (int i = 0; i < C::MI; ++i)
#pragma unroll
        for (int j = 0; j < C::NI; ++j) {
          const double2 v = __ldcg(src + i * C::NI + j);
          acc[i][j][0] += v.x;
          acc[i][j][1] += v.y;
        }
    }
    if (tid == 0) counters[gtile] = 0;   // ready for the next launch (graph replay)
    // the beta term (the unsplit kernel preloads it): acc += beta/alpha * C
    if (cmode) {
#pragma unroll
      for (int i = 0; i < C::MI; ++i)
#pragma unroll
        for (int j = 0; j < C::NI; ++j) {
          const int row = m0 + wm * C::WM + i * 8 + g;
          const int col = n0 + wn * C::WN + j * 8 + 2 * tq;
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            if (row >= M || col + e >= N) continue;
            const double c = Cin[(size_t)row * ldcin + col + e];
            acc[i][j][e] += cmode == 1 ? c : cmode == 2 ? neg_int(c) : cscale * c;
          }
        }
    }
  }

  // epilogue: C = alpha * acc   (acc already holds beta/alpha * C_old); alpha = +-1 stays off the FP64 pipe
  if (idle_warp) return;
  if (alpha == 0.0) {  // degenerate: C = beta * C
#pragma unroll
    for (int i = 0; i < C::MI; ++i) {
      const int row = m0 + wm * C::WM + i * 8 + g;
      if (row >= M) continue;
#pragma unroll
      for (int j = 0; j < C::NI; ++j) {
        const int col = n0 + wn * C::WN + j * 8 + 2 * tq;
        double* cp = Cp + (size_t)row * ldc + col;
#pragma unroll
        for (int e = 0; e < 2; ++e)
          if (col + e < N) cp[e] = beta * Cin[(size_t)row * ldcin + col + e];
      }
    }
    return;
  }
  if (alpha == -1.0) {
#pragma unroll
    for (int i = 0; i < C::MI; ++i)
#pragma unroll
      for (int j = 0; j < C::NI; ++j) {
        acc[i][j][0] = neg_int(acc[i][j][0]);
        acc[i][j][1] = neg_int(acc[i][j][1]);
      }
  } else if (alpha != 1.0) {
#pragma unroll
    for (int i = 0; i < C::MI; ++i)
#pragma unroll
      for (int j = 0; j < C::NI; ++j) {
        acc[i][j][0] *= alpha;
        acc[i][j][1] *= alpha;
      }
  }
  if constexpr (EXT) {
    const int rk = ext[pi].remap_k;
    if (rk <= -2) {
      // column relabel (q_full = [Q[:, k:] | Q[:, :k] s] from Q = I - Yt Y^T, k = -remap_k - 2;
      // dense_core.py:140-148): column b -> b - k (b >= k) or b + (N - k) (b < k), signed by s_b
      const double* __restrict__ sg = ext[pi].sgn;
      const int kc = -rk - 2, rr = N - kc;
#pragma unroll
      for (int i = 0; i < C::MI; ++i) {
        const int a = m0 + wm * C::WM + i * 8 + g;
        if (a >= M) continue;
#pragma unroll
        for (int j = 0; j < C::NI; ++j)
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const int b = n0 + wn * C::WN + j * 8 + 2 * tq + e;
            if (b >= N) continue;
            const int y = b >= kc ? b - kc : b + rr;
            const double v = (b < kc && sg[b] < 0.0) ? neg_int(acc[i][j][e]) : acc[i][j][e];
            Cp[(size_t)a * ldc + y] = v;
          }
      }
      return;
    }
    if (rk >= 0) {
      // compact-WY relabel (diag transform, ulv_factor.py:189-200): the tile holds H' = Q^T A Q in
      // Householder column order (skeleton columns 0..k-1 first); H = q_full^T A q_full puts the
      // redundant columns first: index a -> a - k (a >= k) or a + (M - k) (a < k), and id_basis's
      // signs s (dense_core.py:140-144) scale the skeleton rows / columns.  Only a >= b is stored:
      // every lower entry of H is the image of exactly one lower entry of H' (the SR block lands
      // transposed), so no entry has two writers.
      const double* __restrict__ sg = ext[pi].sgn;
      const int rr = M - rk;
#pragma unroll
      for (int i = 0; i < C::MI; ++i) {
        const int a = m0 + wm * C::WM + i * 8 + g;
        if (a >= M) continue;
        const int x = a >= rk ? a - rk : a + rr;
        const bool fa = a < rk && sg[a] < 0.0;
#pragma unroll
        for (int j = 0; j < C::NI; ++j)
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const int b = n0 + wn * C::WN + j * 8 + 2 * tq + e;
            if (b >= N || b > a) continue;
            const int y = b >= rk ? b - rk : b + rr;
            const bool fb = b < rk && sg[b] < 0.0;
            const double v = (fa != fb) ? neg_int(acc[i][j][e]) : acc[i][j][e];
            if (x >= y) Cp[(size_t)x * ldc + y] = v;
            else Cp[(size_t)y * ldc + x] = v;
          }
      }
      return;
    }
  }
#pragma unroll
  for (int i = 0; i < C::MI; ++i) {
    const int row = m0 + wm * C::WM + i * 8 + g;
    if (row >= M) continue;
#pragma unroll
    for (int j = 0; j < C::NI; ++j) {
      const int col = n0 + wn * C::WN + j * 8 + 2 * tq;
      double* cp = Cp + (size_t)row * ldc + col;
      if (col + 1 < N) {
        cp[0] = acc[i][j][0];
        cp[1] = acc[i][j][1];
      } else if (col < N) {
        cp[0] = acc[i][j][0];
      }
    }
  }
}

template <class C, bool TA, bool TB, bool EXT = false, bool SPLIT = false>
static int launch_gemm(const h2g_gemm_problem* d_probs, const int32_t* d_map, int tiles, cudaStream_t s,
                       const h2g_gemm_ext* d_ext = nullptr, double* ws = nullptr, int nsplit = 1) {
  static int attr_dev = -1;   // cudaFuncSetAttribute is per device
  int dev = 0;
  cudaGetDevice(&dev);
  if (attr_dev != dev) {
    cudaFuncSetAttribute(gemm_grouped_kernel<C, TA, TB, EXT, SPLIT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         C::SMEM);
    attr_dev = dev;
  }
  gemm_grouped_kernel<C, TA, TB, EXT, SPLIT><<<tiles, C::THREADS, C::SMEM, s>>>(d_probs, d_map, d_ext, ws, nsplit,
                                                                                 tiles / nsplit);
  return h2g_check_launch("gemm_grouped");
}

template <class C>
static int dispatch(int trans_a, int trans_b, const h2g_gemm_problem* d_probs, const int32_t* d_map, int tiles,
                    cudaStream_t s) {
  if (!trans_a && !trans_b) return launch_gemm<C, false, false>(d_probs, d_map, tiles, s);
  if (!trans_a && trans_b) return launch_gemm<C, false, true>(d_probs, d_map, tiles, s);
  if (trans_a && !trans_b) return launch_gemm<C, true, false>(d_probs, d_map, tiles, s);
  return launch_gemm<C, true, true>(d_probs, d_map, tiles, s);
}

// EXT variants: NN (the separate-Cin update) and NT (the relabelled symmetric rank-2k update)
template <class C>
static int dispatch_ext(int trans_a, int trans_b, const h2g_gemm_problem* d_probs, const h2g_gemm_ext* d_ext,
                        const int32_t* d_map, int tiles, cudaStream_t s) {
  if (!trans_a && !trans_b) return launch_gemm<C, false, false, true>(d_probs, d_map, tiles, s, d_ext);
  if (!trans_a && trans_b) return launch_gemm<C, false, true, true>(d_probs, d_map, tiles, s, d_ext);
  return h2g_set_error(H2G_EINVAL, "h2g_gemm_grouped_ext: NN or NT only");
}

template <class C>
static int dispatch_split(int trans_a, int trans_b, const h2g_gemm_problem* d_probs, const int32_t* d_map,
                          int ctas, double* ws, int nsplit, cudaStream_t s) {
  if (!trans_a && !trans_b) return launch_gemm<C, false, false, false, true>(d_probs, d_map, ctas, s, nullptr, ws, nsplit);
  if (!trans_a && trans_b) return launch_gemm<C, false, true, false, true>(d_probs, d_map, ctas, s, nullptr, ws, nsplit);
  if (trans_a && !trans_b) return launch_gemm<C, true, false, false, true>(d_probs, d_map, ctas, s, nullptr, ws, nsplit);
  return launch_gemm<C, true, true, false, true>(d_probs, d_map, ctas, s, nullptr, ws, nsplit);
}

}  // namespace h2g

extern "C" size_t h2g_gemm_split_workspace(int tiles, int nsplit) {
  return ((size_t)tiles * 4 + 255) / 256 * 256 + (size_t)tiles * nsplit * 64 * 64 * sizeof(double);
}

extern "C" int h2g_gemm_grouped_split(int trans_a, int trans_b, int tile_cfg, const h2g_gemm_problem* d_probs,
                                      const int32_t* d_tile_map, int total_ctas, int nsplit, void* d_ws,
                                      void* stream) {
  if (total_ctas <= 0) return H2G_OK;
  if (!d_probs || !d_tile_map || !d_ws) return h2g_set_error(H2G_EINVAL, "h2g_gemm_grouped_split: null argument");
  if (nsplit < 1 || total_ctas % nsplit)
    return h2g_set_error(H2G_EINVAL, "h2g_gemm_grouped_split: %d CTAs not a multiple of nsplit %d", total_ctas, nsplit);
  if (tile_cfg != 2) return h2g_set_error(H2G_EINVAL, "h2g_gemm_grouped_split: tile config %d (2 only)", tile_cfg);
  return h2g::dispatch_split<h2g::Cfg64b>(trans_a, trans_b, d_probs, d_tile_map, total_ctas, (double*)d_ws, nsplit,
                                          (cudaStream_t)stream);
}

extern "C" int h2g_gemm_grouped_ext(int trans_a, int trans_b, int tile_cfg, const h2g_gemm_problem* d_probs,
                                    const h2g_gemm_ext* d_ext, const int32_t* d_tile_map, int total_tiles,
                                    void* stream) {
  if (total_tiles <= 0) return H2G_OK;
  if (!d_probs || !d_tile_map || !d_ext) return h2g_set_error(H2G_EINVAL, "h2g_gemm_grouped_ext: null descriptor");
  cudaStream_t s = (cudaStream_t)stream;
  if (tile_cfg == 2) return h2g::dispatch_ext<h2g::Cfg64b>(trans_a, trans_b, d_probs, d_ext, d_tile_map, total_tiles, s);
  if (tile_cfg == 7) return h2g::dispatch_ext<h2g::Cfg64m3>(trans_a, trans_b, d_probs, d_ext, d_tile_map, total_tiles, s);
  if (tile_cfg == 9) return h2g::dispatch_ext<h2g::Cfg32>(trans_a, trans_b, d_probs, d_ext, d_tile_map, total_tiles, s);
  if (tile_cfg == 11) return h2g::dispatch_ext<h2g::Cfg64w8>(trans_a, trans_b, d_probs, d_ext, d_tile_map, total_tiles, s);
  return h2g_set_error(H2G_EINVAL, "h2g_gemm_grouped_ext: unknown tile config %d (2, 7, 9, 11)", tile_cfg);
}

extern "C" int h2g_gemm_tiles(int M, int N, int flags, int tile_cfg) {
  if (M <= 0 || N <= 0) return 0;
  const int T = tile_cfg == 9 ? 32 : 64;   // cfg 9: 32x32 tiles, cfg 2 / 7 / 11: 64x64
  if (flags & H2G_GEMM_LOWER) {
    int t = (M + T - 1) / T;
    return t * (t + 1) / 2;
  }
  return ((M + T - 1) / T) * ((N + T - 1) / T);
}

extern "C" int h2g_gemm_grouped(int trans_a, int trans_b, int tile_cfg, const h2g_gemm_problem* d_probs,
                                const int32_t* d_tile_map, int total_tiles, void* stream) {
  if (total_tiles <= 0) return H2G_OK;
  if (!d_probs || !d_tile_map) return h2g_set_error(H2G_EINVAL, "h2g_gemm_grouped: null descriptor");
  cudaStream_t s = (cudaStream_t)stream;
  if (tile_cfg == 2) return h2g::dispatch<h2g::Cfg64b>(trans_a, trans_b, d_probs, d_tile_map, total_tiles, s);
  if (tile_cfg == 7) return h2g::dispatch<h2g::Cfg64m3>(trans_a, trans_b, d_probs, d_tile_map, total_tiles, s);
  if (tile_cfg == 9) return h2g::dispatch<h2g::Cfg32>(trans_a, trans_b, d_probs, d_tile_map, total_tiles, s);
  if (tile_cfg == 11) return h2g::dispatch<h2g::Cfg64w8>(trans_a, trans_b, d_probs, d_tile_map, total_tiles, s);
  return h2g_set_error(H2G_EINVAL, "h2g_gemm_grouped: unknown tile config %d (2, 7, 9, 11)", tile_cfg);
}
