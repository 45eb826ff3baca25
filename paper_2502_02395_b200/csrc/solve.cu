// Batched substitution kernels (forward / backward sweeps of the ULV
// factors, ulv_solve.py:66-188).  The solve is HBM/latency bound: every
// factor block is read once per sweep, so the kernels are written for
// coalesced streaming of the block rows, one CTA per output segment / box.
#include "common.cuh"

namespace h2g {

constexpr int GV_THREADS = 256;
constexpr int GV_WMAX = 8;        // columns processed per pass
constexpr int GV_ROWS = 2048;     // rows per smem chunk (x GV_WMAX doubles = 128 KB max)

// acc (rows x wc) += sum over terms of op(A) x   for rows [r0, r0+nr), columns [j0, j0+wc)
__global__ void __launch_bounds__(GV_THREADS) gemv_grouped_kernel(const h2g_gemv_out* __restrict__ outs,
                                                                  const h2g_gemv_term* __restrict__ terms,
                                                                  int w) {
  extern __shared__ double acc[];  // GV_ROWS * GV_WMAX
  const h2g_gemv_out O = outs[blockIdx.x];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int nwarps = GV_THREADS / 32;
  const double sign = (O.flags & H2G_GEMV_PLUS) ? 1.0 : -1.0;
  const bool split = (O.flags & H2G_GEMV_SPLIT) != 0;

  for (int j0 = 0; j0 < w; j0 += GV_WMAX) {
    const int wc = min(GV_WMAX, w - j0);
    for (int r0 = 0; r0 < O.m; r0 += GV_ROWS) {
      const int nr = min(GV_ROWS, O.m - r0);
      for (int e = tid; e < nr * GV_WMAX; e += GV_THREADS) acc[e] = 0.0;
      __syncthreads();
      for (int ti = O.term_begin; ti < O.term_end; ++ti) {
        const h2g_gemv_term T = terms[ti];
        const double* __restrict__ A = T.A;
        const double* __restrict__ x = T.x;
        if (!T.trans) {
          // A is m x K: warp per row, lanes stride the (contiguous) columns
          for (int rr = warp; rr < nr; rr += nwarps) {
            const double* arow = A + (size_t)(r0 + rr) * T.lda;
            double s[GV_WMAX];
#pragma unroll
            for (int j = 0; j < GV_WMAX; ++j) s[j] = 0.0;
            for (int c = lane; c < T.K; c += 32) {
              double a = arow[c];
              const double* xc = x + (size_t)c * w + j0;
#pragma unroll
              for (int j = 0; j < GV_WMAX; ++j)
                if (j < wc) s[j] += a * xc[j];
            }
#pragma unroll
            for (int j = 0; j < GV_WMAX; ++j) {
              double v = s[j];
#pragma unroll
              for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
              if (lane == 0 && j < wc) acc[rr * GV_WMAX + j] += v;
            }
          }
        } else {
          // A is K x m: thread per output row, coalesced along the row of A
          for (int rr = tid; rr < nr; rr += GV_THREADS) {
            double s[GV_WMAX];
#pragma unroll
            for (int j = 0; j < GV_WMAX; ++j) s[j] = 0.0;
            const double* acol = A + r0 + rr;
            for (int c = 0; c < T.K; ++c) {
              double a = acol[(size_t)c * T.lda];
              const double* xc = x + (size_t)c * w + j0;
#pragma unroll
              for (int j = 0; j < GV_WMAX; ++j)
                if (j < wc) s[j] += a * xc[j];
            }
#pragma unroll
            for (int j = 0; j < GV_WMAX; ++j)
              if (j < wc) acc[rr * GV_WMAX + j] += s[j];
          }
        }
        __syncthreads();
      }
      for (int e = tid; e < nr * wc; e += GV_THREADS) {
        int rr = e / wc, j = e % wc;
        int r = r0 + rr;
        double v = sign * acc[rr * GV_WMAX + j];
        if (O.init) v += O.init[(size_t)r * w + j0 + j];
        if (split && r >= O.split) O.y2[(size_t)(r - O.split) * w + j0 + j] = v;
        else O.y[(size_t)r * w + j0 + j] = v;
      }
      __syncthreads();
    }
  }
}

// In-place triangular solve with the lower factor L (n x n, ld):
//   trans = 0: x <- L^-1 x (forward);  trans = 1: x <- L^-T x (backward).
// Blocked by 32 rows; the off-block products are warp dot products, the
// 32x32 diagonal triangle is solved by one warp from shared memory.
constexpr int TB = 32;
__global__ void __launch_bounds__(256) trsv_batched_kernel(const h2g_trsv_desc* __restrict__ descs, int trans,
                                                           int w) {
  __shared__ double Ld[TB][TB + 1];
  __shared__ double part[TB];
  const h2g_trsv_desc D = descs[blockIdx.x];
  const int n = D.n, ld = D.ldl;
  const double* __restrict__ L = D.L;
  double* __restrict__ x = D.x;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (n == 0) return;
  const int nblk = (n + TB - 1) / TB;
  for (int j = 0; j < w; ++j) {
    for (int bi = 0; bi < nblk; ++bi) {
      const int blk = trans ? (nblk - 1 - bi) : bi;
      const int i0 = blk * TB;
      const int nb = min(TB, n - i0);
      // diagonal block -> smem
      for (int e = tid; e < TB * TB; e += 256) {
        int r = e / TB, c = e % TB;
        Ld[r][c] = (r < nb && c < nb) ? L[(size_t)(i0 + r) * ld + i0 + c] : 0.0;
      }
      // off-block contribution
      if (!trans) {
        // part[r] = sum_{c < i0} L[i0+r][c] x[c]
        for (int r = warp; r < nb; r += 8) {
          const double* lrow = L + (size_t)(i0 + r) * ld;
          double s = 0.0;
          for (int c = lane; c < i0; c += 32) s += lrow[c] * x[(size_t)c * w + j];
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
          if (lane == 0) part[r] = s;
        }
      } else {
        // part[r] = sum_{c >= i0+nb} L[c][i0+r] x[c]; 8 warps split c, lanes over r
        __shared__ double red[8][TB];
        double s = 0.0;
        if (lane < nb)
          for (int c = i0 + nb + warp; c < n; c += 8) s += L[(size_t)c * ld + i0 + lane] * x[(size_t)c * w + j];
        red[warp][lane] = s;
        __syncthreads();
        if (warp == 0) {
          double t = 0.0;
#pragma unroll
          for (int q = 0; q < 8; ++q) t += red[q][lane];
          part[lane] = t;
        }
      }
      __syncthreads();
      if (warp == 0) {
        double xi = (lane < nb) ? x[(size_t)(i0 + lane) * w + j] - part[lane] : 0.0;
        if (!trans) {
          for (int c = 0; c < nb; ++c) {
            double xc = __shfl_sync(0xffffffffu, xi / Ld[c][c], c);
            if (lane == c) xi = xc;
            else if (lane > c) xi -= Ld[lane][c] * xc;
          }
        } else {
          for (int c = nb - 1; c >= 0; --c) {
            double xc = __shfl_sync(0xffffffffu, xi / Ld[c][c], c);
            if (lane == c) xi = xc;
            else if (lane < c) xi -= Ld[c][lane] * xc;
          }
        }
        if (lane < nb) x[(size_t)(i0 + lane) * w + j] = xi;
      }
      __syncthreads();
    }
  }
}

}  // namespace h2g

extern "C" int h2g_gemv_grouped(const h2g_gemv_out* d_outs, int n_outs, const h2g_gemv_term* d_terms, int w,
                                void* stream) {
  if (n_outs <= 0) return H2G_OK;
  if (!d_outs || w <= 0) return h2g_set_error(H2G_EINVAL, "h2g_gemv_grouped: bad argument");
  static bool attr = false;
  const int smem = h2g::GV_ROWS * h2g::GV_WMAX * 8;
  if (!attr) {
    cudaFuncSetAttribute(h2g::gemv_grouped_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    attr = true;
  }
  h2g::gemv_grouped_kernel<<<n_outs, h2g::GV_THREADS, smem, (cudaStream_t)stream>>>(d_outs, d_terms, w);
  return h2g_check_launch("gemv_grouped");
}

extern "C" int h2g_trsv_batched(const h2g_trsv_desc* d_descs, int count, int trans, int w, void* stream) {
  if (count <= 0) return H2G_OK;
  if (!d_descs || w <= 0) return h2g_set_error(H2G_EINVAL, "h2g_trsv_batched: bad argument");
  h2g::trsv_batched_kernel<<<count, 256, 0, (cudaStream_t)stream>>>(d_descs, trans, w);
  return h2g_check_launch("trsv_batched");
}
