// Batched substitution kernels (forward / backward sweeps of the ULV
// factors, ulv_solve.py:66-188).  The solve streams every factor block once
// per sweep, so the kernels are built for memory-level parallelism: all
// loads of a thread are independent and unrolled, rows of a transposed
// operand are split across warps and reduced through shared memory, and a
// large segment is split over several CTAs (one 64-row output chunk each).
#include "common.cuh"

namespace h2g {

#ifndef H2G_GV_THREADS
#define H2G_GV_THREADS 512
#endif
constexpr int GV_THREADS = H2G_GV_THREADS;
constexpr int GV_CHUNK = 64;    // output rows per CTA (small: many CTAs for memory-level parallelism)
constexpr int GV_W = 4;         // RHS columns per pass
#ifndef H2G_GV_MINB
#define H2G_GV_MINB 4           // CTAs per SM the GEMV / TRSV are compiled for (4: 32 registers)
#endif
#ifndef H2G_GV_UNROLL
#define H2G_GV_UNROLL 4         // rows of a transposed operand in flight per warp
#endif
constexpr int GV_UNROLL = H2G_GV_UNROLL;
#ifndef H2G_GEMV_MINB
#define H2G_GEMV_MINB H2G_GV_MINB   // resident CTAs of 512 threads the grouped GEMV is compiled for
#endif

__device__ __forceinline__ int find_out(const h2g_gemv_out* outs, int n, int x) {
  int lo = 0, hi = n - 1;
  while (lo < hi) {
    int mid = (lo + hi + 1) >> 1;
    if (outs[mid].chunk_start <= x) lo = mid; else hi = mid - 1;
  }
  return lo;
}

// y[r0:r0+nr] (w columns) = init -/+ sum_t op(A_t) x_t, GW right-hand sides per pass
// (GW = 1: the single-vector solve; 4 otherwise)
template <int GW>
__global__ void __launch_bounds__(GV_THREADS, H2G_GEMV_MINB * 512 / GV_THREADS) gemv_grouped_kernel(const h2g_gemv_out* __restrict__ outs, int n_outs,
                                                                  const h2g_gemv_term* __restrict__ terms,
                                                                  const int32_t* __restrict__ chunk_map, int w) {
  __shared__ double acc[GV_CHUNK * GW];
  __shared__ double red[GV_THREADS / 32][GV_CHUNK];
  // the host-built chunk -> output map saves the dependent binary-search loads at CTA start
  const int oi = chunk_map ? chunk_map[blockIdx.x] : find_out(outs, n_outs, blockIdx.x);
  const h2g_gemv_out O = outs[oi];
  const int r0 = (blockIdx.x - O.chunk_start) * GV_CHUNK;
  const int nr = min(GV_CHUNK, O.m - r0);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  constexpr int NW = GV_THREADS / 32;
  const double sign = (O.flags & H2G_GEMV_PLUS) ? 1.0 : -1.0;
  const bool split = (O.flags & H2G_GEMV_SPLIT) != 0;

  for (int j0 = 0; j0 < w; j0 += GW) {
    const int wc = min(GW, w - j0);
    for (int e = tid; e < GV_CHUNK * GW; e += GV_THREADS) acc[e] = 0.0;
    __syncthreads();
    for (int ti = O.term_begin; ti < O.term_end; ++ti) {
      const h2g_gemv_term T = terms[ti];
      const double* __restrict__ A = T.A;
      const double* __restrict__ x = T.x;
      const int K = T.K, lda = T.lda;
      if (A == nullptr) {
        // identity term (K == m): acc += x[rows of this chunk]
        for (int e = tid; e < nr * wc; e += GV_THREADS) {
          const int rr = e / wc, j = e % wc;
          acc[rr * GW + j] += x[(size_t)(r0 + rr) * w + j0 + j];
        }
        __syncthreads();
      } else if (!T.trans) {
        // A is m x K: a warp owns two output rows at a time (twice the loads in flight),
        // lanes over the contiguous K axis
        for (int rr = 2 * warp; rr < nr; rr += 2 * NW) {
          const bool two = rr + 1 < nr;
          const double* arow = A + (size_t)(r0 + rr) * lda;
          const double* brow = two ? arow + lda : arow;
          double s[GW];
          double t[GW];
#pragma unroll
          for (int j = 0; j < GW; ++j) s[j] = t[j] = 0.0;
#pragma unroll 4
          for (int c = lane; c < K; c += 32) {
            const double a = arow[c];
            const double b = brow[c];
            const double* xc = x + (size_t)c * w + j0;
#pragma unroll
            for (int j = 0; j < GW; ++j)
              if (j < wc) {
                const double xv = xc[j];
                s[j] += a * xv;
                t[j] += b * xv;
              }
          }
#pragma unroll
          for (int j = 0; j < GW; ++j) {
            double v = s[j], u = t[j];
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
              v += __shfl_xor_sync(0xffffffffu, v, o);
              u += __shfl_xor_sync(0xffffffffu, u, o);
            }
            if (lane == 0 && j < wc) {
              acc[rr * GW + j] += v;
              if (two) acc[(rr + 1) * GW + j] += u;
            }
          }
        }
        __syncthreads();
      } else {
        // A is K x m: warps split the K rows, lanes own output columns
        for (int j = 0; j < wc; ++j) {
          double s[GV_CHUNK / 32];
#pragma unroll
          for (int t = 0; t < GV_CHUNK / 32; ++t) s[t] = 0.0;
#pragma unroll GV_UNROLL
          for (int c = warp; c < K; c += NW) {
            const double xv = x[(size_t)c * w + j0 + j];
            const double* arow = A + (size_t)c * lda + r0;
#pragma unroll
            for (int t = 0; t < GV_CHUNK / 32; ++t) {
              const int rr = lane + 32 * t;
              if (rr < nr) s[t] += arow[rr] * xv;
            }
          }
#pragma unroll
          for (int t = 0; t < GV_CHUNK / 32; ++t) red[warp][lane + 32 * t] = s[t];
          __syncthreads();
          for (int rr = tid; rr < nr; rr += GV_THREADS) {
            double v = 0.0;
#pragma unroll
            for (int q = 0; q < NW; ++q) v += red[q][rr];
            acc[rr * GW + j] += v;
          }
          __syncthreads();
        }
      }
    }
    for (int e = tid; e < nr * wc; e += GV_THREADS) {
      const int rr = e / wc, j = e % wc;
      const int r = r0 + rr;
      double v = sign * acc[rr * GW + j];
      if (O.init) v += O.init[(size_t)r * w + j0 + j];
      if (split && r >= O.split) O.y2[(size_t)(r - O.split) * w + j0 + j] = v;
      else O.y[(size_t)r * w + j0 + j] = v;
    }
    __syncthreads();
  }
}

// In-place triangular solve with the lower factor L (n x n, ld) of one box,
// blocked by the 64-wide Cholesky panels whose inverses Linv_q (64 x 64,
// written by the factorization's diagonal step) turn every diagonal solve
// into a small GEMV:
//   trans = 0:  x_P <- Linv_q (x_P - L[P, <P] x_<P)       (forward)
//   trans = 1:  x_P <- Linv_q^T (x_P - L[>P, P]^T x_>P)   (backward)
constexpr int TB = 64;
constexpr int TR_THREADS = 512;
constexpr int TR_WARPS = TR_THREADS / 32;
constexpr int TR_RPW = TB / TR_WARPS;   // rows per warp in the forward GEMV (4)
__global__ void __launch_bounds__(TR_THREADS, H2G_GV_MINB) trsv_batched_kernel(const h2g_trsv_desc* __restrict__ descs, int trans,
                                                                  int w) {
  __shared__ double t[TB];
  __shared__ double red[TR_WARPS][TB];
  const h2g_trsv_desc D = descs[blockIdx.x];
  const int n = D.n, ld = D.ldl;
  const double* __restrict__ L = D.L;
  const double* __restrict__ Li = D.Linv;
  double* __restrict__ x = D.x;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (n == 0) return;
  const int nblk = (n + TB - 1) / TB;
  for (int j = 0; j < w; ++j) {
    for (int bi = 0; bi < nblk; ++bi) {
      const int q = trans ? (nblk - 1 - bi) : bi;
      const int i0 = q * TB;
      const int nb = min(TB, n - i0);
      const double* Lq = Li + (size_t)q * TB * TB;
      if (!trans) {
        // t[r] = x[i0+r] - sum_{c < i0} L[i0+r][c] x[c]: each warp owns TR_RPW rows, all loads independent
        double s[TR_RPW];
#pragma unroll
        for (int u = 0; u < TR_RPW; ++u) s[u] = 0.0;
#pragma unroll 2
        for (int c = lane; c < i0; c += 32) {
          const double xv = x[(size_t)c * w + j];
#pragma unroll
          for (int u = 0; u < TR_RPW; ++u) {
            const int r = warp * TR_RPW + u;
            if (r < nb) s[u] += L[(size_t)(i0 + r) * ld + c] * xv;
          }
        }
#pragma unroll
        for (int u = 0; u < TR_RPW; ++u) {
          double v = s[u];
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
          const int r = warp * TR_RPW + u;
          if (lane == 0 && r < nb) t[r] = x[(size_t)(i0 + r) * w + j] - v;
        }
        __syncthreads();
        // x[i0+r] = sum_c Linv[r][c] t[c]
#pragma unroll
        for (int u = 0; u < TR_RPW; ++u) {
          const int r = warp * TR_RPW + u;
          double v = 0.0;
          if (r < nb)
            for (int c = lane; c <= r; c += 32) v += Lq[r * TB + c] * t[c];
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
          if (lane == 0 && r < nb) x[(size_t)(i0 + r) * w + j] = v;
        }
        __syncthreads();
      } else {
        // t[c] = x[i0+c] - sum_{r >= i0+nb} L[r][i0+c] x[r]  (warps split r, lanes own c)
        double s0 = 0.0, s1 = 0.0;
#pragma unroll 4
        for (int r = i0 + nb + warp; r < n; r += TR_WARPS) {
          const double xv = x[(size_t)r * w + j];
          const double* lrow = L + (size_t)r * ld + i0;
          if (lane < nb) s0 += lrow[lane] * xv;
          if (lane + 32 < nb) s1 += lrow[lane + 32] * xv;
        }
        red[warp][lane] = s0;
        red[warp][lane + 32] = s1;
        __syncthreads();
        if (tid < nb) {
          double v = 0.0;
#pragma unroll
          for (int qq = 0; qq < TR_WARPS; ++qq) v += red[qq][tid];
          t[tid] = x[(size_t)(i0 + tid) * w + j] - v;
        }
        __syncthreads();
        // x[i0+c] = sum_r Linv[r][c] t[r]   (r >= c)
        double u0 = 0.0, u1 = 0.0;
        for (int r = warp; r < nb; r += TR_WARPS) {
          const double tv = t[r];
          if (lane <= r) u0 += Lq[r * TB + lane] * tv;
          if (lane + 32 <= r) u1 += Lq[r * TB + lane + 32] * tv;
        }
        red[warp][lane] = u0;
        red[warp][lane + 32] = u1;
        __syncthreads();
        if (tid < nb) {
          double v = 0.0;
#pragma unroll
          for (int qq = 0; qq < TR_WARPS; ++qq) v += red[qq][tid];
          x[(size_t)(i0 + tid) * w + j] = v;
        }
        __syncthreads();
      }
    }
  }
}

// Basis transform of the forward sweep, [b_R; b_S] = q_full^T seg (_transform_in,
// ulv_solve.py:33-41), as a column-chunked GEMV: a CTA owns 128 output
// columns of one box (lane l: columns 4l..4l+3 of the chunk, two 16-byte
// loads per row), its 8 warps split the n rows (4 rows in flight each) and
// reduce through shared memory once at the end.  Every load is part of a
// 1 KB coalesced row segment, so a warp keeps 8 x 16 B per lane in flight
// (the general grouped GEMV reads 64-column chunks, 256 B per row and warp).
constexpr int XT_COLS = 128, XT_WARPS = 8, XT_THREADS = 32 * XT_WARPS;
template <bool VEC>
__global__ void __launch_bounds__(XT_THREADS) xform_t_kernel(const h2g_xform_desc* __restrict__ descs,
                                                             const int32_t* __restrict__ tile_map, int w) {
  __shared__ double red[XT_WARPS][XT_COLS];
  const h2g_xform_desc D = descs[tile_map[blockIdx.x]];
  const int c0 = (blockIdx.x - D.tile_start) * XT_COLS;
  const int n = D.n, ld = D.ldq;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int cl = c0 + 4 * lane;                  // this lane's first column
  for (int j = 0; j < w; ++j) {
    double s[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll 4
    for (int r = warp; r < n; r += XT_WARPS) {
      const double xv = __ldg(D.x + (size_t)r * w + j);
      const double* row = D.Q + (size_t)r * ld + cl;
      if (VEC && cl + 3 < n) {
        const double2 a = __ldg(reinterpret_cast<const double2*>(row));
        const double2 b = __ldg(reinterpret_cast<const double2*>(row) + 1);
        s[0] = fma(a.x, xv, s[0]);
        s[1] = fma(a.y, xv, s[1]);
        s[2] = fma(b.x, xv, s[2]);
        s[3] = fma(b.y, xv, s[3]);
      } else {
#pragma unroll
        for (int e = 0; e < 4; ++e)
          if (cl + e < n) s[e] = fma(__ldg(row + e), xv, s[e]);
      }
    }
#pragma unroll
    for (int e = 0; e < 4; ++e) red[warp][4 * lane + e] = s[e];
    __syncthreads();
    if (threadIdx.x < XT_COLS) {
      const int c = c0 + threadIdx.x;
      double v = 0.0;
#pragma unroll
      for (int q = 0; q < XT_WARPS; ++q) v += red[q][threadIdx.x];
      if (c < n) {
        if (c < D.split) D.y1[(size_t)c * w + j] = v;
        else D.y2[(size_t)(c - D.split) * w + j] = v;
      }
    }
    __syncthreads();
  }
}

// Basis transform of the backward sweep, full_i = q_red x_R + q_skel x_S = q_full [x_R; x_S]
// (ulv_solve.py:178-181): a CTA owns XN_ROWS output rows of one box, [x_R; x_S] is staged
// in shared memory, each warp takes its rows two at a time with the lanes across the
// columns (16-byte loads when the rows are aligned), one shuffle reduction per row.
#ifndef H2G_XN_ROWS
#define H2G_XN_ROWS 32
#endif
constexpr int XN_ROWS = H2G_XN_ROWS, XN_WARPS = 8, XN_THREADS = 32 * XN_WARPS, XN_MAXN = 4096;
template <bool VEC>
__global__ void __launch_bounds__(XN_THREADS) xform_n_kernel(const h2g_xform_n_desc* __restrict__ descs,
                                                             const int32_t* __restrict__ tile_map, int w) {
  extern __shared__ __align__(16) double xs[];   // n doubles (the launch sizes it to the largest box)
  const h2g_xform_n_desc D = descs[tile_map[blockIdx.x]];
  const int r0 = (blockIdx.x - D.tile_start) * XN_ROWS;
  const int n = D.n, r = D.r, ld = D.ldq;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int j = 0; j < w; ++j) {
    for (int c = threadIdx.x; c < n; c += XN_THREADS)
      xs[c] = c < r ? D.xr[(size_t)c * w + j] : D.xs[(size_t)(c - r) * w + j];
    __syncthreads();
    constexpr int RPW = XN_ROWS / XN_WARPS;   // rows per warp, taken two at a time (loads in flight)
#pragma unroll
    for (int u = 0; u < RPW; u += 2) {
      const int row = r0 + warp * RPW + u;
      if (row >= n) break;
      const bool two = row + 1 < n;
      const double* q = D.Q + (size_t)row * ld;
      const double* q2 = two ? q + ld : q;
      double s0 = 0.0, s1 = 0.0, t0 = 0.0, t1 = 0.0;
      if (VEC) {
#pragma unroll 4
        for (int c = 2 * lane; c < n; c += 64) {
          if (c + 1 < n) {
            const double2 a = __ldg(reinterpret_cast<const double2*>(q + c));
            const double2 b = __ldg(reinterpret_cast<const double2*>(q2 + c));
            s0 = fma(a.x, xs[c], s0);
            s1 = fma(a.y, xs[c + 1], s1);
            t0 = fma(b.x, xs[c], t0);
            t1 = fma(b.y, xs[c + 1], t1);
          } else {
            s0 = fma(__ldg(q + c), xs[c], s0);
            t0 = fma(__ldg(q2 + c), xs[c], t0);
          }
        }
      } else {
#pragma unroll 4
        for (int c = lane; c < n; c += 32) {
          s0 = fma(__ldg(q + c), xs[c], s0);
          t0 = fma(__ldg(q2 + c), xs[c], t0);
        }
      }
      double v = s0 + s1, v2 = t0 + t1;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        v += __shfl_xor_sync(0xffffffffu, v, o);
        v2 += __shfl_xor_sync(0xffffffffu, v2, o);
      }
      if (lane == 0) {
        D.out[(size_t)row * w + j] = v;
        if (two) D.out[(size_t)(row + 1) * w + j] = v2;
      }
    }
    __syncthreads();
  }
}

}  // namespace h2g

extern "C" int h2g_xform_n_rows(void) { return h2g::XN_ROWS; }

extern "C" int h2g_xform_n(const h2g_xform_n_desc* d_descs, const int32_t* d_tile_map, int total_tiles, int w,
                           int vec16, int max_n, void* stream) {
  if (total_tiles <= 0) return H2G_OK;
  if (!d_descs || !d_tile_map || w <= 0 || max_n <= 0 || max_n > h2g::XN_MAXN)
    return h2g_set_error(H2G_EINVAL, "h2g_xform_n: bad argument (max_n %d)", max_n);
  const size_t smem = (size_t)max_n * sizeof(double);
  if (vec16)
    h2g::xform_n_kernel<true><<<total_tiles, h2g::XN_THREADS, smem, (cudaStream_t)stream>>>(d_descs, d_tile_map, w);
  else
    h2g::xform_n_kernel<false><<<total_tiles, h2g::XN_THREADS, smem, (cudaStream_t)stream>>>(d_descs, d_tile_map, w);
  return h2g_check_launch("xform_n");
}

extern "C" int h2g_xform_t(const h2g_xform_desc* d_descs, const int32_t* d_tile_map, int total_tiles, int w,
                           int vec16, void* stream) {
  if (total_tiles <= 0) return H2G_OK;
  if (!d_descs || !d_tile_map || w <= 0) return h2g_set_error(H2G_EINVAL, "h2g_xform_t: bad argument");
  if (vec16)
    h2g::xform_t_kernel<true><<<total_tiles, h2g::XT_THREADS, 0, (cudaStream_t)stream>>>(d_descs, d_tile_map, w);
  else
    h2g::xform_t_kernel<false><<<total_tiles, h2g::XT_THREADS, 0, (cudaStream_t)stream>>>(d_descs, d_tile_map, w);
  return h2g_check_launch("xform_t");
}

extern "C" int h2g_gemv_grouped(const h2g_gemv_out* d_outs, int n_outs, const h2g_gemv_term* d_terms,
                                const int32_t* d_chunk_map, int total_chunks, int w, void* stream) {
  if (n_outs <= 0 || total_chunks <= 0) return H2G_OK;
  if (!d_outs || w <= 0) return h2g_set_error(H2G_EINVAL, "h2g_gemv_grouped: bad argument");
  if (w == 1)
    h2g::gemv_grouped_kernel<1><<<total_chunks, h2g::GV_THREADS, 0, (cudaStream_t)stream>>>(d_outs, n_outs, d_terms,
                                                                                           d_chunk_map, w);
  else
    h2g::gemv_grouped_kernel<h2g::GV_W><<<total_chunks, h2g::GV_THREADS, 0, (cudaStream_t)stream>>>(
        d_outs, n_outs, d_terms, d_chunk_map, w);
  return h2g_check_launch("gemv_grouped");
}

extern "C" int h2g_trsv_batched(const h2g_trsv_desc* d_descs, int count, int trans, int w, void* stream) {
  if (count <= 0) return H2G_OK;
  if (!d_descs || w <= 0) return h2g_set_error(H2G_EINVAL, "h2g_trsv_batched: bad argument");
  h2g::trsv_batched_kernel<<<count, h2g::TR_THREADS, 0, (cudaStream_t)stream>>>(d_descs, trans, w);
  return h2g_check_launch("trsv_batched");
}
