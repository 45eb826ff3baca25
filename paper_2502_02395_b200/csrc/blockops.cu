// Batched checks and triangular inverses behind the reference's single-block
// API (dense_core.cholesky / tri_solve, dense_core.py:51-81).
//
//  sym_check_kernel    one CTA per matrix: max |a_ij - a_ji| and max |a_ij|
//                      over the whole n x n block -> the ValueError contract
//                      "not symmetric to 1e-10 relative" (dense_core.py:56-59)
//                      is decided on the device, only two doubles per matrix
//                      come back.
//  tri_inv_kernel      one CTA per 64x64 diagonal block of a lower-triangular
//                      L: the block's inverse (the Linv layout the Cholesky
//                      panels write, so h2g_trsm_rows can solve against any
//                      triangular factor) and the first zero diagonal entry
//                      (SingularTriangularError, dense_core.py:75-76); with
//                      Linv == NULL only the diagonal check.
#include <climits>

#include "common.cuh"

namespace h2g {

constexpr int BO_PB = 64;

__global__ void __launch_bounds__(256) sym_check_kernel(const h2g_symcheck_desc* __restrict__ descs,
                                                        unsigned long long* __restrict__ out) {
  const h2g_symcheck_desc P = descs[blockIdx.x];
  const int n = P.n;
  double dmax = 0.0, amax = 0.0;
  const long long total = (long long)n * n;
  for (long long t = threadIdx.x; t < total; t += blockDim.x) {
    const int i = (int)(t / n), j = (int)(t % n);
    const double a = P.A[(size_t)i * P.lda + j];
    amax = fmax(amax, fabs(a));
    if (j < i) dmax = fmax(dmax, fabs(a - P.A[(size_t)j * P.lda + i]));   // fmax drops NaN, like numpy's NaN > x
  }
  __shared__ double sd[8], sa[8];
  for (int o = 16; o; o >>= 1) {
    dmax = fmax(dmax, __shfl_xor_sync(0xffffffffu, dmax, o));
    amax = fmax(amax, __shfl_xor_sync(0xffffffffu, amax, o));
  }
  const int w = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0) {
    sd[w] = dmax;
    sa[w] = amax;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int k = 1; k < (int)(blockDim.x >> 5); ++k) {
      dmax = fmax(dmax, sd[k]);
      amax = fmax(amax, sa[k]);
    }
    out[2 * blockIdx.x] = (unsigned long long)__double_as_longlong(dmax);
    out[2 * blockIdx.x + 1] = (unsigned long long)__double_as_longlong(amax);
  }
}

// Block q of matrix P: rows/cols p = 64q .. p+b-1.  Thread j < 64 solves
// L_qq x = e_j down its column, right-looking: the column's 64 partial sums
// live in registers and step i, once x_i = s_i / L_ii is known, updates the
// rows below with independent FMAs (the rows of L are broadcast from shared
// memory).  Every element gets the same FMA sequence (m = j .. i-1 in order)
// and the same division as a left-looking dot product, so the bits are those
// of the plain forward substitution; only the dependency chain is 64x shorter.
// Rows/cols >= b hold the identity.
__global__ void __launch_bounds__(BO_PB) tri_inv_kernel(const h2g_triinv_desc* __restrict__ descs,
                                                        const int32_t* __restrict__ tile_map,
                                                        int32_t* __restrict__ status) {
  __shared__ double Ls[BO_PB][BO_PB + 1];
  const int pi = tile_map[blockIdx.x];
  const h2g_triinv_desc P = descs[pi];
  const int q = blockIdx.x - P.tile_start;
  const int p = BO_PB * q, b = min(BO_PB, P.n - p);
  const int j = threadIdx.x;
  if (P.Linv == nullptr) {   // check only: the first zero diagonal entry (SingularTriangularError)
    if (j < b && P.L[(size_t)(p + j) * P.ldl + p + j] == 0.0) atomicMin(&status[P.status_slot], p + j);
    return;
  }
  for (int i = 0; i < BO_PB; ++i) Ls[i][j] = (i < b && j < b && j <= i) ? P.L[(size_t)(p + i) * P.ldl + p + j]
                                                                        : (i == j ? 1.0 : 0.0);
  __syncthreads();
  if (j < b && Ls[j][j] == 0.0) atomicMin(&status[P.status_slot], p + j);
  double sc[BO_PB];
#pragma unroll
  for (int r = 0; r < BO_PB; ++r) sc[r] = (r == j) ? 1.0 : 0.0;
#pragma unroll
  for (int i = 0; i < BO_PB; ++i) {
    const double x = (i >= j) ? sc[i] / Ls[i][i] : 0.0;
    sc[i] = x;
    if (i >= j) {
#pragma unroll
      for (int r = i + 1; r < BO_PB; ++r) sc[r] = fma(-Ls[r][i], x, sc[r]);
    }
  }
  double* out = P.Linv + (size_t)q * BO_PB * BO_PB;
#pragma unroll
  for (int i = 0; i < BO_PB; ++i) out[(size_t)i * BO_PB + j] = sc[i];
}

}  // namespace h2g

extern "C" int h2g_sym_check(const h2g_symcheck_desc* d_descs, int count, unsigned long long* d_out, void* stream) {
  if (count <= 0) return H2G_OK;
  if (!d_descs || !d_out) return h2g_set_error(H2G_EINVAL, "h2g_sym_check: null argument");
  h2g::sym_check_kernel<<<count, 256, 0, (cudaStream_t)stream>>>(d_descs, d_out);
  return h2g_check_launch("sym_check");
}

extern "C" int h2g_tri_inv(const h2g_triinv_desc* d_descs, const int32_t* d_tile_map, int total_tiles,
                           int32_t* d_status, void* stream) {
  if (total_tiles <= 0) return H2G_OK;
  if (!d_descs || !d_tile_map || !d_status) return h2g_set_error(H2G_EINVAL, "h2g_tri_inv: null argument");
  h2g::tri_inv_kernel<<<total_tiles, h2g::BO_PB, 0, (cudaStream_t)stream>>>(d_descs, d_tile_map, d_status);
  return h2g_check_launch("tri_inv");
}
