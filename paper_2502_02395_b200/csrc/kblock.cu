// Kernel-matrix block generation on the device (kernels.gen_block,
// kernels.py:46-64): leaf near blocks G(B_i, B_j) and the skeleton blocks
// G(SK_i, SK_j) behind the couplings (h2_build.py:205-215).
// Distances are evaluated without FMA contraction in the same order as
// scipy's cdist ((dx^2 + dy^2) + dz^2, then a correctly rounded sqrt), and
// 1/r is an IEEE division, so Laplace entries are bit-identical to the
// reference's.  Family 2 is the opt-in Gaussian covariance exp(-r^2 / l^2)
// (BASELINE configs[3]; not a reference family).
#include "common.cuh"

namespace h2g {

__global__ void __launch_bounds__(256) kernel_block_kernel(const h2g_kblock_desc* __restrict__ descs,
                                                           const int32_t* __restrict__ tile_map,
                                                           const double* __restrict__ pts, int family,
                                                           double shift, double decay,
                                                           long long* __restrict__ coincident) {
  const h2g_kblock_desc D = descs[tile_map[blockIdx.x]];
  const int t = blockIdx.x - D.tile_start;
  const int ntc = (D.n + 31) / 32;
  const int r0 = (t / ntc) * 32, c0 = (t % ntc) * 32;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  const int c = c0 + tx;
  if (c >= D.n) return;
  const long long cj = D.cols[c];
  const double xj = pts[3 * cj], yj = pts[3 * cj + 1], zj = pts[3 * cj + 2];
  for (int rr = ty; rr < 32; rr += 8) {
    const int r = r0 + rr;
    if (r >= D.m) break;
    const long long ri = D.rows[r];
    double v;
    if (ri == cj) {
      v = shift;
    } else {
      const double dx = __dsub_rn(pts[3 * ri], xj);
      const double dy = __dsub_rn(pts[3 * ri + 1], yj);
      const double dz = __dsub_rn(pts[3 * ri + 2], zj);
      const double s = __dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)), __dmul_rn(dz, dz));
      const double d = __dsqrt_rn(s);
      if (d == 0.0) {
        atomicExch((unsigned long long*)&coincident[0], 1ULL);  // host locates the pair
        v = __longlong_as_double(0x7ff8000000000000LL);
      } else if (family == 0) {
        v = __ddiv_rn(1.0, d);
      } else if (family == 2) {       // gaussian covariance exp(-(r/l)^2), decay = 1/l^2
        v = exp(-__dmul_rn(__dmul_rn(d, d), decay));   // host: exp(-(r * r) / l^2)
      } else {
        v = __ddiv_rn(exp(-decay * d), d);
      }
    }
    D.out[(size_t)r * D.ldo + c] = v;
  }
}

}  // namespace h2g

extern "C" int h2g_kernel_blocks(const h2g_kblock_desc* d_descs, const int32_t* d_tile_map, int total_tiles,
                                 const double* d_points, int family, double shift, double decay,
                                 int64_t* d_coincident, void* stream) {
  if (total_tiles <= 0) return H2G_OK;
  if (!d_descs || !d_tile_map || !d_points || !d_coincident)
    return h2g_set_error(H2G_EINVAL, "h2g_kernel_blocks: null argument");
  if (family < 0 || family > 2) return h2g_set_error(H2G_EINVAL, "h2g_kernel_blocks: unknown family %d", family);
  h2g::kernel_block_kernel<<<total_tiles, 256, 0, (cudaStream_t)stream>>>(
      d_descs, d_tile_map, d_points, family, shift, decay, (long long*)d_coincident);
  return h2g_check_launch("kernel_blocks");
}
