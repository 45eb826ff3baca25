// Block copy / transpose / symmetric gather: the skeleton merge.
//
// merge_level (ulv_factor.py:115-132) assembles every parent near block
// (pi >= pj) of level l-1 from the four child SS blocks of level l: SS_ii
// after the Schur update (only its lower half is maintained on the GPU ->
// mode 2), stored off-diagonal SS of near pairs or far couplings (mode 0),
// and their transposes when ci < cj (mode 1).  One launch moves a whole
// level; 32x32 tiles are staged through shared memory so both the read and
// the write are coalesced for the transposed quadrants.  HBM-bound.
#include "common.cuh"

namespace h2g {

constexpr int CT = 32;

__global__ void __launch_bounds__(256) block_copy_kernel(const h2g_copy_desc* __restrict__ descs,
                                                         const int32_t* __restrict__ tile_map) {
  __shared__ double tileA[CT][CT + 1];
  __shared__ double tileB[CT][CT + 1];
  const h2g_copy_desc D = descs[tile_map[blockIdx.x]];
  const int t = blockIdx.x - D.tile_start;
  const int ntc = (D.cols + CT - 1) / CT;
  const int r0 = (t / ntc) * CT, c0 = (t % ntc) * CT;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;  // 32 x 8
  const double* __restrict__ src = D.src;
  double* __restrict__ dst = D.dst;
  const int lds = D.lds, ldd = D.ldd;
  int mode = D.mode;
  if (mode == 2) {
    if (r0 >= c0 + CT) mode = 0;          // tile strictly below the diagonal
    else if (c0 >= r0 + CT) mode = 1;     // strictly above: mirror
  }
  if (mode == 3) {  // identity fill (src unused)
    for (int rr = ty; rr < CT; rr += 8) {
      int r = r0 + rr, c = c0 + tx;
      if (r < D.rows && c < D.cols) dst[(size_t)r * ldd + c] = (r == c) ? 1.0 : 0.0;
    }
    return;
  }
  if (mode == 0) {
    for (int rr = ty; rr < CT; rr += 8) {
      int r = r0 + rr, c = c0 + tx;
      if (r < D.rows && c < D.cols) dst[(size_t)r * ldd + c] = src[(size_t)r * lds + c];
    }
    return;
  }
  // tileA[a][b] = src[(c0+a)][r0+b]   (rows of the transposed source)
  for (int a = ty; a < CT; a += 8) {
    int sr = c0 + a, sc = r0 + tx;
    if (sr < D.cols && sc < D.rows) tileA[a][tx] = src[(size_t)sr * lds + sc];
  }
  if (mode == 2) {  // diagonal tile: also the direct orientation
    for (int a = ty; a < CT; a += 8) {
      int sr = r0 + a, sc = c0 + tx;
      if (sr < D.rows && sc < D.cols) tileB[a][tx] = src[(size_t)sr * lds + sc];
    }
  }
  __syncthreads();
  for (int rr = ty; rr < CT; rr += 8) {
    int r = r0 + rr, c = c0 + tx;
    if (r < D.rows && c < D.cols) {
      double v;
      if (mode == 1 || r < c) v = tileA[tx][rr];   // src[c][r]
      else v = tileB[rr][tx];                      // src[r][c]
      dst[(size_t)r * ldd + c] = v;
    }
  }
}

}  // namespace h2g

extern "C" int h2g_copy_tiles(int rows, int cols) {
  if (rows <= 0 || cols <= 0) return 0;
  return ((rows + h2g::CT - 1) / h2g::CT) * ((cols + h2g::CT - 1) / h2g::CT);
}

extern "C" int h2g_block_copy(const h2g_copy_desc* d_descs, const int32_t* d_tile_map, int total_tiles,
                              void* stream) {
  if (total_tiles <= 0) return H2G_OK;
  if (!d_descs || !d_tile_map) return h2g_set_error(H2G_EINVAL, "h2g_block_copy: null argument");
  h2g::block_copy_kernel<<<total_tiles, 256, 0, (cudaStream_t)stream>>>(d_descs, d_tile_map);
  return h2g_check_launch("block_copy");
}
