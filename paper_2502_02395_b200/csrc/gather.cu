// Block copy / transpose / symmetric gather: the skeleton merge.
//
// merge_level (ulv_factor.py:115-132) assembles every parent near block
// (pi >= pj) of level l-1 from the four child SS blocks of level l: SS_ii
// after the Schur update (only its lower half is maintained on the GPU ->
// mode 2), stored off-diagonal SS of near pairs or far couplings (mode 0),
// and their transposes when ci < cj (mode 1).  One launch moves a whole
// level; 64x64 tiles are staged through shared memory so both the read and
// the write are coalesced for the transposed quadrants.  HBM-bound.
#include "common.cuh"

namespace h2g {

// 64x64 tiles, 256 threads (32 x 8): every thread moves 16 elements and issues
// all its loads before its stores (a CTA per 32x32 tile spent most of its
// time on the descriptor chain: 3.4 TB/s on the merges).
constexpr int CT = 64;
constexpr int CR = CT / 8;   // rows per thread
constexpr int CC = CT / 32;  // columns per thread

__global__ void __launch_bounds__(256) block_copy_kernel(const h2g_copy_desc* __restrict__ descs,
                                                         const int32_t* __restrict__ tile_map) {
  __shared__ double tileA[CT][CT + 1];
  const h2g_copy_desc D = descs[tile_map[blockIdx.x]];
  const int t = blockIdx.x - D.tile_start;
  const int ntc = (D.cols + CT - 1) / CT;
  const int r0 = (t / ntc) * CT, c0 = (t % ntc) * CT;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;  // 32 x 8
  const double* __restrict__ src = D.src;
  double* __restrict__ dst = D.dst;
  const int lds = D.lds, ldd = D.ldd, rows = D.rows, cols = D.cols;
  int mode = D.mode;
  if (mode == 2) {
    if (r0 >= c0 + CT) mode = 0;          // tile strictly below the diagonal
    else if (c0 >= r0 + CT) mode = 1;     // strictly above: mirror
  }
  double v[CR][CC];
  if (mode == 3) {  // identity fill (src unused)
#pragma unroll
    for (int i = 0; i < CR; ++i)
#pragma unroll
      for (int j = 0; j < CC; ++j) {
        const int r = r0 + ty + 8 * i, c = c0 + tx + 32 * j;
        if (r < rows && c < cols) dst[(size_t)r * ldd + c] = (r == c) ? 1.0 : 0.0;
      }
    return;
  }
  if (mode != 1) {  // direct orientation: src[r][c]
#pragma unroll
    for (int i = 0; i < CR; ++i)
#pragma unroll
      for (int j = 0; j < CC; ++j) {
        const int r = r0 + ty + 8 * i, c = c0 + tx + 32 * j;
        v[i][j] = (r < rows && c < cols && (mode == 0 || r >= c)) ? src[(size_t)r * lds + c] : 0.0;
      }
  }
  if (mode != 0) {
    // tileA[a][b] = src[c0 + a][r0 + b]   (rows of the transposed source)
#pragma unroll
    for (int i = 0; i < CR; ++i)
#pragma unroll
      for (int j = 0; j < CC; ++j) {
        const int a = ty + 8 * i, bb = tx + 32 * j;
        const int sr = c0 + a, sc = r0 + bb;
        if (sr < cols && sc < rows && (mode == 1 || sr > sc)) tileA[a][bb] = src[(size_t)sr * lds + sc];
      }
    __syncthreads();
#pragma unroll
    for (int i = 0; i < CR; ++i)
#pragma unroll
      for (int j = 0; j < CC; ++j) {
        const int rr = ty + 8 * i, cc = tx + 32 * j;
        if (mode == 1 || r0 + rr < c0 + cc) v[i][j] = tileA[cc][rr];   // src[c][r]
      }
  }
#pragma unroll
  for (int i = 0; i < CR; ++i)
#pragma unroll
    for (int j = 0; j < CC; ++j) {
      const int r = r0 + ty + 8 * i, c = c0 + tx + 32 * j;
      if (r < rows && c < cols) dst[(size_t)r * ldd + c] = v[i][j];
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
