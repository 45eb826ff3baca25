// ① Complementary basis: batched blocked Householder QR (LAPACK dgeqrf /
// dlarfg / dlarft / dorgqr conventions) of Z_i = T_i or W_i T_i, every box of
// a level at once (id_basis, dense_core.py:136-148, called per box from
// construct, h2_build.py:193-199).
//
// h2g_qr_panel: per box one CTA factors the panel Z[p:n, p:p+b] (b <= 32)
// in place — Householder vectors below the diagonal, R on/above it — writes
// tau, and the upper-triangular block factor T (b x b) with
// H_p ... H_{p+b-1} = I - V T V^T.  The trailing update of Z and the explicit
// formation of Q are grouped GEMMs issued by the host plan.
// h2g_basis_finish: sign fix (diag R >= 0) and [q_red | q_skel] assembly.
#include "common.cuh"

namespace h2g {

constexpr int QB = 32;
constexpr int QR_THREADS = 256;

__device__ __forceinline__ double block_sum(double v, double* red) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  __syncthreads();
  if (lane == 0) red[warp] = v;
  __syncthreads();
  double t = 0.0;
#pragma unroll
  for (int q = 0; q < QR_THREADS / 32; ++q) t += red[q];
  return t;
}

// SM = true: the panel Z[p:n, p:p+b] is staged in shared memory (stride QB+1)
// for the whole column loop and written back once; SM = false works on Z in
// global memory (panels too tall for shared memory).
template <bool SM>
__global__ void __launch_bounds__(QR_THREADS) qr_panel_kernel(const h2g_qr_panel_desc* __restrict__ descs) {
  extern __shared__ double psm[];
  __shared__ double red[QR_THREADS / 32];
  __shared__ double dots[QB];
  __shared__ double G[QB][QB + 1];
  __shared__ double taus[QB];
  const h2g_qr_panel_desc D = descs[blockIdx.x];
  const int n = D.n, ld = D.ldz, p = D.p, b = D.b;
  double* __restrict__ Z = D.Z;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  // element (r, c) of the panel, r >= p, p <= c < p + b
  auto ZA = [&](int r, int c) -> double& {
    if constexpr (SM) return psm[(size_t)(r - p) * (QB + 1) + (c - p)];
    else return Z[(size_t)r * ld + c];
  };
  if constexpr (SM) {
    for (int e = tid; e < (n - p) * b; e += QR_THREADS) {
      const int r = e / b, c = e % b;
      psm[(size_t)r * (QB + 1) + c] = Z[(size_t)(p + r) * ld + p + c];
    }
    __syncthreads();
  }

  for (int j = 0; j < b; ++j) {
    const int c = p + j;             // global column / diagonal row
    // --- dlarfg on Z[c:n, c]
    double ss = 0.0;
    for (int r = c + 1 + tid; r < n; r += QR_THREADS) {
      double v = ZA(r, c);
      ss += v * v;
    }
    const double xnorm2 = block_sum(ss, red);
    const double alpha = ZA(c, c);
    double tau = 0.0, scal = 0.0, beta = alpha;
    if (xnorm2 > 0.0) {
      const double xnorm = sqrt(xnorm2);
      beta = -copysign(hypot(alpha, xnorm), alpha);
      tau = (beta - alpha) / beta;
      scal = 1.0 / (alpha - beta);
    }
    __syncthreads();  // everyone has read alpha before it is overwritten
    if (tau != 0.0) {
      for (int r = c + 1 + tid; r < n; r += QR_THREADS) ZA(r, c) *= scal;
    }
    if (tid == 0) {
      ZA(c, c) = beta;
      taus[j] = tau;
      D.tau[c] = tau;
    }
    __syncthreads();
    if (tau == 0.0) continue;
    // --- apply H = I - tau v v^T (v = [1; Z[c+1:n, c]]) to panel columns c+1 .. p+b-1
    for (int q = warp; q < b - j - 1; q += QR_THREADS / 32) {
      const int cc = c + 1 + q;
      double s = (lane == 0) ? ZA(c, cc) : 0.0;
      for (int r = c + 1 + lane; r < n; r += 32) s += ZA(r, c) * ZA(r, cc);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
      if (lane == 0) dots[q] = s;
    }
    __syncthreads();
    for (int q = warp; q < b - j - 1; q += QR_THREADS / 32) {
      const int cc = c + 1 + q;
      const double f = tau * dots[q];
      if (lane == 0) ZA(c, cc) -= f;
      for (int r = c + 1 + lane; r < n; r += 32) ZA(r, cc) -= f * ZA(r, c);
    }
    __syncthreads();
  }

  if constexpr (SM) {   // the factored panel back to Z (R on/above the diagonal, reflectors below)
    for (int e = tid; e < (n - p) * b; e += QR_THREADS) {
      const int r = e / b, c = e % b;
      Z[(size_t)(p + r) * ld + p + c] = psm[(size_t)r * (QB + 1) + c];
    }
  }
  // --- explicit reflectors V[p:n, p:p+b] (unit diagonal, zeros above)
  for (int e = tid; e < (n - p) * b; e += QR_THREADS) {
    const int r = p + e / b, j = e % b;
    const int c = p + j;
    double v = (r < c) ? 0.0 : (r == c ? 1.0 : ZA(r, c));
    if (taus[j] == 0.0 && r != c) v = 0.0;
    D.V[(size_t)r * ld + c] = v;
  }
  // --- T (dlarft, forward / columnwise): G = V^T V of the panel reflectors
  for (int e = warp; e < b * b; e += QR_THREADS / 32) {
    const int i = e / b, j = e % b;
    if (i >= j) continue;
    // V[:, i] = e_{p+i} + Z[p+i+1:, p+i];  V[:, j] = e_{p+j} + Z[p+j+1:, p+j]; overlap rows >= p+j
    double s = (lane == 0) ? ZA((p + j), p + i) : 0.0;  // row p+j: V_i entry * 1
    for (int r = p + j + 1 + lane; r < n; r += 32) s += ZA(r, p + i) * ZA(r, p + j);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) G[i][j] = s;
  }
  __syncthreads();
  if (warp == 0) {
    // T[0:j, j] = -tau_j * T[0:j, 0:j] * G[0:j, j];  T[j][j] = tau_j   (column by column)
    double* T = D.T;
    for (int j = 0; j < QB; ++j) {
      double tj = 0.0;
      if (j < b && lane < j) {
        for (int m = lane; m < j; ++m) tj += T[lane * QB + m] * G[m][j];
        tj *= -taus[j];
      }
      __syncwarp();
      if (lane < QB) {
        double v = 0.0;
        if (j < b) v = (lane < j) ? tj : (lane == j ? taus[j] : 0.0);
        T[lane * QB + j] = v;
      }
      __syncwarp();
      __threadfence_block();
    }
  }
}

__global__ void __launch_bounds__(256) basis_finish_kernel(const h2g_basis_desc* __restrict__ descs) {
  __shared__ double s[2048 + 8];
  const h2g_basis_desc D = descs[blockIdx.x];
  const int n = D.n, k = D.k, r = n - k;
  for (int i = threadIdx.x; i < k; i += 256) {
    double d = D.Z[(size_t)i * D.ldz + i];
    s[i] = (d < 0.0) ? -1.0 : 1.0;   // sign(0) -> +1
  }
  __syncthreads();
  // rows [r0, r1) of this CTA (blockIdx.y of gridDim.y slices)
  const int r0 = (int)((long long)n * blockIdx.y / gridDim.y), r1 = (int)((long long)n * (blockIdx.y + 1) / gridDim.y);
  for (size_t e = (size_t)r0 * n + threadIdx.x; e < (size_t)r1 * n; e += 256) {
    int row = (int)(e / n), col = (int)(e % n);
    double v;
    if (col < r) v = D.Q[(size_t)row * n + k + col];
    else v = D.Q[(size_t)row * n + (col - r)] * s[col - r];
    D.qfull[e] = v;
  }
  if (blockIdx.y == 0) {
    for (size_t e = threadIdx.x; e < (size_t)k * k; e += 256) {
      int i = (int)(e / k), j = (int)(e % k);
      D.frame[e] = (j >= i) ? s[i] * D.Z[(size_t)i * D.ldz + j] : 0.0;
    }
  }
}

}  // namespace h2g

extern "C" int h2g_qr_panel(const h2g_qr_panel_desc* d_descs, int count, int max_rows, void* stream) {
  if (count <= 0) return H2G_OK;
  if (!d_descs) return h2g_set_error(H2G_EINVAL, "h2g_qr_panel: null descriptors");
  // panels up to ~780 rows are factored in shared memory (one global read / write of the panel)
  const size_t smem = (size_t)max_rows * (h2g::QB + 1) * sizeof(double);
  if (max_rows > 0 && smem <= 200 * 1024) {
    static size_t attr[64] = {};   // per device (function attributes are per device)
    int dev = 0;
    cudaGetDevice(&dev);
    dev &= 63;
    if (smem > attr[dev]) {
      cudaFuncSetAttribute(h2g::qr_panel_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      attr[dev] = smem;
    }
    h2g::qr_panel_kernel<true><<<count, h2g::QR_THREADS, smem, (cudaStream_t)stream>>>(d_descs);
  } else {
    h2g::qr_panel_kernel<false><<<count, h2g::QR_THREADS, 0, (cudaStream_t)stream>>>(d_descs);
  }
  return h2g_check_launch("qr_panel");
}

extern "C" int h2g_basis_finish(const h2g_basis_desc* d_descs, int count, void* stream) {
  if (count <= 0) return H2G_OK;
  if (!d_descs) return h2g_set_error(H2G_EINVAL, "h2g_basis_finish: null descriptors");
  h2g::basis_finish_kernel<<<dim3(count, 16), 256, 0, (cudaStream_t)stream>>>(d_descs);   // 16 row slices per box
  return h2g_check_launch("basis_finish");
}
