#include <cstdio>
#include <vector>
#include "cutlass/cutlass.h"
#include "cutlass/gemm/gemm.h"
#include "cutlass/gemm/kernel/gemm_grouped.h"
#include "cutlass/gemm/kernel/default_gemm_grouped.h"
#include "cutlass/gemm/device/gemm_grouped.h"
#include "cutlass/epilogue/thread/linear_combination.h"

using ElementA = double; using ElementB = double; using ElementC = double; using ElementAcc = double;
using LayoutA = cutlass::layout::RowMajor; using LayoutB = cutlass::layout::RowMajor; using LayoutC = cutlass::layout::RowMajor;

using GemmKernel = typename cutlass::gemm::kernel::DefaultGemmGrouped<
  ElementA, LayoutA, cutlass::ComplexTransform::kNone, 1,
  ElementB, LayoutB, cutlass::ComplexTransform::kNone, 1,
  ElementC, LayoutC, ElementAcc,
  cutlass::arch::OpClassTensorOp, cutlass::arch::Sm80,
  cutlass::gemm::GemmShape<64, 128, 16>, cutlass::gemm::GemmShape<32, 64, 16>, cutlass::gemm::GemmShape<8, 8, 4>,
  cutlass::epilogue::thread::LinearCombination<ElementC, 1, ElementAcc, ElementAcc>,
  cutlass::gemm::threadblock::GemmBatchedIdentityThreadblockSwizzle,
  3, cutlass::gemm::kernel::GroupScheduleMode::kDeviceOnly>::GemmKernel;
using Gemm = cutlass::gemm::device::GemmGrouped<GemmKernel>;

int main(int argc, char** argv) {
  int nb = 4096, n = 256;
  size_t sz = (size_t)nb * n * n;
  double *A, *B, *C;
  cudaMalloc(&A, sz * 8); cudaMalloc(&B, sz * 8); cudaMalloc(&C, sz * 8);
  std::vector<double> h(sz); for (size_t i = 0; i < sz; ++i) h[i] = (i % 17) * 0.01;
  cudaMemcpy(A, h.data(), sz * 8, cudaMemcpyHostToDevice); cudaMemcpy(B, h.data(), sz * 8, cudaMemcpyHostToDevice);
  std::vector<cutlass::gemm::GemmCoord> ps(nb, cutlass::gemm::GemmCoord(n, n, n));
  std::vector<double*> pa(nb), pb(nb), pc(nb);
  std::vector<int64_t> ld(nb, n);
  for (int i = 0; i < nb; ++i) { pa[i] = A + (size_t)i * n * n; pb[i] = B + (size_t)i * n * n; pc[i] = C + (size_t)i * n * n; }
  cutlass::gemm::GemmCoord* dps; double **dpa, **dpb, **dpc; int64_t* dld;
  cudaMalloc(&dps, nb * sizeof(cutlass::gemm::GemmCoord)); cudaMalloc(&dpa, nb * 8); cudaMalloc(&dpb, nb * 8); cudaMalloc(&dpc, nb * 8); cudaMalloc(&dld, nb * 8);
  cudaMemcpy(dps, ps.data(), nb * sizeof(cutlass::gemm::GemmCoord), cudaMemcpyHostToDevice);
  cudaMemcpy(dpa, pa.data(), nb * 8, cudaMemcpyHostToDevice); cudaMemcpy(dpb, pb.data(), nb * 8, cudaMemcpyHostToDevice);
  cudaMemcpy(dpc, pc.data(), nb * 8, cudaMemcpyHostToDevice); cudaMemcpy(dld, ld.data(), nb * 8, cudaMemcpyHostToDevice);
  int tb = Gemm::sufficient(ps.data(), nb);
  printf("threadblock count %d\n", tb);
  typename Gemm::EpilogueOutputOp::Params ep(1.0, 0.0);
  typename Gemm::Arguments args(dps, nb, tb, ep, dpa, dpb, dpc, dpc, dld, dld, dld, dld, ps.data());
  Gemm gemm;
  size_t ws = gemm.get_workspace_size(args); void* wsp = nullptr; if (ws) cudaMalloc(&wsp, ws);
  auto st = gemm.initialize(args, wsp);
  printf("init %d\n", (int)st);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int r = 0; r < 3; ++r) gemm.run();
  cudaEventRecord(e0);
  for (int r = 0; r < 10; ++r) gemm.run();
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1); ms /= 10;
  printf("cutlass grouped 4096x256^3: %.3f ms %.1f TF (err %s)\n", ms, 2.0 * nb * n * n * (double)n / ms / 1e9, cudaGetErrorString(cudaGetLastError()));
  return 0;
}
