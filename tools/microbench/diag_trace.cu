// Phase timeline (clock64 of CTA 0, thread 0) of the diagonal-block factorization
// inside chol_diag_kernel: 16 start, 17+2kb after chol16 of block kb, 18+2kb after
// its TRSM/trailing update, 25 before the L^-1 off-diagonal blocks, 26 end.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o diag_trace tools/microbench/diag_trace.cu
// Usage: diag_trace nbox
#define H2G_PANEL_TRACE 1
#include "../../paper_2502_02395_b200/csrc/panel.cu"
#include <cstdio>
#include <cstdlib>
#include <vector>
int h2g_set_error(int code, const char*, ...) { return code; }
int h2g_check_launch(const char* w) {
  cudaError_t e = cudaGetLastError();
  if (e) { printf("%s: %s\n", w, cudaGetErrorString(e)); return 2; }
  return 0;
}
int main(int argc, char** argv) {
  const int nbox = argc > 1 ? atoi(argv[1]) : 1, n = 64;
  std::vector<double> h((size_t)nbox * n * n);
  srand(1);
  for (auto& x : h) x = (rand() / (double)RAND_MAX - 0.5) * 0.01;
  for (int b = 0; b < nbox; ++b)
    for (int i = 0; i < n; ++i) h[(size_t)b * n * n + i * n + i] = 4.0;
  double *dH, *dL; int* dnpd;
  cudaMalloc(&dH, h.size() * 8); cudaMalloc(&dL, (size_t)nbox * 4096 * 8); cudaMalloc(&dnpd, nbox * 4);
  std::vector<h2g_chol_panel_desc> ds(nbox);
  for (int i = 0; i < nbox; ++i) ds[i] = {dH + (size_t)i * n * n, dL + (size_t)i * 4096, n, 64, n, 0, 64, i, 0, 0};
  h2g_chol_panel_desc* dd; cudaMalloc(&dd, nbox * sizeof(h2g_chol_panel_desc));
  cudaMemcpy(dd, ds.data(), nbox * sizeof(h2g_chol_panel_desc), cudaMemcpyHostToDevice);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int rep = 0; rep < 4; ++rep) {
    cudaMemcpy(dH, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
    cudaEventRecord(e0);
    h2g_chol_panel(dd, nbox, nullptr, 0, dnpd, 0);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    long long tr[32]; cudaMemcpyFromSymbol(tr, h2g::g_panel_trace, sizeof(tr));
    printf("nbox %d: %.1f us | cycles from 16:", nbox, ms * 1e3);
    for (int k = 17; k <= 26; ++k) printf(" %d:%lld", k, tr[k] - tr[16]);
    printf("\n");
  }
  return 0;
}
