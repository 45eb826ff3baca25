// Standalone timing of the diagonal-block factorization kernel (potrf_diag).
#include "../../paper_2502_02395_b200/csrc/panel.cu"
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cmath>
int h2g_set_error(int code, const char*, ...) { return code; }
int h2g_check_launch(const char* w) { cudaError_t e = cudaGetLastError(); if (e) { printf("%s: %s\n", w, cudaGetErrorString(e)); return 2; } return 0; }
int main(int argc, char** argv) {
  int nbox = argc > 1 ? atoi(argv[1]) : 256, n = 256;
  std::vector<double> h((size_t)nbox * n * n);
  srand(1);
  for (int bx = 0; bx < nbox; ++bx) {
    double* a = h.data() + (size_t)bx * n * n;
    std::vector<double> g(n * 64);
    for (auto& x : g) x = rand() / (double)RAND_MAX - 0.5;
    for (int i = 0; i < n; ++i) for (int j = 0; j < n; ++j) {
      double s = (i == j) ? 64.0 : 0.0;
      if (i < 64 && j < 64) for (int k = 0; k < 64; ++k) s += g[i * 64 + k] * g[j * 64 + k];
      a[(size_t)i * n + j] = s;
    }
  }
  double *dH, *dL; int* dnpd;
  cudaMalloc(&dH, h.size() * 8); cudaMalloc(&dL, (size_t)nbox * 4096 * 8); cudaMalloc(&dnpd, nbox * 4);
  std::vector<h2g_panel_desc> ds(nbox);
  for (int i = 0; i < nbox; ++i) ds[i] = {dH + (size_t)i * n * n, dL + (size_t)i * 4096, n, 64, 0, 64, i, 0};
  h2g_panel_desc* dd; cudaMalloc(&dd, nbox * sizeof(h2g_panel_desc));
  cudaMemcpy(dd, ds.data(), nbox * sizeof(h2g_panel_desc), cudaMemcpyHostToDevice);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int rep = 0; rep < 3; ++rep) {
    cudaMemcpy(dH, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
    cudaMemset(dnpd, 0x7f, nbox * 4);
    cudaEventRecord(e0);
    h2g_panel_potrf(dd, nbox, dnpd, 0);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    printf("rep %d nbox %d: %.1f us\n", rep, nbox, ms * 1e3);
  }
  // check: L L^T = D for box 0
  std::vector<double> L(n * n), Li(4096);
  cudaMemcpy(L.data(), dH, n * n * 8, cudaMemcpyDeviceToHost);
  cudaMemcpy(Li.data(), dL, 4096 * 8, cudaMemcpyDeviceToHost);
  double err = 0, erri = 0;
  for (int i = 0; i < 64; ++i) for (int j = 0; j <= i; ++j) {
    double s = 0, t = 0;
    for (int k = 0; k <= j; ++k) s += L[i * n + k] * L[j * n + k];
    err = fmax(err, fabs(s - h[(size_t)i * n + j]));
    for (int k = j; k <= i; ++k) t += Li[i * 64 + k] * L[k * n + j];
    erri = fmax(erri, fabs(t - (i == j)));
  }
  printf("max |LL^T - D| = %.3e   max |Linv L - I| = %.3e\n", err, erri);
  return 0;
}
