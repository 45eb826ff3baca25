// Standalone timing of the fused Cholesky panel kernel (h2g_chol_panel) and of
// the stand-alone DIAG kernel, with per-phase clock64 tracing of CTA 0.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 [-DH2G_DIAG_BS=2] \
//        -o panel_bench tools/microbench/panel_bench.cu
// Usage: panel_bench nbox n p
#define H2G_PANEL_TRACE 1
#include "../../paper_2502_02395_b200/csrc/panel.cu"
#include <cmath>
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
  int nbox = argc > 1 ? atoi(argv[1]) : 256, n = argc > 2 ? atoi(argv[2]) : 256, p = argc > 3 ? atoi(argv[3]) : 64;
  int b = 64;
  std::vector<double> h((size_t)nbox * n * n);
  srand(1);
  for (auto& x : h) x = (rand() / (double)RAND_MAX - 0.5) * 0.01;
  for (int bx = 0; bx < nbox; ++bx)
    for (int i = 0; i < n; ++i) h[(size_t)bx * n * n + (size_t)i * n + i] = 4.0;
  double *dH, *dL; int* dnpd;
  cudaMalloc(&dH, h.size() * 8); cudaMalloc(&dL, (size_t)nbox * 4096 * 8);
  cudaMalloc(&dnpd, nbox * 4);
  int tiles = h2g_chol_panel_tiles(n, p, b);
  std::vector<h2g_chol_panel_desc> ds(nbox);
  std::vector<int> map;
  for (int i = 0; i < nbox; ++i) {
    ds[i] = {dH + (size_t)i * n * n, dL + (size_t)i * 4096, n, 64, n, p, b, i, i * tiles, 0};
    for (int t = 0; t < tiles; ++t) map.push_back(i);
  }
  h2g_chol_panel_desc* dd; int* dmap;
  cudaMalloc(&dd, nbox * sizeof(h2g_chol_panel_desc)); cudaMalloc(&dmap, map.size() * 4);
  cudaMemcpy(dd, ds.data(), nbox * sizeof(h2g_chol_panel_desc), cudaMemcpyHostToDevice);
  cudaMemcpy(dmap, map.data(), map.size() * 4, cudaMemcpyHostToDevice);
  std::vector<h2g_panel_desc> pd(nbox);
  for (int i = 0; i < nbox; ++i) pd[i] = {dH + (size_t)i * n * n, dL + (size_t)i * 4096, n, 64, p, b, i, 0};
  h2g_panel_desc* dpd; cudaMalloc(&dpd, nbox * sizeof(h2g_panel_desc));
  cudaMemcpy(dpd, pd.data(), nbox * sizeof(h2g_panel_desc), cudaMemcpyHostToDevice);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int rep = 0; rep < 3; ++rep) {
    cudaMemcpy(dH, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
    cudaEventRecord(e0);
    h2g_chol_panel(dd, nbox, dmap, (int)map.size(), dnpd, 0);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    long long tr[32]; cudaMemcpyFromSymbol(tr, h2g::g_panel_trace, sizeof(tr));
    printf("chol_panel nbox %d n %d p %d row CTAs %zu: %.1f us | rows kernel cycles from start:", nbox, n, p, map.size(), ms * 1e3);
    for (int k = 1; k <= 5; ++k) printf(" %d:%lld", k, tr[k] - tr[0]);
    printf("\n");
  }
  for (int rep = 0; rep < 3; ++rep) {
    cudaMemcpy(dH, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
    cudaEventRecord(e0);
    h2g_panel_potrf(dpd, nbox, dnpd, 0);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    long long tr[32]; cudaMemcpyFromSymbol(tr, h2g::g_panel_trace, sizeof(tr));
    printf("potrf_diag nbox %d: %.1f us | cycles from start: load %lld factor %lld [", nbox, ms * 1e3, tr[11] - tr[10], tr[12] - tr[11]);
    for (int k = 16; k <= 26; ++k) printf(" %lld", tr[k] - tr[16]);
    printf(" ]\n");
  }
  // check box 0: L_pp L_pp^T = D - X X^T (X = H[p:p+b, p-64:p]) and Linv L = I
  std::vector<double> Lp(4096), Li(4096);
  cudaMemcpy(dH, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
  h2g_chol_panel(dd, nbox, dmap, (int)map.size(), dnpd, 0);
  std::vector<double> hh((size_t)n * n);
  cudaMemcpy(hh.data(), dH, (size_t)n * n * 8, cudaMemcpyDeviceToHost);
  for (int i = 0; i < 64; ++i) for (int j = 0; j < 64; ++j) Lp[i * 64 + j] = j <= i ? hh[(size_t)(p + i) * n + p + j] : 0.0;
  cudaMemcpy(Li.data(), dL, 4096 * 8, cudaMemcpyDeviceToHost);
  double err = 0, erri = 0;
  for (int i = 0; i < b; ++i) for (int j = 0; j <= i; ++j) {
    double s = 0, t = 0, ref = h[(size_t)(p + i) * n + p + j];
    if (p > 0) for (int k = p - 64; k < p; ++k) ref -= h[(size_t)(p + i) * n + k] * h[(size_t)(p + j) * n + k];
    for (int k = 0; k <= j; ++k) s += Lp[i * 64 + k] * Lp[j * 64 + k];
    err = fmax(err, fabs(s - ref));
    for (int k = j; k <= i; ++k) t += Li[i * 64 + k] * Lp[k * 64 + j];
    erri = fmax(erri, fabs(t - (i == j)));
  }
  printf("max |LL^T - D'| = %.3e   max |Linv L - I| = %.3e\n", err, erri);
  return 0;
}
