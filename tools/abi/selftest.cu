// Standalone C-ABI self test (no torch): partition + tile plan + spmm on a tiny CSR.
#include <cstdio>
#include <vector>
#include <cuda_runtime.h>
#include "../../include/hcspmm.h"
#define CK(x) do { int rc = (x); if (rc) { printf("%s -> %d: %s\n", #x, rc, hcs_last_error()); return 1; } } while (0)
int main() {
  int n = 40, ncol = 30;
  std::vector<long long> rp(n + 1, 0);
  std::vector<int> ci;
  for (int r = 0; r < n; ++r) { for (int c = r % 3; c < ncol; c += 4) ci.push_back(c); rp[r + 1] = ci.size(); }
  long long nnz = ci.size();
  int64_t *d_rp; int32_t* d_ci;
  cudaMalloc(&d_rp, 8 * (n + 1)); cudaMalloc(&d_ci, 4 * nnz);
  cudaMemcpy(d_rp, rp.data(), 8 * (n + 1), cudaMemcpyHostToDevice);
  cudaMemcpy(d_ci, ci.data(), 4 * nnz, cudaMemcpyHostToDevice);
  int W = (n + 15) / 16;
  size_t wsb = 0;
  CK(hcs_partition_workspace_bytes(n, ncol, nnz, 16, &wsb));
  printf("ws bytes %zu\n", wsb);
  void* ws; cudaMalloc(&ws, wsb + 16);
  int64_t* wcp; double *dens, *ci2; uint8_t* codes; double* sel;
  cudaMalloc(&wcp, 8 * (W + 1)); cudaMalloc(&dens, 8 * W); cudaMalloc(&ci2, 8 * W); cudaMalloc(&codes, W);
  double hsel[7] = {-0.1454848214145233, -9.249873814861964, -15.105252482198011, 140.38659793814432, 0.5, 123.08273985946481, 0.2570676399373035};
  cudaMalloc(&sel, 56); cudaMemcpy(sel, hsel, 56, cudaMemcpyHostToDevice);
  printf("calling count\n"); fflush(stdout);
  CK(hcs_partition_count(d_rp, d_ci, n, ncol, nnz, 16, hsel, wcp, dens, ci2, codes, ws, wsb, nullptr));
  cudaDeviceSynchronize();
  std::vector<long long> hw(W + 1);
  cudaMemcpy(hw.data(), wcp, 8 * (W + 1), cudaMemcpyDeviceToHost);
  for (int i = 0; i <= W; ++i) printf("wcp[%d]=%lld\n", i, hw[i]);
  int32_t *nzc, *cond; cudaMalloc(&nzc, 4 * hw[W] + 4); cudaMalloc(&cond, 4 * nnz);
  CK(hcs_partition_fill(d_rp, d_ci, n, ncol, nnz, 16, wcp, nzc, cond, ws, wsb, nullptr));
  printf("sync: %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  return 0;
}
