// Probe: random-row gather throughput into shared memory on B200 (not product code).
//   mode 0: cp.async 16B (LDGSTS) ring, commit/wait_group pipelining, W warps/CTA
//   mode 1: LDG.128 -> registers -> STS.128, unrolled U rows in flight per warp
// rows of ROWB bytes (64/128/256) gathered from a table of R rows (L2-resident)
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <random>
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s: %s\n", #x, cudaGetErrorString(e)); exit(1);} } while (0)

__device__ __forceinline__ void cp16(unsigned dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
}
template <int N> __device__ __forceinline__ void cpwait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

// each warp gathers its own sequence of rows: per "step" 32*VECS/ (ROWB/16) rows
template <int ROWB, int DEPTH>
__global__ void k_ldgsts(const int4* __restrict__ tbl, const int* __restrict__ idx, long nsteps_per_warp, int* out) {
  extern __shared__ int4 sm[];
  constexpr int VPR = ROWB / 16;       // vectors per row
  constexpr int RPS = 32 / VPR * 4;    // rows per step (4 instrs per step)
  int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  long gw = blockIdx.x * (blockDim.x >> 5) + warp;
  int4* ring = sm + warp * (DEPTH + 1) * 128;  // 128 int4 (2 KB) per step slot
  unsigned rbase = (unsigned)__cvta_generic_to_shared(ring);
  const int* ip = idx + gw * nsteps_per_warp * RPS;
  for (long s = 0; s < nsteps_per_warp; ++s) {
    int slot = (int)(s % (DEPTH + 1));
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      int r = u * (32 / VPR) + lane / VPR, v = lane % VPR;
      int g = __ldg(ip + s * RPS + r);
      cp16(rbase + (slot * 128 + u * 32 + lane) * 16, tbl + (long)g * VPR + v);
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
    cpwait<DEPTH>();
  }
  cpwait<0>();
  __syncwarp();
  if (ring[lane].x == 0x7fffffff) out[0] = 1;
}

template <int ROWB, int U>
__global__ void k_ldg_sts(const int4* __restrict__ tbl, const int* __restrict__ idx, long nsteps_per_warp, int* out) {
  extern __shared__ int4 sm[];
  constexpr int VPR = ROWB / 16;
  constexpr int RPI = 32 / VPR;
  int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  long gw = blockIdx.x * (blockDim.x >> 5) + warp;
  int4* ring = sm + warp * U * 32;
  const int* ip = idx + gw * nsteps_per_warp * RPI * U;
  for (long s = 0; s < nsteps_per_warp; ++s) {
    int4 r[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      int g = __ldg(ip + (s * U + u) * RPI + lane / VPR);
      r[u] = __ldg(tbl + (long)g * VPR + lane % VPR);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) ring[u * 32 + lane] = r[u];
  }
  __syncwarp();
  if (ring[lane].x == 0x7fffffff) out[0] = 1;
}

int main() {
  long rows = 232965;
  int* dout; CK(cudaMalloc(&dout, 4));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int rowb : {64, 256}) {
    int4* tbl; CK(cudaMalloc(&tbl, rows * rowb)); CK(cudaMemset(tbl, 1, rows * rowb));
    long total_rows = 64L << 20;
    std::vector<int> h(total_rows); std::mt19937 rng(1); std::uniform_int_distribution<int> U(0, rows - 1);
    for (auto& v : h) v = U(rng);
    int* didx; CK(cudaMalloc(&didx, total_rows * 4)); CK(cudaMemcpy(didx, h.data(), total_rows * 4, cudaMemcpyHostToDevice));
    for (int mode = 0; mode < 2; ++mode) {
      for (int warps : {4, 8, 16}) {
        int ctas = 148;
        long nwarps = (long)ctas * warps;
        int vpr = rowb / 16;
        long rows_per_step = mode == 0 ? (32 / vpr) * 4 : (32 / vpr) * 8;
        long steps = total_rows / (nwarps * rows_per_step);
        size_t smem = mode == 0 ? (size_t)warps * 9 * 2048 : (size_t)warps * 8 * 512;
        auto launch = [&]() {
          if (mode == 0 && rowb == 64) { cudaFuncSetAttribute(k_ldgsts<64, 8>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem); k_ldgsts<64, 8><<<ctas, warps * 32, smem>>>(tbl, didx, steps, dout); }
          if (mode == 0 && rowb == 256) { cudaFuncSetAttribute(k_ldgsts<256, 8>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem); k_ldgsts<256, 8><<<ctas, warps * 32, smem>>>(tbl, didx, steps, dout); }
          if (mode == 1 && rowb == 64) { cudaFuncSetAttribute(k_ldg_sts<64, 8>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem); k_ldg_sts<64, 8><<<ctas, warps * 32, smem>>>(tbl, didx, steps, dout); }
          if (mode == 1 && rowb == 256) { cudaFuncSetAttribute(k_ldg_sts<256, 8>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem); k_ldg_sts<256, 8><<<ctas, warps * 32, smem>>>(tbl, didx, steps, dout); }
        };
        launch(); CK(cudaDeviceSynchronize());
        cudaEventRecord(e0);
        for (int i = 0; i < 5; ++i) launch();
        cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
        float ms; cudaEventElapsedTime(&ms, e0, e1); ms /= 5;
        double bytes = (double)steps * nwarps * rows_per_step * rowb;
        printf("mode=%s rowB=%d warps/CTA=%d : %.1f GB/s (%.3f ms)\n", mode == 0 ? "LDGSTS(depth8)" : "LDG->STS(U8)", rowb, warps,
               bytes / (ms * 1e-3) / 1e9, ms);
      }
    }
    cudaFree(tbl); cudaFree(didx);
  }
  return 0;
}
