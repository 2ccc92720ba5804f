// Probe: legacy mma.sync m16n8k16 bf16 throughput per SM on B200 (not product code),
// registers only, W warps per CTA, independent accumulators (4 chains per warp).
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>

template <int CHAINS>
__global__ void k_hmma(float* out, int iters) {
  uint32_t a0 = threadIdx.x, a1 = a0 * 3, a2 = a0 * 5, a3 = a0 * 7, b0 = a0 * 11, b1 = a0 * 13;
  float c[CHAINS][4] = {};
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < CHAINS; ++k)
      asm volatile(
          "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
          : "+f"(c[k][0]), "+f"(c[k][1]), "+f"(c[k][2]), "+f"(c[k][3])
          : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
  }
  float s = 0;
#pragma unroll
  for (int k = 0; k < CHAINS; ++k) s += c[k][0] + c[k][1] + c[k][2] + c[k][3];
  if (s == 1234.5f) out[0] = s;
}

int main() {
  float* d; cudaMalloc(&d, 4);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int warps : {4, 8, 16, 32}) {
    int iters = 20000;
    k_hmma<4><<<148, warps * 32>>>(d, iters);
    cudaDeviceSynchronize();
    cudaEventRecord(e0);
    k_hmma<4><<<148, warps * 32>>>(d, iters);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double mmas = 148.0 * warps * iters * 4;
    printf("warps/SM=%2d: %.2f HMMA.16816 per SM per ns, %.1f TFLOP/s, %.2f cycles/HMMA/SM @1.9GHz\n", warps,
           mmas / 148 / (ms * 1e6), mmas * 4096 / (ms * 1e-3) / 1e12, 148 * (ms * 1e-3) * 1.9e9 / mmas);
  }
  return 0;
}
