// Probe (not product code): random 256-B X-row gathers into shared memory with one
// cp.async.bulk (TMA, non-tensor) per row, mbarrier completion.  Tells whether the TMA
// engine's per-copy rate can replace the LSU's cp.async (8 cycles per 512 B) on the tile path.
// P producer warps per CTA, each with its own ring of S stages x R rows.
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <vector>
#include <random>
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s: %s\n", #x, cudaGetErrorString(e)); exit(1);} } while (0)

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, int c) { asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(c)); }
__device__ __forceinline__ void expect_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t ph) {
  asm volatile("{\n .reg .pred P1;\n W:\n mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n @P1 bra D;\n bra W;\n D:\n }" ::"r"(su32(b)), "r"(ph) : "memory");
}
__device__ __forceinline__ void bulk(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               ::"r"(su32(dst)), "l"(src), "r"(bytes), "r"(su32(bar)) : "memory");
}

template <int ROWB, int R, int S>
__global__ void k_bulk(const uint8_t* __restrict__ tbl, const int* __restrict__ idx, long chunks_per_warp, int* out) {
  extern __shared__ __align__(128) uint8_t sm[];
  __shared__ uint64_t full[32][S];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint8_t* ring = sm + (size_t)warp * S * R * ROWB;
  if (lane < S) mbar_init(&full[warp][lane], 1);
  asm volatile("fence.mbarrier_init.release.cluster;");
  __syncwarp();
  const long gw = (long)blockIdx.x * (blockDim.x >> 5) + warp;
  const int* ip = idx + gw * chunks_per_warp * R;
  uint32_t sink = 0;
  for (long c = 0; c < chunks_per_warp + S - 1; ++c) {
    if (c >= S - 1) {  // consume chunk c - (S-1)
      const long cc = c - (S - 1);
      const int st = (int)(cc % S);
      mbar_wait(&full[warp][st], (uint32_t)((cc / S) & 1));
      sink ^= *(const uint32_t*)(ring + (size_t)st * R * ROWB + lane * 4);
      __syncwarp();
    }
    if (c < chunks_per_warp) {
      const int st = (int)(c % S);
      if (lane == 0) expect_tx(&full[warp][st], R * ROWB);
      __syncwarp();
      for (int r = lane; r < R; r += 32) {
        const int g = __ldg(ip + c * R + r);
        bulk(ring + (size_t)st * R * ROWB + r * ROWB, tbl + (long)g * ROWB, ROWB, &full[warp][st]);
      }
    }
  }
  if (sink == 0x12345678) out[0] = sink;
}

template <int ROWB, int R, int S>
void run(const uint8_t* tbl, const int* idx, long m, int* out) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int warps : {4, 8, 12, 16, 24, 32}) {
    const int smem = warps * S * R * ROWB;
    if (smem > 220 * 1024) continue;
    CK(cudaFuncSetAttribute(k_bulk<ROWB, R, S>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    const long nw = 148L * warps;
    const long cpw = m / (nw * R);
    k_bulk<ROWB, R, S><<<148, warps * 32, smem>>>(tbl, idx, cpw, out);
    CK(cudaDeviceSynchronize());
    cudaEventRecord(e0);
    k_bulk<ROWB, R, S><<<148, warps * 32, smem>>>(tbl, idx, cpw, out);
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double rows = (double)nw * cpw * R;
    printf("bulk rowB=%d R=%d S=%d warps/SM=%d: %.2f TB/s, %.1f cycles/row/SM @1.965GHz\n", ROWB, R, S, warps,
           rows * ROWB / (ms * 1e-3) / 1e12, ms * 1e-3 * 1.965e9 / (rows / 148));
  }
}

int main() {
  const long R = 232965, M = 1L << 24;
  std::mt19937_64 rng(1);
  std::vector<int> h(M);
  for (long i = 0; i < M; ++i) h[i] = (int)(rng() % R);
  int *idx, *out;
  uint8_t* tbl;
  CK(cudaMalloc(&idx, M * 4));
  CK(cudaMalloc(&tbl, R * 256));
  CK(cudaMalloc(&out, 4));
  CK(cudaMemcpy(idx, h.data(), M * 4, cudaMemcpyHostToDevice));
  CK(cudaMemset(tbl, 1, R * 256));
  run<256, 16, 3>(tbl, idx, M, out);
  run<256, 8, 4>(tbl, idx, M, out);
  run<128, 16, 4>(tbl, idx, M, out);
  return 0;
}
