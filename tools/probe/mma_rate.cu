// Probe: tcgen05.mma issue/throughput on one SM for small-N shapes (not product code).
// Each CTA issues ITER MMAs back-to-back from fixed smem descriptors (zero data)
// and reports cycles per MMA.  Variants: M in {64,128}, N in {16..256}, A K- or MN-major.
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s: %s\n", #x, cudaGetErrorString(e)); return 1;} } while (0)

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;
  return d;
}

template <int M, int N, int AMN, int COMMIT_EVERY = 0, int CYCLE = 0, int NOISE = 0>
__global__ void __launch_bounds__(256, 1) k_rate(long long* out, int iters) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* s = (uint8_t*)(((uintptr_t)sm + 1023) & ~(uintptr_t)1023);
  __shared__ uint32_t tslot;
  __shared__ uint64_t bar, bar2;
  int warp = threadIdx.x / 32;
  for (int i = threadIdx.x; i < 64 * 1024 / 4; i += blockDim.x) ((uint32_t*)s)[i] = 0;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1000000;" ::"r"(smem_u32(&bar2)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(smem_u32(&tslot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  uint32_t tmem = tslot;
  if (threadIdx.x == 0) {
    uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)AMN << 15) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
    uint32_t a = smem_u32(s), b = smem_u32(s + 32768);
    uint64_t ad = AMN ? sdesc(a, 8192, 1024) : sdesc(a, 0, 1024);
    uint64_t bd = sdesc(b, 0, 1024);
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
      uint64_t adi = ad, bdi = bd;
      if (CYCLE) { adi = ad + (uint64_t)(((i % 10) * 2048) >> 4); bdi = bd + (uint64_t)((((i & 3) * 32)) >> 4); }
      asm volatile("{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n }"
                   ::"r"(tmem), "l"(adi), "l"(bdi), "r"(idesc), "r"(1));
      if (COMMIT_EVERY && (i % COMMIT_EVERY) == COMMIT_EVERY - 1)
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar2)));
    }
    long long t1 = clock64();
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)));
    asm volatile("{\n .reg .pred P1;\n W:\n mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n @P1 bra D;\n bra W;\n D:\n }" ::"r"(smem_u32(&bar)));
    long long t2 = clock64();
    out[blockIdx.x * 2] = t1 - t0;
    out[blockIdx.x * 2 + 1] = t2 - t0;
  }
  if (NOISE && warp >= 4) {  // smem write traffic from 4 other warps (like cp.async landing)
    int4* q = (int4*)(s + 40960);
    for (int i = 0; i < iters * 8; ++i) q[(i * 32 + threadIdx.x) & 2047] = make_int4(i, i, i, i);
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tmem));
}

template <int M, int N, int AMN, int CE = 0, int CY = 0, int NO = 0>
int run() {
  long long* d; CK(cudaMalloc(&d, 148 * 16));
  int smem = 64 * 1024 + 1024;
  CK(cudaFuncSetAttribute(k_rate<M, N, AMN, CE, CY, NO>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  int iters = 4096;
  k_rate<M, N, AMN, CE, CY, NO><<<148, 256, smem>>>(d, iters);
  CK(cudaDeviceSynchronize());
  k_rate<M, N, AMN, CE, CY, NO><<<148, 256, smem>>>(d, iters);
  CK(cudaDeviceSynchronize());
  long long h[2]; CK(cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost));
  printf("commit%d cycle%d noise%d M=%3d N=%3d A=%s : issue %.1f cyc/mma, complete %.1f cyc/mma  (%.0f MAC/cyc)\n", CE, CY, NO, M, N, AMN ? "MN" : "K ",
         (double)h[0] / iters, (double)h[1] / iters, (double)M * N * 16 / ((double)h[1] / iters));
  cudaFree(d);
  return 0;
}

int main() {
  run<128, 16, 1>(); run<128, 16, 1, 4>(); run<128, 16, 1, 4, 1>(); run<128, 16, 1, 4, 1, 1>(); run<128, 16, 1, 0, 0, 1>();
  run<64, 16, 1, 4, 1>(); run<128, 64, 1, 4, 1>();
  return 0;
}
