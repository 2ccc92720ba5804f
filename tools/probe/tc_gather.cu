// Probe (not product code): does tcgen05.mma reading cp.async-staged rows from shared memory
// compete with the LDGSTS gather for the SM's L1/shared-memory bandwidth?
//
// k_tile_warp is bound at 8 + 4 LSU cycles per 512 B gathered (LDGSTS + ldmatrix of the same
// bytes).  A tcgen05 engine would drop the ldmatrix (the tensor core reads
// shared memory through descriptors).  This probe runs the bare data flow of such an engine:
// a CTA of 128 threads gathers 64 random 256-B rows (128 bf16 features) per chunk into an
// S-stage ring (SW128 MN-major, two 64-feature blocks), and
//   mode 0: gather only (the ingest ceiling),
//   mode 1: + one elected thread issues 4 x tcgen05.mma (M = 128 features, N = 16 rows,
//           K = 16) on each landed chunk against a 16 x 64 slab, committing to the stage's
//           mbarrier, which the gather waits on before reusing the stage,
//   mode 2: + mma.sync from ldmatrix.trans of the chunk (every warp 16 of the 64 rows x all
//           128 features, i.e. the LSU traffic of k_tile_warp's compute step).
// Reports SM cycles per 512 B gathered.
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <random>
#include <vector>

#define CK(x)                                                                          \
  do {                                                                                 \
    cudaError_t e = (x);                                                               \
    if (e != cudaSuccess) {                                                            \
      printf("CUDA %s: %s\n", #x, cudaGetErrorString(e));                              \
      exit(1);                                                                         \
    }                                                                                  \
  } while (0)

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void cp16(uint32_t dst, const void* src, uint64_t pol) {
  asm volatile("cp.async.cg.shared.global.L2::cache_hint [%0], [%1], 16, %2;" ::"r"(dst), "l"(src), "l"(pol)
               : "memory");
}
template <int N>
__device__ __forceinline__ void cpwait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ void mbar_init(uint64_t* b, int cnt) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(cnt));
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t phase) {
  asm volatile(
      "{\n .reg .pred p;\n W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra W;\n }" ::"r"(
          smem_u32(b)),
      "r"(phase)
      : "memory");
}
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;  // SWIZZLE_128B
  return d;
}
__host__ __device__ constexpr uint32_t idesc(uint32_t m, uint32_t n) {  // bf16 x bf16 -> f32, A MN-major, B K-major
  return (1u << 4) | (1u << 7) | (1u << 10) | (1u << 15) | (0u << 16) | ((n >> 3) << 17) | ((m >> 4) << 24);
}
__device__ __forceinline__ void umma(uint32_t tmem, uint64_t ad, uint64_t bd, uint32_t id, uint32_t acc) {
  asm volatile(
      "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n }" ::"r"(tmem),
      "l"(ad), "l"(bd), "r"(id), "r"(acc));
}
__device__ __forceinline__ void ldsm_x4_trans(uint32_t addr, uint32_t (&r)[4]) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(addr));
}
__device__ __forceinline__ void hmma(float (&d)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

template <int MODE, int S, int R = 64>
__global__ void __launch_bounds__(128) k_tc(const uint8_t* __restrict__ tbl, const int* __restrict__ idx, int nidx,
                                           long chunks, float* out) {
  constexpr int kStage = R * 256;  // R rows x 256 B
  constexpr int NC = R / 8;          // copies per thread per chunk
  extern __shared__ uint8_t raw[];
  uint8_t* sm = (uint8_t*)(((uintptr_t)raw + 1023) & ~(uintptr_t)1023);
  const uint32_t a0 = smem_u32(sm), slab = a0 + S * kStage;
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm + S * kStage + 2048);
  uint32_t* tslot = reinterpret_cast<uint32_t*>(bar + S);
  const int t = threadIdx.x, warp = t >> 5, lane = t & 31;
  for (int i = t; i < 2048 / 4; i += 128) reinterpret_cast<uint32_t*>(sm + S * kStage)[i] = 0x3c003c00u ^ (i & 0x0101);
  if (t == 0) {
    for (int s = 0; s < S; ++s) mbar_init(&bar[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (MODE == 1 && warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 32;" ::"r"(smem_u32(tslot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = MODE == 1 ? *tslot : 0u;
  uint64_t keep;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(keep));
  // thread t copies vector v = t % 16 of rows t/16 + 8i
  const int v = t & 15, rb = t >> 4;
  uint32_t dofs[NC];
#pragma unroll
  for (int i = 0; i < NC; ++i) {
    const int r = rb + 8 * i;
    dofs[i] = (uint32_t)(v >> 3) * (R * 128u) + (uint32_t)r * 128u + ((uint32_t)((v & 7) ^ (r & 7)) << 4);
  }
  constexpr int D = S - 2;  // chunks in flight beyond the one being multiplied
  float acc[8][4] = {};
  const long base = (long)blockIdx.x * chunks;
  for (long c = 0; c < chunks + D; ++c) {
    if (c < chunks) {
      const int s = (int)(c % S);
      if (MODE == 1 && c >= S) mbar_wait(&bar[s], (uint32_t)(((c / S) - 1) & 1));
      const int* ip = idx + ((base + c) * R) % nidx;
#pragma unroll
      for (int i = 0; i < NC; ++i) {
        const int g = __ldg(ip + rb + 8 * i);
        cp16(a0 + s * kStage + dofs[i], tbl + (size_t)g * 256 + v * 16, keep);
      }
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
    cpwait<D>();
    const long cm = c - D;  // chunk to multiply
    if (MODE == 1) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    if (cm < 0) continue;
    const int sm_ = (int)(cm % S);
    if (MODE == 1) {
      if (t == 0) {
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
#pragma unroll
        for (int k = 0; k < R / 16; ++k) {
          const uint64_t ad = sdesc(a0 + sm_ * kStage + k * 2048, R * 128, 1024);
          const uint64_t bd = sdesc(slab + k * 32, 0, 1024);
          umma(tmem, ad, bd, idesc(128, 16), (cm == 0 && k == 0) ? 0u : 1u);
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                         smem_u32(&bar[sm_]))
                     : "memory");
      }
    } else if (MODE == 2) {
      // warp w: k rows 16w..16w+15, all 128 features (16 n8 tiles): 8 ldmatrix.x4.trans
      if (16 * warp >= R) continue;
      uint32_t a[4] = {0x3c003c00u, 0x3c003c00u, 0x3c003c00u, 0x3c003c00u};
      const int kr = 16 * warp + (lane & 7) + ((lane >> 3) & 1) * 8, fc = lane >> 4;
#pragma unroll
      for (int nb = 0; nb < 8; ++nb) {  // 16 features per ldmatrix.x4 (two n8 tiles)
        const int vv = nb * 2 + fc;     // 16-B vector 0..15
        const uint32_t addr =
            a0 + sm_ * kStage + (uint32_t)(vv >> 3) * (R * 128u) + kr * 128u + ((uint32_t)((vv & 7) ^ (kr & 7)) << 4);
        uint32_t b[4];
        ldsm_x4_trans(addr, b);
        hmma(acc[nb], a, b[0], b[1]);
        hmma(acc[nb], a, b[2], b[3]);
      }
    }
  }
  if (MODE == 1) {
    const long last = chunks - 1;
    mbar_wait(&bar[last % S], (uint32_t)((last / S) & 1));
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 32;" ::"r"(tmem));
  }
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += acc[i][0] + acc[i][1] + acc[i][2] + acc[i][3];
  if (s == 1234.5f) out[0] = s;
}

template <int MODE, int S, int R = 64>
void run(const uint8_t* tbl, const int* idx, int nidx, int cps, int sms, float* out, double clock_ghz) {
  constexpr int kStage = R * 256;
  const long chunks = 4096 * 64 / R;
  const int smem = S * kStage + 2048 + 8 * S + 16 + 1024;
  CK(cudaFuncSetAttribute(k_tc<MODE, S, R>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  const int grid = sms * cps;
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  k_tc<MODE, S, R><<<grid, 128, smem>>>(tbl, idx, nidx, 256, out);
  CK(cudaGetLastError());
  CK(cudaDeviceSynchronize());
  CK(cudaEventRecord(e0));
  k_tc<MODE, S, R><<<grid, 128, smem>>>(tbl, idx, nidx, chunks, out);
  CK(cudaEventRecord(e1));
  CK(cudaEventSynchronize(e1));
  CK(cudaGetLastError());
  float ms;
  CK(cudaEventElapsedTime(&ms, e0, e1));
  const double bytes = (double)grid * chunks * kStage;
  const double cyc512 = ms * 1e-3 * clock_ghz * 1e9 * sms / (bytes / 512);
  printf("mode %d  rows/chunk %d  S %d  CTAs/SM %d  smem %6d  %8.3f ms  %6.2f TB/s  %5.2f SM-cycles per 512 B\n", MODE, R, S, cps,
         smem, ms, bytes / (ms * 1e-3) / 1e12, cyc512);
}

int main() {
  int dev = 0, sms = 0, clk = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  CK(cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev));
  const double ghz = clk / 1e6;
  const int rows = 232965;
  uint8_t* tbl;
  CK(cudaMalloc(&tbl, (size_t)rows * 256));
  CK(cudaMemset(tbl, 0, (size_t)rows * 256));
  const int nidx = 1 << 24;
  std::vector<int> h(nidx);
  std::mt19937 rng(1);
  for (auto& x : h) x = (int)(rng() % rows);
  int* idx;
  CK(cudaMalloc(&idx, nidx * 4));
  CK(cudaMemcpy(idx, h.data(), nidx * 4, cudaMemcpyHostToDevice));
  float* out;
  CK(cudaMalloc(&out, 4));
  printf("SMs %d, clock %.3f GHz; 64 random 256-B rows per chunk, 60 MB table\n", sms, ghz);
  for (int cps = 1; cps <= 3; ++cps) {
    run<0, 4>(tbl, idx, nidx, cps, sms, out, ghz);
    run<1, 4>(tbl, idx, nidx, cps, sms, out, ghz);
    run<2, 4>(tbl, idx, nidx, cps, sms, out, ghz);
  }
  for (int cps = 1; cps <= 2; ++cps) {
    run<0, 6>(tbl, idx, nidx, cps, sms, out, ghz);
    run<1, 6>(tbl, idx, nidx, cps, sms, out, ghz);
    run<2, 6>(tbl, idx, nidx, cps, sms, out, ghz);
  }
  run<0, 3>(tbl, idx, nidx, 4, sms, out, ghz);
  run<1, 3>(tbl, idx, nidx, 4, sms, out, ghz);
  run<2, 3>(tbl, idx, nidx, 4, sms, out, ghz);
  for (int cps = 4; cps <= 8; cps += 2) {
    run<0, 4, 32>(tbl, idx, nidx, cps, sms, out, ghz);
    run<1, 4, 32>(tbl, idx, nidx, cps, sms, out, ghz);
    run<2, 4, 32>(tbl, idx, nidx, cps, sms, out, ghz);
  }
  run<0, 3, 32>(tbl, idx, nidx, 8, sms, out, ghz);
  run<1, 3, 32>(tbl, idx, nidx, 8, sms, out, ghz);
  return 0;
}
