// Hardware probe for the B200 tile-path design (not product code).
//  mode "ldg"    : L2/HBM random row-gather bandwidth with LDG.128 (64/128/256 B rows)
//  mode "gather4": TMA tile::gather4 correctness + throughput (box rows 1 or 4)
//  mode "mma"    : tcgen05.mma bf16 with MN-major A (gathered X rows, SW128) and
//                  K-major B (16-row slab, SW128); M=128 and M=64 TMEM layouts
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o probe probe.cu
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <cstring>
#include <vector>
#include <random>
#include <cmath>
#include <algorithm>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s @%d: %s\n", #x, __LINE__, cudaGetErrorString(e)); exit(1);} } while (0)

static PFN_cuTensorMapEncodeTiled_v12000 encodeTiled = nullptr;
static void init_driver() {
  cudaDriverEntryPointQueryResult q;
  CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&encodeTiled, cudaEnableDefault, &q));
}

// ---------------------------------------------------------------- LDG gather
template <int VEC>  // 16-byte vectors per row
__global__ void gather_ldg(const uint4* __restrict__ table, const int* __restrict__ idx, long m, uint32_t* out) {
  constexpr int G = 32 / VEC;  // rows per warp per step
  int lane = threadIdx.x & 31;
  int sub = lane / VEC, v = lane % VEC;
  long warp = (blockIdx.x * (long)blockDim.x + threadIdx.x) >> 5;
  long nwarps = (gridDim.x * (long)blockDim.x) >> 5;
  uint32_t acc = 0;
  for (long base = warp * G * 4; base < m; base += nwarps * G * 4) {
    uint4 r[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      long k = base + u * G + sub;
      r[u] = make_uint4(0, 0, 0, 0);
      if (k < m) r[u] = __ldg(table + (long)idx[k] * VEC + v);
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) acc ^= r[u].x + r[u].y + r[u].z + r[u].w;
  }
  if (acc == 0x12345678) out[0] = acc;
}

__global__ void stream_read(const uint4* __restrict__ p, long n, uint32_t* out) {
  uint32_t acc = 0;
  for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < n; i += gridDim.x * (long)blockDim.x) {
    uint4 r = __ldg(p + i);
    acc ^= r.x + r.y + r.z + r.w;
  }
  if (acc == 0x12345678) out[0] = acc;
}

static void run_ldg() {
  int dev_sms = 148;
  std::mt19937_64 rng(1);
  uint32_t* dout; CK(cudaMalloc(&dout, 64));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  // HBM streaming read
  {
    long bytes = 4L << 30; uint4* p; CK(cudaMalloc(&p, bytes)); CK(cudaMemset(p, 1, bytes));
    for (int it = 0; it < 3; ++it) stream_read<<<dev_sms * 8, 256>>>(p, bytes / 16, dout);
    cudaEventRecord(e0);
    for (int it = 0; it < 5; ++it) stream_read<<<dev_sms * 8, 256>>>(p, bytes / 16, dout);
    cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); float ms; cudaEventElapsedTime(&ms, e0, e1);
    printf("stream_read 4GiB: %.1f GB/s\n", 5.0 * bytes / (ms * 1e-3) / 1e9);
    cudaFree(p);
  }
  long m = 64L << 20;  // 64M gathers
  std::vector<int> hidx(m);
  int* didx; CK(cudaMalloc(&didx, m * 4));
  for (long tbl_mb : {15L, 60L, 4096L}) {
    for (int dist = 0; dist < 2; ++dist) {
      for (int rowbytes : {64, 128, 256}) {
        long rows = (tbl_mb << 20) / rowbytes;
        // dist 0: uniform; dist 1: Chung-Lu capped power law, ids scrambled by multiplicative hash
        if (dist == 0) {
          std::uniform_int_distribution<long> U(0, rows - 1);
          for (long i = 0; i < m; ++i) hidx[i] = (int)U(rng);
        } else {
          std::vector<double> cdf(rows);
          double s = 0, i0 = 350.7 * rows / 232965.0;
          for (long i = 0; i < rows; ++i) { s += std::pow(1.0 + i / i0, -1.0 / 1.3); cdf[i] = s; }
          std::uniform_real_distribution<double> U(0, s);
          for (long i = 0; i < m; ++i) {
            long r = std::lower_bound(cdf.begin(), cdf.end(), U(rng)) - cdf.begin();
            if (r >= rows) r = rows - 1;
            hidx[i] = (int)((r * 2654435761L) % rows);
          }
        }
        CK(cudaMemcpy(didx, hidx.data(), m * 4, cudaMemcpyHostToDevice));
        uint4* tbl; CK(cudaMalloc(&tbl, rows * (long)rowbytes)); CK(cudaMemset(tbl, 1, rows * (long)rowbytes));
        auto launch = [&]() {
          if (rowbytes == 64) gather_ldg<4><<<dev_sms * 8, 256>>>(tbl, didx, m, dout);
          if (rowbytes == 128) gather_ldg<8><<<dev_sms * 8, 256>>>(tbl, didx, m, dout);
          if (rowbytes == 256) gather_ldg<16><<<dev_sms * 8, 256>>>(tbl, didx, m, dout);
        };
        for (int it = 0; it < 3; ++it) launch();
        cudaEventRecord(e0);
        for (int it = 0; it < 5; ++it) launch();
        cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); float ms; cudaEventElapsedTime(&ms, e0, e1);
        double gbs = 5.0 * m * rowbytes / (ms * 1e-3) / 1e9;
        printf("ldg_gather table=%ldMB dist=%s row=%dB : %.1f GB/s (%.3f ms per 64M rows)\n", tbl_mb,
               dist ? "powerlaw" : "uniform", rowbytes, gbs, ms / 5);
        cudaFree(tbl);
      }
    }
  }
}

// ---------------------------------------------------------------- PTX helpers
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, int cnt) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(cnt));
}
__device__ __forceinline__ void fence_barrier_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t phase) {
  asm volatile(
      "{\n .reg .pred P1;\n LAB_WAIT:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1, %2;\n"
      "@P1 bra DONE;\n bra LAB_WAIT;\n DONE:\n }" ::"r"(smem_u32(b)),
      "r"(phase), "r"(0x989680) : "memory");
}
__device__ __forceinline__ void gather4(const CUtensorMap* tm, uint64_t* bar, void* dst, int col, int r0, int r1, int r2, int r3) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cta.global.tile::gather4.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5, %6}], [%7];"
      ::"r"(smem_u32(dst)), "l"(tm), "r"(col), "r"(r0), "r"(r1), "r"(r2), "r"(r3), "r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ uint64_t make_sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo, uint32_t layout) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;  // version
  d |= (uint64_t)layout << 61;
  return d;
}
__device__ __forceinline__ void mma_bf16(uint32_t tmem, uint64_t ad, uint64_t bd, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n }" ::"r"(tmem),
      "l"(ad), "l"(bd), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar)) : "memory");
}

// ---------------------------------------------------------------- gather4 probe
// grid-persistent: each CTA gathers rows idx[...] in groups of BK rows per stage.
// verify mode: copy first stage's smem (un-swizzled) to out
template <int STAGES, int BK, int NBLK>  // NBLK = number of 64-col blocks (feat/64)
__global__ void __launch_bounds__(128, 1) gather4_kernel(const __grid_constant__ CUtensorMap tm, const int* __restrict__ idx, long m,
                                                        __nv_bfloat16* verify_out, int verify) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  constexpr int STAGE_BYTES = BK * 128 * NBLK;
  __shared__ uint64_t full[STAGES], empty[STAGES];
  int warp = threadIdx.x / 32, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
    fence_barrier_init();
  }
  __syncthreads();
  long nchunks = m / BK;
  if (warp == 0) {
    int stage = 0; uint32_t phase = 0;
    // warp-cooperative producer: lanes 0..BK/4-1 each own 4 rows of the chunk
    int4 nxt = make_int4(0, 0, 0, 0);
    long c = blockIdx.x;
    if (c < nchunks && lane < BK / 4) nxt = __ldg(reinterpret_cast<const int4*>(idx + c * BK) + lane);
    for (; c < nchunks; c += gridDim.x) {
      int4 cur = nxt;
      long cn = c + gridDim.x;
      if (cn < nchunks && lane < BK / 4) nxt = __ldg(reinterpret_cast<const int4*>(idx + cn * BK) + lane);
      mbar_wait(&empty[stage], phase ^ 1);
      if (lane == 0) mbar_expect_tx(&full[stage], STAGE_BYTES);
      __syncwarp();
      if (lane < BK / 4)
        for (int b = 0; b < NBLK; ++b)
          gather4(&tm, &full[stage], smem + stage * STAGE_BYTES + b * BK * 128 + lane * 4 * 128, b * 64, cur.x, cur.y, cur.z, cur.w);
      if (++stage == STAGES) { stage = 0; phase ^= 1; }
    }
  } else if (warp == 1) {
    int stage = 0; uint32_t phase = 0;
    for (long c = blockIdx.x; c < nchunks; c += gridDim.x) {
      mbar_wait(&full[stage], phase);
      if (verify && c < 4) {
        // un-swizzle: element (row r, feat f) at block b=f/64: byte = r*128 + ((f%64)*2)
        // swizzled chunk = (byte>>4) ^ (r&7)
        for (int e = lane; e < BK * 64 * NBLK; e += 32) {
          int r = e / (64 * NBLK), f = e % (64 * NBLK);
          int b = f / 64, ff = f % 64;
          int ch = ((ff * 2) >> 4) ^ (r & 7);
          int off = b * BK * 128 + r * 128 + ch * 16 + (ff * 2 & 15);
          verify_out[(c * BK + r) * 64 * NBLK + f] = *(__nv_bfloat16*)(smem + stage * STAGE_BYTES + off);
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[stage]);
      if (++stage == STAGES) { stage = 0; phase ^= 1; }
    }
  }
}

static void make_tmap(CUtensorMap* tm, void* base, long rows, int feat, int box_rows) {
  cuuint64_t gdim[2] = {(cuuint64_t)feat, (cuuint64_t)rows};
  cuuint64_t gstride[1] = {(cuuint64_t)feat * 2};
  cuuint32_t box[2] = {64, (cuuint32_t)box_rows};
  cuuint32_t es[2] = {1, 1};
  CUresult r = encodeTiled(tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, base, gdim, gstride, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                           CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("encodeTiled(feat=%d, box_rows=%d) -> %d\n", feat, box_rows, (int)r);
}

static void run_gather4(int box_rows) {
  init_driver();
  const int BK = 64, STAGES = 12;
  for (int feat : {64, 128, 32}) {
    int nblk = feat >= 64 ? feat / 64 : 1;
    long rows = 232965;
    std::vector<__nv_bfloat16> hx(rows * feat);
    for (long i = 0; i < rows * feat; ++i) hx[i] = __float2bfloat16((float)((i * 7919) % 1000) / 1000.0f);
    __nv_bfloat16* dx; CK(cudaMalloc(&dx, rows * feat * 2)); CK(cudaMemcpy(dx, hx.data(), rows * feat * 2, cudaMemcpyHostToDevice));
    long m = 32L << 20;
    std::vector<int> hidx(m);
    std::mt19937_64 rng(5); std::uniform_int_distribution<long> U(0, rows - 1);
    for (long i = 0; i < m; ++i) hidx[i] = (int)U(rng);
    int* didx; CK(cudaMalloc(&didx, m * 4)); CK(cudaMemcpy(didx, hidx.data(), m * 4, cudaMemcpyHostToDevice));
    CUtensorMap tm; make_tmap(&tm, dx, rows, feat, box_rows);
    __nv_bfloat16* vout; CK(cudaMalloc(&vout, 4L * BK * 64 * nblk * 2 * 148));
    int smem = STAGES * BK * 128 * nblk + 1024;
    auto kern = nblk == 1 ? gather4_kernel<STAGES, BK, 1> : gather4_kernel<STAGES, BK, 2>;
    CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    kern<<<148, 128, smem>>>(tm, didx, m, vout, 1);
    cudaError_t err = cudaDeviceSynchronize();
    printf("gather4 verify launch feat=%d: %s\n", feat, cudaGetErrorString(err));
    if (err != cudaSuccess) exit(2);
    // check the first 4 chunks of CTA 0..147
    std::vector<__nv_bfloat16> hv(4L * BK * 64 * nblk);
    CK(cudaMemcpy(hv.data(), vout, hv.size() * 2, cudaMemcpyDeviceToHost));
    long bad = 0, tot = 0;
    for (int c = 0; c < 4; ++c)
      for (int r = 0; r < BK; ++r)
        for (int f = 0; f < 64 * nblk; ++f) {
          // chunk c is handled by CTA c (c < 148)
          long row = hidx[(long)c * BK + r];
          float want = f < feat ? __bfloat162float(hx[row * feat + f]) : 0.0f;
          float got = __bfloat162float(hv[((long)c * BK + r) * 64 * nblk + f]);
          ++tot; if (want != got) { if (bad < 5) printf("  mismatch c%d r%d f%d want %f got %f\n", c, r, f, want, got); ++bad; }
        }
    printf("gather4 verify feat=%d: %ld / %ld mismatches\n", feat, bad, tot);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    for (int ctas_per_sm : {1}) {
      for (int it = 0; it < 2; ++it) kern<<<148 * ctas_per_sm, 128, smem>>>(tm, didx, m, vout, 0);
      cudaEventRecord(e0);
      for (int it = 0; it < 5; ++it) kern<<<148 * ctas_per_sm, 128, smem>>>(tm, didx, m, vout, 0);
      cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); float ms; cudaEventElapsedTime(&ms, e0, e1);
      double gbs = 5.0 * m * std::min(feat, 64 * nblk) * 2 / (ms * 1e-3) / 1e9;
      printf("gather4 throughput feat=%d ctas/sm=%d: %.1f GB/s useful (%.3f ms per 32M rows)\n", feat, ctas_per_sm, gbs, ms / 5);
    }
    cudaFree(dx); cudaFree(didx); cudaFree(vout);
  }
}

// ---------------------------------------------------------------- tcgen05 probe
// One CTA: gathers BK=64 X rows (feat=FEAT) via gather4 into MN-major SW128 A tile,
// builds a 16x64 K-major SW128 B slab from a dense host matrix, D[feat][16] = sum_k A[f][k] B[k][n]
// M = 128 (FEAT=128) or M=64 (FEAT=64). Dumps all 128 lanes x 16 cols of TMEM.
template <int FEAT, int MDIM>
__global__ void __launch_bounds__(128, 1) mma_probe(const __grid_constant__ CUtensorMap tm, const int* __restrict__ idx,
                                                   const __nv_bfloat16* __restrict__ slab, float* dump, int sbo_a_alias) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  constexpr int BK = 64, NBLK = FEAT / 64 > 0 ? FEAT / 64 : 1;
  uint8_t* a_s = smem;                          // NBLK * BK * 128
  uint8_t* b_s = smem + NBLK * BK * 128;        // 16 * 128 = 2048
  __shared__ uint64_t bar_full, bar_mma;
  __shared__ uint32_t tmem_base;
  int warp = threadIdx.x / 32, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) { mbar_init(&bar_full, 1); mbar_init(&bar_mma, 1); fence_barrier_init(); }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 32;" ::"r"(smem_u32(&tmem_base)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  // B slab: element (n, k) -> row n, 128B per row, swizzled
  for (int e = threadIdx.x; e < 16 * BK; e += blockDim.x) {
    int n = e / BK, k = e % BK;
    int ch = ((k * 2) >> 4) ^ (n & 7);
    int off = (n >> 3) * 1024 + (n & 7) * 128 + ch * 16 + (k * 2 & 15);
    *(__nv_bfloat16*)(b_s + off) = slab[n * BK + k];
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  uint32_t tmem = tmem_base;
  if (threadIdx.x == 0) {
    mbar_expect_tx(&bar_full, NBLK * BK * 128);
    for (int b = 0; b < NBLK; ++b)
      for (int r = 0; r < BK; r += 4) gather4(&tm, &bar_full, a_s + b * BK * 128 + r * 128, b * 64, idx[r], idx[r + 1], idx[r + 2], idx[r + 3]);
    mbar_wait(&bar_full, 0);
    asm volatile("tcgen05.fence::after_thread_sync;");
    // idesc: F32 accum, BF16 A/B, A MN-major, B K-major, N=16, M=MDIM
    uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | (1u << 15) | ((16u >> 3) << 17) | ((uint32_t)(MDIM >> 4) << 24);
    for (int k = 0; k < BK / 16; ++k) {
      uint64_t ad = make_sdesc(smem_u32(a_s) + k * 2048, sbo_a_alias ? 0 : BK * 128, 1024, 2);
      uint64_t bd = make_sdesc(smem_u32(b_s) + k * 32, 0, 1024, 2);
      mma_bf16(tmem, ad, bd, idesc, k > 0);
    }
    mma_commit(&bar_mma);
  }
  __syncwarp();
  mbar_wait(&bar_mma, 0);
  asm volatile("tcgen05.fence::after_thread_sync;");
  uint32_t r[16];
  uint32_t taddr = tmem + ((uint32_t)(warp * 32) << 16);
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]), "=r"(r[9]),
        "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
  for (int j = 0; j < 16; ++j) dump[(warp * 32 + lane) * 16 + j] = __uint_as_float(r[j]);
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 32;" ::"r"(tmem));
}

template <int FEAT, int MDIM>
static void run_mma_case(int alias) {
  const int BK = 64;
  long rows = 5000;
  std::vector<__nv_bfloat16> hx(rows * FEAT);
  std::mt19937 rng(3); std::uniform_real_distribution<float> U(-1, 1);
  for (auto& v : hx) v = __float2bfloat16(U(rng));
  std::vector<int> hidx(BK);
  for (int i = 0; i < BK; ++i) hidx[i] = (i * 977 + 13) % rows;
  std::vector<__nv_bfloat16> hs(16 * BK);
  for (int i = 0; i < 16 * BK; ++i) hs[i] = __float2bfloat16((i % 7 == 0) ? U(rng) : 0.0f);
  __nv_bfloat16 *dx, *ds; int* di; float* dd;
  CK(cudaMalloc(&dx, hx.size() * 2)); CK(cudaMalloc(&ds, hs.size() * 2)); CK(cudaMalloc(&di, BK * 4)); CK(cudaMalloc(&dd, 128 * 16 * 4));
  CK(cudaMemcpy(dx, hx.data(), hx.size() * 2, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(ds, hs.data(), hs.size() * 2, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(di, hidx.data(), BK * 4, cudaMemcpyHostToDevice));
  CK(cudaMemset(dd, 0, 128 * 16 * 4));
  CUtensorMap tm; make_tmap(&tm, dx, rows, FEAT, 1);
  int smem = 2 * BK * 128 + 2048 + 1024;
  CK(cudaFuncSetAttribute(mma_probe<FEAT, MDIM>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  mma_probe<FEAT, MDIM><<<1, 128, smem>>>(tm, di, ds, dd, alias);
  cudaError_t err = cudaDeviceSynchronize();
  printf("mma_probe FEAT=%d M=%d alias=%d: %s\n", FEAT, MDIM, alias, cudaGetErrorString(err));
  if (err != cudaSuccess) exit(3);
  std::vector<float> hd(128 * 16);
  CK(cudaMemcpy(hd.data(), dd, hd.size() * 4, cudaMemcpyDeviceToHost));
  // reference D[f][n] = sum_k X[idx[k]][f] * S[n][k]  (f < FEAT; for alias f>=FEAT maps to f-FEAT)
  int mism = 0;
  for (int f = 0; f < MDIM; ++f) {
    for (int n = 0; n < 16; ++n) {
      double want = 0; int ff = f % FEAT;
      for (int k = 0; k < BK; ++k) want += (double)__bfloat162float(hx[(long)hidx[k] * FEAT + ff]) * __bfloat162float(hs[n * BK + k]);
      // find which lane holds it
      int lane_found = -1;
      for (int l = 0; l < 128; ++l) if (fabs(hd[l * 16 + n] - want) < 1e-3 * (1 + fabs(want))) { lane_found = l; if (l == f) break; }
      if (n == 0 && (f < 4 || (f % 16) == 0 || lane_found != f)) printf("  D row f=%3d col0 want %+.5f lane(match)=%d lane[f]=%+.5f\n", f, want, lane_found, hd[f * 16 + n]);
      if (fabs(hd[f * 16 + n] - want) > 1e-3 * (1 + fabs(want))) ++mism;
    }
  }
  printf("mma_probe FEAT=%d M=%d alias=%d: %d mismatches assuming lane==row\n", FEAT, MDIM, alias, mism);
}

int main(int argc, char** argv) {
  const char* mode = argc > 1 ? argv[1] : "ldg";
  cudaDeviceProp p; CK(cudaGetDeviceProperties(&p, 0));
  printf("device %s sms=%d l2=%d MB smem/blk optin=%zu\n", p.name, p.multiProcessorCount, p.l2CacheSize >> 20, p.sharedMemPerBlockOptin);
  if (!strcmp(mode, "ldg")) run_ldg();
  if (!strcmp(mode, "gather4")) run_gather4(argc > 2 ? atoi(argv[2]) : 1);
  if (!strcmp(mode, "mma")) {
    init_driver();
    int which = argc > 2 ? atoi(argv[2]) : 0;
    if (which == 0) run_mma_case<128, 128>(0);
    if (which == 1) run_mma_case<64, 64>(0);
    if (which == 2) run_mma_case<64, 128>(1);
  }
  return 0;
}
