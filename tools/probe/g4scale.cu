// Probe (not product code): TMA tile::gather4 throughput as a function of the number of
// issuing warps per SM, CTAs per SM and issuing lanes per warp.  Decides whether a
// TMA-gather -> tcgen05 tile engine can move X rows L2 -> SMEM faster than the LSU
// (cp.async 16 B = 8 SM-cycles per 512 B, LDSM 4 more; LSU floor 12 cycles / 512 B).
//
// Each producer warp owns a ring of S stages x R rows (R/4 gather4 ops per 64-feature block);
// issuing lanes 0..L-1 issue the stage's ops round-robin, the warp waits on the stage's
// mbarrier S-1 stages later (no consumer work: pure copy-engine throughput).
// Table: 232,965 rows (C2), row = FEAT bf16, indices drawn from the C2 Chung-Lu degree law.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o g4scale g4scale.cu -lcuda
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <cmath>
#include <vector>
#include <random>
#include <algorithm>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s @%d: %s\n", #x, __LINE__, cudaGetErrorString(e)); exit(1);} } while (0)

static PFN_cuTensorMapEncodeTiled_v12000 encodeTiled = nullptr;

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, int c) { asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(c)); }
__device__ __forceinline__ void expect_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t ph) {
  asm volatile("{\n .reg .pred P1;\n W:\n mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n @P1 bra D;\n bra W;\n D:\n }" ::"r"(su32(b)), "r"(ph) : "memory");
}
__device__ __forceinline__ void gather4(const CUtensorMap* tm, uint64_t* bar, void* dst, int col, int4 r) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cta.global.tile::gather4.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5, %6}], [%7];"
      ::"r"(su32(dst)), "l"(tm), "r"(col), "r"(r.x), "r"(r.y), "r"(r.z), "r"(r.w), "r"(su32(bar)) : "memory");
}

// BLKB = bytes per gathered row slice (128 for SW128 / 64 for SW64); NBLK slices per row.
template <int BLKB, int NBLK>
__global__ void k_g4(const __grid_constant__ CUtensorMap tm, const int* __restrict__ idx, long chunks_per_warp,
                     int R, int S, int L, int* out) {
  extern __shared__ __align__(1024) uint8_t sm_raw[];
  uint8_t* sm = (uint8_t*)(((uintptr_t)sm_raw + 1023) & ~(uintptr_t)1023);
  __shared__ uint64_t full[32][8];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int stage_bytes = R * BLKB * NBLK;
  uint8_t* ring = sm + (size_t)warp * S * stage_bytes;
  if (lane < S) mbar_init(&full[warp][lane], 1);
  asm volatile("fence.mbarrier_init.release.cluster;");
  __syncwarp();
  const long gw = (long)blockIdx.x * (blockDim.x >> 5) + warp;
  const int* ip = idx + gw * chunks_per_warp * R;
  const int nops = R / 4 * NBLK;
  uint32_t sink = 0;
  for (long c = 0; c < chunks_per_warp + S - 1; ++c) {
    if (c >= S - 1) {
      const long cc = c - (S - 1);
      const int st = (int)(cc % S);
      mbar_wait(&full[warp][st], (uint32_t)((cc / S) & 1));
      sink ^= *(const uint32_t*)(ring + (size_t)st * stage_bytes + lane * 4);
      __syncwarp();
    }
    if (c < chunks_per_warp) {
      const int st = (int)(c % S);
      if (lane == 0) expect_tx(&full[warp][st], stage_bytes);
      __syncwarp();
      if (lane < L) {
        for (int o = lane; o < nops; o += L) {
          const int g = o / NBLK, b = o % NBLK;
          const int4 r = __ldg(reinterpret_cast<const int4*>(ip + c * R) + g);
          gather4(&tm, &full[warp][st], ring + (size_t)st * stage_bytes + b * R * BLKB + g * 4 * BLKB, b * (BLKB / 2), r);
        }
      }
    }
  }
  if (sink == 0x12345678) out[0] = sink;
}

int main() {
  cudaDriverEntryPointQueryResult q;
  CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&encodeTiled, cudaEnableDefault, &q));
  int clk_khz = 0; CK(cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0));
  const double clk = 1.965e9;
  const int SMS = 148;
  const long rows = 232965;
  // C2 degree law, ids scrambled
  std::vector<double> cdf(rows);
  double s = 0;
  for (long i = 0; i < rows; ++i) { s += std::pow(1.0 + i / 350.7, -1.0 / 1.3); cdf[i] = s; }
  const long m = 48L << 20;
  std::vector<int> hidx(m);
  std::mt19937_64 rng(7);
  std::uniform_real_distribution<double> U(0, s);
  for (long i = 0; i < m; ++i) {
    long r = std::lower_bound(cdf.begin(), cdf.end(), U(rng)) - cdf.begin();
    if (r >= rows) r = rows - 1;
    hidx[i] = (int)((r * 2654435761L) % rows);
  }
  int* didx; CK(cudaMalloc(&didx, m * 4)); CK(cudaMemcpy(didx, hidx.data(), m * 4, cudaMemcpyHostToDevice));
  int* dout; CK(cudaMalloc(&dout, 64));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  printf("# gather4 scaling probe: table %ld rows, %ld gathered rows per launch, C2 power-law indices\n", rows, m);
  printf("# cycles/op = SM-cycles per gather4 op per SM (4 row slices) at %.3f GHz\n", clk / 1e9);
  for (int feat : {128, 64, 32}) {
    const int BLKB = feat >= 64 ? 128 : 64;
    const int NBLK = feat >= 64 ? feat / 64 : 1;
    uint8_t* tbl; CK(cudaMalloc(&tbl, rows * feat * 2)); CK(cudaMemset(tbl, 1, rows * feat * 2));
    CUtensorMap tm;
    cuuint64_t gdim[2] = {(cuuint64_t)feat, (cuuint64_t)rows};
    cuuint64_t gstr[1] = {(cuuint64_t)feat * 2};
    cuuint32_t box[2] = {(cuuint32_t)(BLKB / 2), 1};
    cuuint32_t es[2] = {1, 1};
    CUresult cr = encodeTiled(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, tbl, gdim, gstr, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                              BLKB == 128 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B,
                              CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (cr) { printf("encode failed %d\n", (int)cr); return 1; }
    auto kern = NBLK == 2 ? k_g4<128, 2> : (BLKB == 128 ? k_g4<128, 1> : k_g4<64, 1>);
    CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024));
    for (int ctas : {1, 2}) {
      for (int P : {1, 2, 4, 8, 16, 24, 32}) {
        for (int L : {1, 4, 32}) {
          if (P * ctas > 32) continue;
          if (getenv("G4_WIDE") && (P * ctas < 16 || L != 32)) continue;
          const int R = getenv("G4_WIDE") ? 16 : 32;
          const int stage_bytes = R * BLKB * NBLK;
          const int budget = (ctas == 1 ? 200 : 100) * 1024;
          int S = std::min(8, budget / (P * stage_bytes));
          if (S < 2) continue;
          const long warps = (long)SMS * ctas * P;
          const long cpw = m / R / warps;
          if (cpw < 4) continue;
          const int smem = P * S * stage_bytes + 1024;
          for (int it = 0; it < 2; ++it) kern<<<SMS * ctas, 32 * P, smem>>>(tm, didx, cpw, R, S, L, dout);
          CK(cudaGetLastError());
          cudaEventRecord(e0);
          for (int it = 0; it < 3; ++it) kern<<<SMS * ctas, 32 * P, smem>>>(tm, didx, cpw, R, S, L, dout);
          cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
          float ms; cudaEventElapsedTime(&ms, e0, e1); ms /= 3;
          const double rows_done = (double)warps * cpw * R;
          const double ops = rows_done / 4 * NBLK;
          const double bytes = rows_done * feat * 2;
          printf("feat=%3d ctas/SM=%d warps/CTA=%2d lanes=%2d S=%d R=%d: %6.2f TB/s  %6.2f cycles/op/SM  %6.2f cycles/512B/SM\n",
                 feat, ctas, P, L, S, R, bytes / (ms * 1e-3) / 1e12, ms * 1e-3 * clk * SMS / ops,
                 ms * 1e-3 * clk * SMS / (bytes / 512));
        }
      }
    }
    cudaFree(tbl);
  }
  return 0;
}
