// Probe (not product code): random-row gather L2 -> registers with LDG.128, no shared memory.
// Table of R rows x ROWB bytes (L2-resident at 233K x 256 B = 60 MB), M random indices.
// Each warp: per step U independent row groups in flight; lanes cover a row with ROWB/16
// lanes.  Variants: plain __ldg, L1::no_allocate, evict_last policy.  Reports TB/s delivered.
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <vector>
#include <random>
#include <cstdlib>
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s: %s\n", #x, cudaGetErrorString(e)); exit(1);} } while (0)

template <int MODE>
__device__ __forceinline__ uint4 ld16(const uint4* p, uint64_t pol) {
  uint4 v;
  if (MODE == 0) {
    v = __ldg(p);
  } else if (MODE == 1) {
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
  } else {
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.u32 {%0,%1,%2,%3}, [%4], %5;"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p), "l"(pol));
  }
  return v;
}

template <int VEC, int U, int MODE>
__global__ void k_gather(const uint4* __restrict__ table, const int* __restrict__ idx, long m, uint32_t* out) {
  constexpr int G = 32 / VEC;
  const int lane = threadIdx.x & 31, sub = lane / VEC, v = lane % VEC;
  const long warp = (blockIdx.x * (long)blockDim.x + threadIdx.x) >> 5;
  const long nwarps = (gridDim.x * (long)blockDim.x) >> 5;
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  uint32_t acc = 0;
  long base = warp * G * U;
  int g[U];
#pragma unroll
  for (int u = 0; u < U; ++u) g[u] = base + u * G + sub < m ? __ldg(idx + ((base + u * G + sub) & ((1 << 22) - 1))) : 0;
  for (; base < m; base += nwarps * G * U) {
    const long nb = base + nwarps * G * U;
    int gn[U];
#pragma unroll
    for (int u = 0; u < U; ++u) gn[u] = nb + u * G + sub < m ? __ldg(idx + ((nb + u * G + sub) & ((1 << 22) - 1))) : 0;
    uint4 r[U];
#pragma unroll
    for (int u = 0; u < U; ++u) r[u] = ld16<MODE>(table + (long)g[u] * VEC + v, pol);
#pragma unroll
    for (int u = 0; u < U; ++u) acc ^= r[u].x + r[u].y + r[u].z + r[u].w;
#pragma unroll
    for (int u = 0; u < U; ++u) g[u] = gn[u];
  }
  if (acc == 0x12345678) out[0] = acc;
}

template <int VEC, int U, int MODE>
void run(const uint4* tbl, const int* idx, long m, uint32_t* out, const char* name) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int warps : {8, 12, 16, 24, 32, 48, 64}) {
    const int bw = warps > 16 ? 16 : warps, nb = 148 * (warps / bw);
    k_gather<VEC, U, MODE><<<nb, bw * 32>>>(tbl, idx, m, out);
    CK(cudaDeviceSynchronize());
    cudaEventRecord(e0);
    for (int it = 0; it < 5; ++it) k_gather<VEC, U, MODE><<<nb, bw * 32>>>(tbl, idx, m, out);
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    ms /= 5;
    double bytes = (double)m * VEC * 16;
    printf("%-14s rowB=%3d U=%2d warps/SM=%2d : %7.2f TB/s (%.3f ms)\n", name, VEC * 16, U, warps, bytes / (ms * 1e-3) / 1e12, ms);
  }
}


// 32-byte loads: VEC32 = 32-B vectors per row
template <int VEC32, int U>
__global__ void k_gather256(const uint4* __restrict__ table, const int* __restrict__ idx, long m, uint32_t* out) {
  constexpr int G = 32 / VEC32;
  const int lane = threadIdx.x & 31, sub = lane / VEC32, v = lane % VEC32;
  const long warp = (blockIdx.x * (long)blockDim.x + threadIdx.x) >> 5;
  const long nwarps = (gridDim.x * (long)blockDim.x) >> 5;
  uint32_t acc = 0;
  long base = warp * G * U;
  int g[U];
#pragma unroll
  for (int u = 0; u < U; ++u) g[u] = base + u * G + sub < m ? __ldg(idx + ((base + u * G + sub) & ((1 << 22) - 1))) : 0;
  for (; base < m; base += nwarps * G * U) {
    const long nb = base + nwarps * G * U;
    int gn[U];
#pragma unroll
    for (int u = 0; u < U; ++u) gn[u] = nb + u * G + sub < m ? __ldg(idx + ((nb + u * G + sub) & ((1 << 22) - 1))) : 0;
    uint32_t r[U][8];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint4* p = table + (long)g[u] * VEC32 * 2 + v * 2;
      asm volatile("ld.global.nc.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                   : "=r"(r[u][0]), "=r"(r[u][1]), "=r"(r[u][2]), "=r"(r[u][3]), "=r"(r[u][4]), "=r"(r[u][5]), "=r"(r[u][6]), "=r"(r[u][7])
                   : "l"(p));
    }
#pragma unroll
    for (int u = 0; u < U; ++u) acc ^= r[u][0] + r[u][1] + r[u][2] + r[u][3] + r[u][4] + r[u][5] + r[u][6] + r[u][7];
#pragma unroll
    for (int u = 0; u < U; ++u) g[u] = gn[u];
  }
  if (acc == 0x12345678) out[0] = acc;
}

template <int VEC32, int U>
void run256(const uint4* tbl, const int* idx, long m, uint32_t* out) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int warps : {4, 8, 12, 16, 32}) {
    const int bw = warps > 16 ? 16 : warps, nb = 148 * (warps / bw);
    k_gather256<VEC32, U><<<nb, bw * 32>>>(tbl, idx, m, out);
    CK(cudaDeviceSynchronize());
    cudaEventRecord(e0);
    for (int it = 0; it < 5; ++it) k_gather256<VEC32, U><<<nb, bw * 32>>>(tbl, idx, m, out);
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    ms /= 5;
    double bytes = (double)m * VEC32 * 32;
    printf("ldg256 rowB=%3d U=%2d warps/SM=%2d : %7.2f TB/s (%.3f ms)\n", VEC32 * 32, U, warps, bytes / (ms * 1e-3) / 1e12, ms);
  }
}

int main(int argc, char** argv) {
  const long R = argc > 1 ? atol(argv[1]) : 232965;
  const long M = 115374529 / 4;  // rows gathered per launch (a quarter of C2's nnz)
  std::mt19937_64 rng(1);
  std::vector<int> h(M);
  for (long i = 0; i < (1 << 22); ++i) h[i] = (int)(rng() % R);
  printf("table rows %ld (%.1f MB)\n", R, R * 256 / 1e6);
  int* idx;
  uint4* tbl;
  uint32_t* out;
  CK(cudaMalloc(&idx, M * 4 + 4096));
  CK(cudaMalloc(&tbl, R * 256));
  CK(cudaMalloc(&out, 4));
  CK(cudaMemset(idx, 0, M * 4 + 4096));
  CK(cudaMemcpy(idx, h.data(), M * 4, cudaMemcpyHostToDevice));
  CK(cudaMemset(tbl, 1, R * 256));
  run<16, 8, 0>(tbl, idx, M, out, "ldg");
  run256<8, 4>(tbl, idx, M, out);
  run256<8, 8>(tbl, idx, M, out);
  run256<8, 16>(tbl, idx, M, out);
  run256<4, 8>(tbl, idx, M, out);
  run256<4, 16>(tbl, idx, M, out);
  return 0;
}
