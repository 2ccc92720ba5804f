// Dense GEMMs of the GCN layer (reference gnn.py:142-143, 188-189, 199-202), hand-written for
// sm_100a so no GCN pass calls cuBLAS:
//
//   hcs_grad_w : C[M x N] = A^T B, A = z_cache [K x M], B = grad_out [K x N], K = rows (233 K at C3)
//                -- the layer's weight gradient grad_W = Z^T G (gnn.py:188, 195-199).  Deterministic
//                split-K: CTA (s, mt, nt) multiplies its contiguous row slice into a 64 x 64 partial,
//                a second launch sums the partials of every output in slice order (no float atomics,
//                so the result is bitwise run-to-run stable, like the reference's ascending-window
//                accumulation).
//   hcs_gemm   : C[K x N] = A[K x M] B[M x N] -- the tall-skinny update (x_next = Z W, G W^T) of the
//                unfused mode and of layer shapes outside the fused epilogues' on-chip budget.
//
// Both stage 32-row K slabs with cp.async (2 stages) into padded shared tiles (conflict-free
// fragment loads) and multiply on mma.sync m16n8k8 tf32 (operands RNA-rounded to tf32, fp32
// accumulate).  They are HBM-bound at the C3 shapes: grad_W reads K * (M + N) * 4 bytes once.
#include <type_traits>

#include "common.cuh"
#include "mma_helpers.cuh"

namespace hcs {

constexpr int kDenseThreads = 128;  // 4 warps, 16 output rows each
constexpr int kKT = 32;             // K rows per stage (grad_W) / M columns per stage (gemm)
constexpr int kLdT = 72;            // padded row of a 64-wide tile (conflict-free b / a^T loads)
constexpr int kLdA = 36;            // padded row of a 32-wide A tile (gemm)

__device__ __forceinline__ uint32_t tf32_rna(float v) {
  uint32_t t;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(t) : "f"(v));
  return t;
}

// 16-byte chunk (row r, columns c..c+3) of a row-major fp32 matrix into shared memory; columns
// past `cols` and rows past `rows` are zero-filled (cp.async src-size < 16).
__device__ __forceinline__ void ld_chunk(uint32_t dst, const float* __restrict__ src, int64_t ld, int64_t r,
                                         int64_t rows, int c, int cols, uint64_t pol) {
  const int valid = (r < rows) ? max(0, min(4, cols - c)) : 0;
  const float* p = valid ? src + r * ld + c : src;
  cp_async16(dst, p, (uint32_t)(valid * 4), pol);
}

// The same 4 columns element by element (4-byte cp.async, zero-filled past the bounds) for
// operands whose rows are not 16-byte aligned (e.g. a 41-wide gradient).
__device__ __forceinline__ void ld_elems(uint32_t dst, const float* __restrict__ src, int64_t ld, int64_t r,
                                         int64_t rows, int c, int cols) {
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    const bool ok = r < rows && c + e < cols;
    const float* p = ok ? src + r * ld + c + e : src;
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;" ::"r"(dst + 4 * e), "l"(p), "r"(ok ? 4 : 0)
                 : "memory");
  }
}

template <bool V>
__device__ __forceinline__ void ld4(uint32_t dst, const float* __restrict__ src, int64_t ld, int64_t r, int64_t rows,
                                    int c, int cols, uint64_t pol) {
  if (V) ld_chunk(dst, src, ld, r, rows, c, cols, pol);
  else ld_elems(dst, src, ld, r, rows, c, cols);
}

// grad_W partials: grid (S, ceil(M/64), ceil(N/64)); CTA s covers rows [s*rps, (s+1)*rps).
template <bool VA, bool VB>
__global__ void __launch_bounds__(kDenseThreads) k_gradw_partial(const float* __restrict__ a, int64_t lda,
                                                                  const float* __restrict__ b, int64_t ldb, int64_t K,
                                                                  int M, int N, int64_t rps, float* __restrict__ part) {
  __shared__ __align__(16) float As[2][kKT][kLdT];
  __shared__ __align__(16) float Bs[2][kKT][kLdT];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int g = lane >> 2, t = lane & 3;
  const int s = blockIdx.x, m0 = blockIdx.y * 64, n0 = blockIdx.z * 64;
  const int64_t k_begin = (int64_t)s * rps, k_end = min(K, k_begin + rps);
  const uint64_t pol = policy_evict_first();
  float acc[8][4];
#pragma unroll
  for (int i = 0; i < 8; ++i) acc[i][0] = acc[i][1] = acc[i][2] = acc[i][3] = 0.f;
  auto load = [&](int stage, int64_t k0) {
#pragma unroll
    for (int q = 0; q < 4; ++q) {  // 32 rows x 16 chunks of A and of B: 4 + 4 per thread
      const int i = tid + q * kDenseThreads, r = i >> 4, c = (i & 15) * 4;
      ld4<VA>(smem_u32(&As[stage][r][c]), a, lda, k0 + r, k_end, m0 + c, M, pol);
      ld4<VB>(smem_u32(&Bs[stage][r][c]), b, ldb, k0 + r, k_end, n0 + c, N, pol);
    }
    cp_async_commit();
  };
  if (k_begin < k_end) load(0, k_begin);
  int stage = 0;
  for (int64_t k0 = k_begin; k0 < k_end; k0 += kKT) {
    if (k0 + kKT < k_end) {
      load(stage ^ 1, k0 + kKT);
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < kKT / 8; ++kk) {
      const int kr = kk * 8 + t, mr = warp * 16 + g;
      uint32_t af[4];
      af[0] = tf32_rna(As[stage][kr][mr]);
      af[1] = tf32_rna(As[stage][kr][mr + 8]);
      af[2] = tf32_rna(As[stage][kr + 4][mr]);
      af[3] = tf32_rna(As[stage][kr + 4][mr + 8]);
#pragma unroll
      for (int nt = 0; nt < 8; ++nt) {
        const uint32_t b0 = tf32_rna(Bs[stage][kr][nt * 8 + g]);
        const uint32_t b1 = tf32_rna(Bs[stage][kr + 4][nt * 8 + g]);
        mma_tf32_1688(acc[nt], af, b0, b1);
      }
    }
    __syncthreads();  // the next iteration's load overwrites this stage
    stage ^= 1;
  }
  float* p = part + ((((int64_t)s * gridDim.y + blockIdx.y) * gridDim.z + blockIdx.z) << 12);
#pragma unroll
  for (int nt = 0; nt < 8; ++nt) {
    const int r = warp * 16 + g, c = nt * 8 + 2 * t;
    *reinterpret_cast<float2*>(p + r * 64 + c) = make_float2(acc[nt][0], acc[nt][1]);
    *reinterpret_cast<float2*>(p + (r + 8) * 64 + c) = make_float2(acc[nt][2], acc[nt][3]);
  }
}

// C[m, n] = sum of the S partials: one warp per output, lane l sums s = l, l + 32, ... ascending,
// then a fixed shuffle tree (deterministic).  Replaces one thread per output summing all S in
// sequence (C3 grad_W2: 2,624 outputs x 296 partials, 20 -> ~5 us).
__global__ void k_gradw_reduce_warp(const float* __restrict__ part, int S, int mtiles, int ntiles, int M, int N,
                                    float* __restrict__ c, int64_t ldc) {
  const int lane = threadIdx.x & 31;
  const int64_t i = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (i >= (int64_t)M * N) return;
  const int m = (int)(i / N), n = (int)(i - (int64_t)m * N);
  const int mt = m >> 6, nt = n >> 6, off = ((m & 63) << 6) | (n & 63);
  const int64_t tile = (int64_t)mtiles * ntiles, base = (int64_t)mt * ntiles + nt;
  float v = 0.f;
  for (int s = lane; s < S; s += 32) v += __ldg(part + ((s * tile + base) << 12) + off);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  if (lane == 0) c[(int64_t)m * ldc + n] = v;
}

// C[m, n] = sum over s = 0..S-1 (ascending) of the partials.
__global__ void k_gradw_reduce(const float* __restrict__ part, int S, int mtiles, int ntiles, int M, int N,
                               float* __restrict__ c, int64_t ldc) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= M * N) return;
  const int m = i / N, n = i - m * N;
  const int mt = m >> 6, nt = n >> 6, off = ((m & 63) << 6) | (n & 63);
  const int64_t tile = (int64_t)mtiles * ntiles, base = (int64_t)mt * ntiles + nt;
  float v = 0.f;
  for (int s = 0; s < S; ++s) v += part[((s * tile + base) << 12) + off];
  c[(int64_t)m * ldc + n] = v;
}

// C = A B, A [K x M] (lda), B [M x N] (ldb), C [K x N] (ldc).  grid (ceil(K/64), ceil(n_store/64)).
// BF16OUT: C is bf16 (RNE), multiplied by 1[mask > 0] where mask != nullptr (the ReLU backward of
// the next aggregation's operand), and columns [N, n_store) are written as zeros (slice padding).
// MT = m16 tiles per warp (64 * MT rows per CTA): with MT = 2 each W (B) fragment loaded and
// rounded from shared memory feeds two MMAs -- the kernel is bound by those shared loads.
template <bool VA, bool VB, bool BF16OUT = false, int MT = 1>
__global__ void __launch_bounds__(kDenseThreads) k_gemm_tall(const float* __restrict__ a, int64_t lda,
                                                              const float* __restrict__ b, int64_t ldb, int64_t K,
                                                              int M, int N, void* __restrict__ cv, int64_t ldc,
                                                              const float* __restrict__ mask, int64_t ldm,
                                                              int n_store) {
  constexpr int ROWS = 64 * MT;
  extern __shared__ __align__(16) float gsm[];
  float (*As)[ROWS][kLdA] = reinterpret_cast<float (*)[ROWS][kLdA]>(gsm);
  float (*Bs)[kKT][kLdT] = reinterpret_cast<float (*)[kKT][kLdT]>(gsm + 2 * ROWS * kLdA);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int g = lane >> 2, t = lane & 3;
  const int64_t r0 = (int64_t)blockIdx.x * ROWS;
  const int n0 = blockIdx.y * 64;
  const uint64_t pol = policy_evict_first(), keep = policy_evict_last();
  float acc[MT][8][4];
#pragma unroll
  for (int m = 0; m < MT; ++m)
#pragma unroll
    for (int i = 0; i < 8; ++i) acc[m][i][0] = acc[m][i][1] = acc[m][i][2] = acc[m][i][3] = 0.f;
  auto load = [&](int stage, int k0) {
#pragma unroll
    for (int q = 0; q < 4 * MT; ++q) {
      const int i = tid + q * kDenseThreads;
      const int ar = i >> 3, ac = (i & 7) * 4;  // A: ROWS rows x 8 chunks
      ld4<VA>(smem_u32(&As[stage][ar][ac]), a, lda, r0 + ar, K, k0 + ac, M, pol);
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int i = tid + q * kDenseThreads;
      const int br = i >> 4, bc = (i & 15) * 4;  // B: 32 rows x 16 chunks (rows past M zero-filled)
      ld4<VB>(smem_u32(&Bs[stage][br][bc]), b, ldb, k0 + br, M, n0 + bc, N, keep);
    }
    cp_async_commit();
  };
  load(0, 0);
  int stage = 0;
  for (int k0 = 0; k0 < M; k0 += kKT) {
    if (k0 + kKT < M) {
      load(stage ^ 1, k0 + kKT);
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < kKT / 8; ++kk) {
      const int kc = kk * 8 + t;
      uint32_t af[MT][4];
#pragma unroll
      for (int m = 0; m < MT; ++m) {
        const int mr = warp * 16 * MT + m * 16 + g;
        af[m][0] = tf32_rna(As[stage][mr][kc]);
        af[m][1] = tf32_rna(As[stage][mr + 8][kc]);
        af[m][2] = tf32_rna(As[stage][mr][kc + 4]);
        af[m][3] = tf32_rna(As[stage][mr + 8][kc + 4]);
      }
#pragma unroll
      for (int nt = 0; nt < 8; ++nt) {
        const uint32_t b0 = tf32_rna(Bs[stage][kc][nt * 8 + g]);
        const uint32_t b1 = tf32_rna(Bs[stage][kc + 4][nt * 8 + g]);
#pragma unroll
        for (int m = 0; m < MT; ++m) mma_tf32_1688(acc[m][nt], af[m], b0, b1);
      }
    }
    __syncthreads();
    stage ^= 1;
  }
  if (BF16OUT) {
    __nv_bfloat16* c = static_cast<__nv_bfloat16*>(cv);
#pragma unroll
    for (int m = 0; m < MT; ++m)
#pragma unroll
    for (int nt = 0; nt < 8; ++nt) {
      const int col = n0 + nt * 8 + 2 * t;  // even; ldc even, n_store even
      if (col >= n_store) continue;
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int64_t r = r0 + warp * 16 * MT + m * 16 + g + 8 * h;
        if (r >= K) continue;
        float v0 = col < N ? acc[m][nt][2 * h] : 0.f, v1 = col + 1 < N ? acc[m][nt][2 * h + 1] : 0.f;
        if (mask != nullptr) {
          const float* mp = mask + r * ldm + col;
          if (col + 1 < N && ((ldm & 1) == 0) && (((uintptr_t)mask & 7) == 0)) {  // one 8-B load for the pair
            const float2 mk = __ldg(reinterpret_cast<const float2*>(mp));
            if (!(mk.x > 0.f)) v0 = 0.f;
            if (!(mk.y > 0.f)) v1 = 0.f;
          } else {
            if (col < N && !(__ldg(mp) > 0.f)) v0 = 0.f;
            if (col + 1 < N && !(__ldg(mp + 1) > 0.f)) v1 = 0.f;
          }
        }
        *reinterpret_cast<__nv_bfloat162*>(c + r * ldc + col) = __floats2bfloat162_rn(v0, v1);
      }
    }
    return;
  }
  float* c = static_cast<float*>(cv);
#pragma unroll
  for (int m = 0; m < MT; ++m)
#pragma unroll
  for (int nt = 0; nt < 8; ++nt) {
    const int col = n0 + nt * 8 + 2 * t;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int64_t r = r0 + warp * 16 * MT + m * 16 + g + 8 * h;
      if (r >= K) continue;
      float* cp = c + r * ldc + col;
      if (col + 1 < N && ((ldc & 1) == 0)) {
        *reinterpret_cast<float2*>(cp) = make_float2(acc[m][nt][2 * h], acc[m][nt][2 * h + 1]);
      } else {
        if (col < N) cp[0] = acc[m][nt][2 * h];
        if (col + 1 < N) cp[1] = acc[m][nt][2 * h + 1];
      }
    }
  }
}

#ifndef HCS_GEMM_MT
#define HCS_GEMM_MT 2  // m16 tiles per warp of the tall GEMMs (64 * MT rows per CTA)
#endif
// dynamic shared memory of k_gemm_tall<..., MT>: the A and B double buffers
inline int gemm_smem(int mt) { return (2 * 64 * mt * kLdA + 2 * kKT * kLdT) * (int)sizeof(float); }

// rows staged with 16-byte copies need a 16-byte aligned base and a row stride of 4 floats
static bool vec_ok(const float* p, int64_t ld) { return ((uintptr_t)p & 15) == 0 && ld % 4 == 0; }

static int64_t gradw_splits(int64_t K, int mtiles, int ntiles) {
  const int64_t tiles = (int64_t)mtiles * ntiles;
  int64_t s = std::max<int64_t>(1, (2 * (int64_t)num_sms() + tiles - 1) / tiles);  // ~2 CTAs per SM
  s = std::min<int64_t>(s, std::max<int64_t>(1, (K + kKT - 1) / kKT));
  return s;
}

}  // namespace hcs

using namespace hcs;

extern "C" int hcs_grad_w_workspace_bytes(int64_t K, int32_t M, int32_t N, size_t* bytes) {
  HCS_REQUIRE(bytes != nullptr && K >= 0 && M > 0 && N > 0, HCS_EINVAL, "bad grad_W shape");
  const int mt = (M + 63) / 64, nt = (N + 63) / 64;
  *bytes = (size_t)gradw_splits(K, mt, nt) * mt * nt * 4096 * sizeof(float);
  return HCS_OK;
}

extern "C" int hcs_grad_w(const float* a, int64_t lda, const float* b, int64_t ldb, int64_t K, int32_t M, int32_t N,
                          float* c, int64_t ldc, void* workspace, size_t ws_bytes, void* stream) {
  HCS_REQUIRE(K >= 0 && M > 0 && N > 0 && ldc >= N, HCS_EINVAL, "bad grad_W shape (K %lld, M %d, N %d, ldc %lld)",
              (long long)K, M, N, (long long)ldc);
  HCS_REQUIRE(lda >= M && ldb >= N, HCS_EINVAL, "grad_W operands need lda >= M, ldb >= N");
  HCS_REQUIRE(((uintptr_t)a & 3) == 0 && ((uintptr_t)b & 3) == 0, HCS_EINVAL, "grad_W operands must be fp32-aligned");
  const int mt = (M + 63) / 64, nt = (N + 63) / 64;
  const int64_t S = gradw_splits(K, mt, nt);
  HCS_REQUIRE(workspace != nullptr && ws_bytes >= (size_t)S * mt * nt * 4096 * sizeof(float), HCS_EINVAL,
              "grad_W workspace too small (hcs_grad_w_workspace_bytes)");
  cudaStream_t st = as_stream(stream);
  const int64_t rps = ((K + S - 1) / S + kKT - 1) / kKT * kKT;
  const bool va = vec_ok(a, lda), vb = vec_ok(b, ldb);
  auto kern = va ? (vb ? k_gradw_partial<true, true> : k_gradw_partial<true, false>)
                 : (vb ? k_gradw_partial<false, true> : k_gradw_partial<false, false>);
  kern<<<dim3((unsigned)S, mt, nt), kDenseThreads, 0, st>>>(a, lda, b, ldb, K, M, N, rps, (float*)workspace);
  HCS_LAUNCH_CHECK("k_gradw_partial");
  if (S >= 64) {
    k_gradw_reduce_warp<<<(unsigned)(((int64_t)M * N + 7) / 8), 256, 0, st>>>((const float*)workspace, (int)S, mt, nt,
                                                                          M, N, c, ldc);
    HCS_LAUNCH_CHECK("k_gradw_reduce_warp");
  } else {
    k_gradw_reduce<<<(M * N + 255) / 256, 256, 0, st>>>((const float*)workspace, (int)S, mt, nt, M, N, c, ldc);
    HCS_LAUNCH_CHECK("k_gradw_reduce");
  }
  return HCS_OK;
}

extern "C" int hcs_gemm(const float* a, int64_t lda, const float* b, int64_t ldb, int64_t K, int32_t M, int32_t N,
                        float* c, int64_t ldc, void* stream) {
  HCS_REQUIRE(K >= 0 && M > 0 && N > 0 && ldc >= N, HCS_EINVAL, "bad GEMM shape (K %lld, M %d, N %d, ldc %lld)",
              (long long)K, M, N, (long long)ldc);
  HCS_REQUIRE(lda >= M && ldb >= N, HCS_EINVAL, "GEMM operands need lda >= M, ldb >= N");
  HCS_REQUIRE(((uintptr_t)a & 3) == 0 && ((uintptr_t)b & 3) == 0, HCS_EINVAL, "GEMM operands must be fp32-aligned");
  if (K == 0) return HCS_OK;
  constexpr int MT = HCS_GEMM_MT;
  const int64_t bx = (K + 64 * MT - 1) / (64 * MT);
  HCS_REQUIRE(bx < (1ll << 31), HCS_EINVAL, "too many rows");
  const bool va = vec_ok(a, lda), vb = vec_ok(b, ldb);
  auto kern = va ? (vb ? k_gemm_tall<true, true, false, MT> : k_gemm_tall<true, false, false, MT>)
                 : (vb ? k_gemm_tall<false, true, false, MT> : k_gemm_tall<false, false, false, MT>);
  HCS_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, gemm_smem(MT)));
  kern<<<dim3((unsigned)bx, (N + 63) / 64), kDenseThreads, gemm_smem(MT), as_stream(stream)>>>(a, lda, b, ldb, K, M, N, c, ldc,
                                                                                  nullptr, 0, N);
  HCS_LAUNCH_CHECK("k_gemm_tall");
  return HCS_OK;
}

// hcs_gemm with a bf16 destination: C[K x n_store] = bf16((A B) * 1[mask > 0]) for columns < N,
// zeros for columns [N, n_store) -- the next aggregation's operand, staged (padded to whole gather
// slices) by the GEMM itself instead of a conversion pass.
extern "C" int hcs_gemm_bf16(const float* a, int64_t lda, const float* b, int64_t ldb, int64_t K, int32_t M,
                             int32_t N, void* c, int64_t ldc, int32_t n_store, const float* mask, int64_t ld_mask,
                             void* stream) {
  HCS_REQUIRE(K >= 0 && M > 0 && N > 0 && n_store >= N && ldc >= n_store, HCS_EINVAL,
              "bad GEMM shape (K %lld, M %d, N %d, n_store %d, ldc %lld)", (long long)K, M, N, n_store, (long long)ldc);
  HCS_REQUIRE(n_store % 2 == 0 && ldc % 2 == 0 && ((uintptr_t)c & 3) == 0, HCS_EINVAL,
              "bf16 GEMM output needs an even n_store and ldc and a 4-byte aligned base");
  HCS_REQUIRE(lda >= M && ldb >= N, HCS_EINVAL, "GEMM operands need lda >= M, ldb >= N");
  HCS_REQUIRE(mask == nullptr || ld_mask >= N, HCS_EINVAL, "mask needs ld_mask >= N");
  HCS_REQUIRE(((uintptr_t)a & 3) == 0 && ((uintptr_t)b & 3) == 0, HCS_EINVAL, "GEMM operands must be fp32-aligned");
  if (K == 0) return HCS_OK;
  // MT = 2 (two m16 tiles per warp) for the plain GEMMs; the masked one keeps MT = 1 (its epilogue's
  // mask loads, twice as many per thread at MT = 2, made it slower: 49.6 -> 60.7 us, tools/exp_gemm.py)
  const bool va = vec_ok(a, lda), vb = vec_ok(b, ldb);
  auto launch = [&](auto mt_tag) -> int {
    constexpr int MT = decltype(mt_tag)::value;
    const int64_t bx = (K + 64 * MT - 1) / (64 * MT);
    HCS_REQUIRE(bx < (1ll << 31), HCS_EINVAL, "too many rows");
    auto kern = va ? (vb ? k_gemm_tall<true, true, true, MT> : k_gemm_tall<true, false, true, MT>)
                   : (vb ? k_gemm_tall<false, true, true, MT> : k_gemm_tall<false, false, true, MT>);
    HCS_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, gemm_smem(MT)));
    kern<<<dim3((unsigned)bx, (n_store + 63) / 64), kDenseThreads, gemm_smem(MT), as_stream(stream)>>>(
        a, lda, b, ldb, K, M, N, c, ldc, mask, ld_mask, n_store);
    return HCS_OK;
  };
  const int rc = mask != nullptr ? launch(std::integral_constant<int, 1>{})
                                 : launch(std::integral_constant<int, HCS_GEMM_MT>{});
  if (rc != HCS_OK) return rc;
  HCS_LAUNCH_CHECK("k_gemm_tall");
  return HCS_OK;
}
