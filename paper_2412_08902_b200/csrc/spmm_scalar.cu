// K3: CUDA-core SpMM path (executors.py:100-108 scalar_window, 191-213 spmm_scalar).
//
// One warp per output row.  Each lane loads 16 bytes of an X row per entry
// (8 bf16 or 4 fp32 features), so a row of X is covered by VEC = dim*s/16 lanes
// and the warp works on G = 32/VEC entries at once.  Partial sums of the G lane
// groups are combined by a fixed shuffle tree, so the result is deterministic.
// CSR indices/values stream with L2::evict_first; X rows are gathered with
// L2::evict_last so the feature table stays resident in L2.
#include "common.cuh"
#include "mma_helpers.cuh"

#include <algorithm>

namespace hcs {

template <typename XT>
struct XVec;  // 16-byte vector of X elements -> 8 or 4 floats
template <>
struct XVec<__nv_bfloat16> {
  static constexpr int kElems = 8;
  __device__ __forceinline__ static void fma(float (&acc)[8], int4 v, float a) {
    const uint32_t w[4] = {(uint32_t)v.x, (uint32_t)v.y, (uint32_t)v.z, (uint32_t)v.w};
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      acc[2 * i] = fmaf(a, bf16lo(w[i]), acc[2 * i]);
      acc[2 * i + 1] = fmaf(a, bf16hi(w[i]), acc[2 * i + 1]);
    }
  }
};
template <>
struct XVec<float> {
  static constexpr int kElems = 4;
  __device__ __forceinline__ static void fma(float (&acc)[8], int4 v, float a) {
    acc[0] = fmaf(a, __int_as_float(v.x), acc[0]);
    acc[1] = fmaf(a, __int_as_float(v.y), acc[1]);
    acc[2] = fmaf(a, __int_as_float(v.z), acc[2]);
    acc[3] = fmaf(a, __int_as_float(v.w), acc[3]);
  }
};

template <typename VT>
__device__ __forceinline__ float load_val(const VT* p, uint64_t pol);
template <>
__device__ __forceinline__ float load_val<float>(const float* p, uint64_t pol) { return ld_stream_f32(p, pol); }
template <>
__device__ __forceinline__ float load_val<__nv_bfloat16>(const __nv_bfloat16* p, uint64_t pol) {
  return __uint_as_float(ld_stream_u16(p, pol) << 16);
}

constexpr int kFusedMaxDim = 128;  // fused GCN epilogue: d_in, d_out <= 128
constexpr int kFusedMaxRows = 16;

// grid: one block per listed window; 8 warps walk the window's rows.
// FUSED (K6/K7 on CUDA cores): the window's rows are also kept in shared memory and
// multiplied by M (fp32 [dim x d_out], W or W^T) before out[rows] is written; fp32 FMA.
template <typename XT, typename VT, bool FUSED>
__global__ void __launch_bounds__(256) k_spmm_scalar(const int64_t* __restrict__ row_ptr, const int32_t* __restrict__ col,
                                                     const VT* __restrict__ val, int64_t n_rows, int wh,
                                                     const int32_t* __restrict__ win_list, const XT* __restrict__ x,
                                                     int dim, int64_t ldx, float* __restrict__ z, int64_t ldz,
                                                     const float* __restrict__ mw, int d_out, float* __restrict__ out,
                                                     int64_t ldo) {
  __shared__ float zs[FUSED ? kFusedMaxRows : 1][FUSED ? kFusedMaxDim + 4 : 1];
  constexpr int E = XVec<XT>::kElems;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint64_t keep = policy_evict_last();
  const uint64_t strm = stream_policy();
  const int64_t w = win_list[blockIdx.x];
  const int64_t rs = w * wh, re = min(rs + wh, n_rows);
  const int nvec_total = (dim + E - 1) / E;  // 16B vectors per X row
  for (int fs = 0; fs < nvec_total; fs += 32) {  // feature slices of <= 32 vectors
    const int VEC = min(32, nvec_total - fs);
    const int G = 32 / VEC;
    const int g = lane / VEC, v = lane % VEC;
    const bool active = g < G;
    for (int64_t r = rs + warp; r < re; r += 8) {
      const int64_t e0 = row_ptr[r], e1 = row_ptr[r + 1];
      float acc[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) acc[i] = 0.f;
      if (active) {
        const XT* xb = x + (int64_t)(fs + v) * E;
        int64_t k = e0 + g;
        // 4 entries per group in flight
        for (; k + 3 * G < e1; k += 4 * G) {
          int c0 = ld_stream_s32(col + k, strm), c1 = ld_stream_s32(col + k + G, strm);
          int c2 = ld_stream_s32(col + k + 2 * G, strm), c3 = ld_stream_s32(col + k + 3 * G, strm);
          float a0 = load_val(val + k, strm), a1 = load_val(val + k + G, strm), a2 = load_val(val + k + 2 * G, strm),
                a3 = load_val(val + k + 3 * G, strm);
          int4 x0 = ld_keep_v4(xb + (int64_t)c0 * ldx, keep);
          int4 x1 = ld_keep_v4(xb + (int64_t)c1 * ldx, keep);
          int4 x2 = ld_keep_v4(xb + (int64_t)c2 * ldx, keep);
          int4 x3 = ld_keep_v4(xb + (int64_t)c3 * ldx, keep);
          XVec<XT>::fma(acc, x0, a0);
          XVec<XT>::fma(acc, x1, a1);
          XVec<XT>::fma(acc, x2, a2);
          XVec<XT>::fma(acc, x3, a3);
        }
        for (; k < e1; k += G) {
          int c0 = ld_stream_s32(col + k, strm);
          float a0 = load_val(val + k, strm);
          int4 x0 = ld_keep_v4(xb + (int64_t)c0 * ldx, keep);
          XVec<XT>::fma(acc, x0, a0);
        }
      }
      // fixed-order tree over the G lane groups
      for (int s = 1; s < G; s <<= 1) {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          float o = __shfl_down_sync(0xffffffffu, acc[i], s * VEC);
          if ((g % (2 * s)) == 0 && g + s < G) acc[i] += o;
        }
      }
      if (FUSED && g == 0) {
        const int f0 = (fs + v) * E;
#pragma unroll
        for (int i = 0; i < E; ++i)
          if (f0 + i < dim) zs[r - rs][f0 + i] = acc[i];
      }
      if (g == 0 && z != nullptr) {
        float* zr = z + r * ldz + (int64_t)(fs + v) * E;
        const int f0 = (fs + v) * E;
        if (f0 + E <= dim) {
          if (E == 8) {
            reinterpret_cast<float4*>(zr)[0] = make_float4(acc[0], acc[1], acc[2], acc[3]);
            reinterpret_cast<float4*>(zr)[1] = make_float4(acc[4], acc[5], acc[6], acc[7]);
          } else {
            reinterpret_cast<float4*>(zr)[0] = make_float4(acc[0], acc[1], acc[2], acc[3]);
          }
        } else {
          for (int i = 0; i < E && f0 + i < dim; ++i) zr[i] = acc[i];
        }
      }
    }
  }
  if (FUSED) {
    __syncthreads();
    const int nr = (int)(re - rs);
    for (int i = threadIdx.x; i < nr * d_out; i += blockDim.x) {
      const int r = i / d_out, j = i - r * d_out;
      float a = 0.f;
      for (int k = 0; k < dim; ++k) a = fmaf(zs[r][k], __ldg(mw + (int64_t)k * d_out + j), a);
      out[(rs + r) * ldo + j] = a;
    }
  }
}

// ---------------------------------------------------------------- warp-per-window kernel
// K3 as launched for SpMM and the fused GCN layer (the block-per-window kernel above is kept
// as a selectable variant).  Measured on C5 (R-MAT scale 24: 910 K scalar windows, 7.3 nnz
// per row; profiles/r01_scalar_c5.txt) the block kernel is latency-bound: every row is a
// chain row_ptr -> col/val -> X gather, 1.6 TB/s of DRAM.  Here one warp owns a window:
//   1. lanes 0..nr load the window's row pointers in one coalesced load (rows are read back
//      with shuffles); windows of <= kScalarCap entries stage all (col, value) pairs in
//      shared memory with one batch of coalesced loads -- one latency for the whole window;
//   2. a row of X is covered by L lanes of VB-byte vectors (VB = 32: 256-bit LDG, 16 bf16
//      per lane, so a 128-feature row is 8 lanes, and the warp's G = 32 / L lane groups work
//      on G different rows at once: each row is summed by one group in CSR order, U gathers
//      in flight per group, no cross-lane reduction);
//   3. windows with more entries (long rows) are walked row by row with the whole warp: the
//      G groups take entries k = g (mod G) and are combined by a fixed shuffle tree.
// Both orders are fixed, so results are run-to-run deterministic, and the fused GCN
// epilogue (FUSED) aggregates with exactly the same code as the plain SpMM.
constexpr int kScalarCap = 512;
constexpr int kScalarWarps = 8;
constexpr int kScalarZsLd = kFusedMaxDim + 4;  // fused: per-warp window rows in shared memory
#ifndef HCS_SCALAR_U32
#define HCS_SCALAR_U32 3  // entries in flight per lane group (32-byte vectors)
#endif
#ifndef HCS_SCALAR_U16
#define HCS_SCALAR_U16 6  // entries in flight per lane group (16-byte vectors; C5 sweep: 4/5/6/7/8 -> 7.47/6.51/6.17/6.41/6.96 ms)
#endif
#ifndef HCS_SCALAR_MINB
#define HCS_SCALAR_MINB 3  // resident blocks per SM the register budget is sized for
#endif

#define HCS_TRY(call)                  \
  do {                                 \
    const int _rc = (call);            \
    if (_rc != HCS_OK) return _rc;     \
  } while (0)

__device__ __forceinline__ int64_t ld_stream_s64(const int64_t* p, uint64_t pol) {
  int64_t r;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.s64 %0, [%1], %2;" : "=l"(r) : "l"(p), "l"(pol));
  return r;
}

template <int VB>
struct XRaw;
template <>
struct XRaw<16> {
  uint32_t w[4];
  __device__ __forceinline__ void load(const void* p, uint64_t pol) {
    asm volatile("ld.global.nc.L2::cache_hint.v4.b32 {%0,%1,%2,%3}, [%4], %5;"
                 : "=r"(w[0]), "=r"(w[1]), "=r"(w[2]), "=r"(w[3])
                 : "l"(p), "l"(pol));
  }
  __device__ __forceinline__ void zero() { w[0] = w[1] = w[2] = w[3] = 0u; }
};
template <>
struct XRaw<32> {
  uint32_t w[8];
  __device__ __forceinline__ void load(const void* p, uint64_t pol) {
    asm volatile("ld.global.nc.L2::cache_hint.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8], %9;"
                 : "=r"(w[0]), "=r"(w[1]), "=r"(w[2]), "=r"(w[3]), "=r"(w[4]), "=r"(w[5]), "=r"(w[6]), "=r"(w[7])
                 : "l"(p), "l"(pol));
  }
  __device__ __forceinline__ void zero() {
#pragma unroll
    for (int i = 0; i < 8; ++i) w[i] = 0u;
  }
};

template <typename XT, int VB>
__device__ __forceinline__ void fma_raw(float* acc, const uint32_t* w, float a) {
  if (sizeof(XT) == 2) {
#pragma unroll
    for (int i = 0; i < VB / 4; ++i) {
      acc[2 * i] = fmaf(a, bf16lo(w[i]), acc[2 * i]);
      acc[2 * i + 1] = fmaf(a, bf16hi(w[i]), acc[2 * i + 1]);
    }
  } else {
#pragma unroll
    for (int i = 0; i < VB / 4; ++i) acc[i] = fmaf(a, __uint_as_float(w[i]), acc[i]);
  }
}

template <typename XT, typename VT, int VB, int U, bool FUSED>
__global__ void __launch_bounds__(kScalarWarps * 32, FUSED ? 1 : HCS_SCALAR_MINB)
    k_spmm_scalar_w(const int64_t* __restrict__ row_ptr, const int32_t* __restrict__ col, const VT* __restrict__ val,
                    int64_t n_rows, int wh, const int32_t* __restrict__ win_list, int64_t n_list,
                    const XT* __restrict__ x, int dim, int64_t ldx, float* __restrict__ z, int64_t ldz,
                    const float* __restrict__ mw, int d_out, float* __restrict__ out, int64_t ldo) {
  constexpr int E = VB / (int)sizeof(XT);  // features per lane vector
  extern __shared__ __align__(16) uint8_t wsm[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int32_t* scol = reinterpret_cast<int32_t*>(wsm) + warp * kScalarCap;
  float* sval = reinterpret_cast<float*>(wsm + kScalarWarps * kScalarCap * 4) + warp * kScalarCap;
  float* zs = reinterpret_cast<float*>(wsm + kScalarWarps * kScalarCap * 8) + warp * (kFusedMaxRows * kScalarZsLd);
  const int64_t nwarps = (int64_t)gridDim.x * kScalarWarps;
  const int64_t gw0 = (int64_t)blockIdx.x * kScalarWarps + warp;
  if (gw0 >= n_list) return;
  const uint64_t keep = policy_evict_last();
  const uint64_t strm = stream_policy();
  // persistent warps, windows dealt round-robin (a block's warps never idle on a slow
  // sibling's window); the next window's row pointers are loaded one window ahead
  auto load_rp = [&](int64_t wi, int64_t& rs_, int& nr_) -> int64_t {
    if (wi >= n_list) {
      rs_ = 0;
      nr_ = 0;
      return 0;
    }
    rs_ = (int64_t)__ldg(win_list + wi) * wh;
    nr_ = (int)(n_rows - rs_ < wh ? n_rows - rs_ : wh);
    return lane <= nr_ ? ld_stream_s64(row_ptr + rs_ + lane, strm) : 0;
  };
  int64_t rs_n;
  int nr_n;
  int64_t rp_n = load_rp(gw0, rs_n, nr_n);
  for (int64_t gw = gw0; gw < n_list; gw += nwarps) {
  const int64_t rs = rs_n;
  const int nr = nr_n;
  const int64_t rp = rp_n;
  rp_n = load_rp(gw + nwarps, rs_n, nr_n);
  const int64_t e0 = __shfl_sync(0xffffffffu, rp, 0), e1 = __shfl_sync(0xffffffffu, rp, nr);
  const bool staged = e1 - e0 <= kScalarCap;
  const int32_t* cw = col + e0;  // the window's entries
  const VT* vw = val + e0;
  if (staged) {
    const int n = (int)(e1 - e0);
#pragma unroll
    for (int q = 0; q < kScalarCap / 32; ++q) {
      const int i = lane + 32 * q;
      if (i < n) {
        scol[i] = ld_stream_s32(cw + i, strm);
        sval[i] = load_val(vw + i, strm);
      }
    }
    __syncwarp();
  }
  const int nvec_total = (dim + E - 1) / E;
  const int64_t ldxb = ldx * (int64_t)sizeof(XT);
  auto store_row = [&](int r, int f0, const float (&acc)[E]) {
    if (z != nullptr) {
      float* zr = z + (rs + r) * ldz + f0;
      if (f0 + E <= dim) {
#pragma unroll
        for (int i = 0; i < E; i += 4)
          reinterpret_cast<float4*>(zr)[i / 4] = make_float4(acc[i], acc[i + 1], acc[i + 2], acc[i + 3]);
      } else {
#pragma unroll
        for (int i = 0; i < E; ++i)
          if (f0 + i < dim) zr[i] = acc[i];
      }
    }
    if (FUSED) {
#pragma unroll
      for (int i = 0; i < E; ++i)
        if (f0 + i < dim) zs[r * kScalarZsLd + f0 + i] = acc[i];
    }
  };
  for (int fs = 0; fs < nvec_total; fs += 32) {
    const int L = min(32, nvec_total - fs);
    const int G = 32 / L;
    const int g = lane / L, v = lane - g * L;
    const int f0 = (fs + v) * E;
    const char* xb = reinterpret_cast<const char*>(x + f0);
    if (staged) {
      for (int r0 = 0; r0 < nr; r0 += G) {
        const int r = r0 + g;
        // entry offsets relative to e0 (a window holds < 2^31 entries)
        const int kb = (int)(__shfl_sync(0xffffffffu, rp, min(r, 31)) - e0);
        const int ke = (int)(__shfl_sync(0xffffffffu, rp, min(r + 1, 31)) - e0);
        if (g < G && r < nr) {
          float acc[E];
#pragma unroll
          for (int i = 0; i < E; ++i) acc[i] = 0.f;
          for (int k = kb; k < ke; k += U) {
            XRaw<VB> xv[U];
            float a[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
              const int kk = k + u;
              a[u] = 0.f;
              xv[u].zero();
              if (kk < ke) {
                a[u] = sval[kk];
                xv[u].load(xb + (int64_t)scol[kk] * ldxb, keep);
              }
            }
#pragma unroll
            for (int u = 0; u < U; ++u) fma_raw<XT, VB>(acc, xv[u].w, a[u]);
          }
          store_row(r, f0, acc);
        }
      }
    } else {
      for (int r = 0; r < nr; ++r) {
        const int kb = (int)(__shfl_sync(0xffffffffu, rp, r) - e0);
        const int ke = (int)(__shfl_sync(0xffffffffu, rp, r + 1) - e0);
        float acc[E];
#pragma unroll
        for (int i = 0; i < E; ++i) acc[i] = 0.f;
        if (g < G) {
          for (int k = kb + g; k < ke; k += U * G) {
            XRaw<VB> xv[U];
            float a[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
              const int kk = k + u * G;
              a[u] = 0.f;
              xv[u].zero();
              if (kk < ke) {
                a[u] = load_val(vw + kk, strm);
                xv[u].load(xb + (int64_t)ld_stream_s32(cw + kk, strm) * ldxb, keep);
              }
            }
#pragma unroll
            for (int u = 0; u < U; ++u) fma_raw<XT, VB>(acc, xv[u].w, a[u]);
          }
        }
        // fixed-order tree over the G lane groups
        for (int sft = 1; sft < G; sft <<= 1) {
#pragma unroll
          for (int i = 0; i < E; ++i) {
            const float o = __shfl_down_sync(0xffffffffu, acc[i], sft * L);
            if ((g % (2 * sft)) == 0 && g + sft < G) acc[i] += o;
          }
        }
        if (g == 0) store_row(r, f0, acc);
      }
    }
  }
  if (FUSED) {
    // out[rs + r, j] = sum_k zs[r][k] * M[k][j], k ascending (fp32 FMA)
    __syncwarp();
    for (int j = lane; j < d_out; j += 32) {
      for (int r = 0; r < nr; ++r) {
        float o = 0.f;
        for (int k = 0; k < dim; ++k) o = fmaf(zs[r * kScalarZsLd + k], __ldg(mw + (int64_t)k * d_out + j), o);
        out[(rs + r) * ldo + j] = o;
      }
    }
  }
  __syncwarp();  // staging / zs buffers are reused by the warp's next window
  }
}

// K3, small window lists (C1-sized graphs, where one product is a few microseconds and latency
// bound).  The warp-per-window kernel walks a window's rows in dependent rounds: 22.6 us for C1's
// 169 scalar windows at N = 128.  Here one warp per ROW: the row's (col, value) pairs are read 32
// at a time (one coalesced load per lane, the next batch prefetched), broadcast by shuffles, and
// the warp's G = 32/L lane groups gather the X rows of entries g, g+G, ... of the batch with all
// of a group's loads in flight; a fixed shuffle tree sums the groups (deterministic).  C1 scalar
// windows: 10.3 us (tools/exp_c1.py; a variant that also cut hub rows into pieces spread over the
// block's warps, summed in shared memory, was slower: 12.3 us -- the barrier and the extra
// prologue cost more than the hub row's serial batches).
template <typename XT, typename VT, int VB, int U>
__global__ void __launch_bounds__(256, 1) k_spmm_scalar_rows(const int64_t* __restrict__ row_ptr,
                                                          const int32_t* __restrict__ col, const VT* __restrict__ val,
                                                          int64_t n_rows, int wh, const int32_t* __restrict__ win_list,
                                                          int64_t n_list, const XT* __restrict__ x, int dim,
                                                          int64_t ldx, float* __restrict__ z, int64_t ldz) {
  constexpr int E = VB / (int)sizeof(XT);
  const int lane = threadIdx.x & 31;
  const int64_t gw = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5);
  const int64_t wi = gw / wh;
  if (wi >= n_list) return;
  const int64_t rs = (int64_t)__ldg(win_list + wi) * wh + (gw - wi * wh);
  if (rs >= n_rows) return;
  const uint64_t keep = policy_evict_last();
  const uint64_t strm = stream_policy();
  const int64_t kb = __ldg(row_ptr + rs), ke = __ldg(row_ptr + rs + 1);
  const int nvec_total = (dim + E - 1) / E;
  const int64_t ldxb = ldx * (int64_t)sizeof(XT);
  for (int fs = 0; fs < nvec_total; fs += 32) {
    const int L = min(32, nvec_total - fs);
    const int G = 32 / L;
    const int g = lane / L, v = lane - g * L;
    const int f0 = (fs + v) * E;
    const char* xb = reinterpret_cast<const char*>(x + f0);
    float acc[E];
#pragma unroll
    for (int i = 0; i < E; ++i) acc[i] = 0.f;
    int cn = 0;
    float an = 0.f;
    if (kb + lane < ke) {
      cn = ld_stream_s32(col + kb + lane, strm);
      an = load_val(val + kb + lane, strm);
    }
    for (int64_t k0 = kb; k0 < ke; k0 += 32) {
      const int nb = (int)(ke - k0 < 32 ? ke - k0 : 32);
      const int c = cn;
      const float a = an;
      if (k0 + 32 + lane < ke) {  // next batch's pairs under this batch's gathers
        cn = ld_stream_s32(col + k0 + 32 + lane, strm);
        an = load_val(val + k0 + 32 + lane, strm);
      }
      for (int j0 = 0; j0 < nb; j0 += G * U) {
        XRaw<VB> xv[U];
        float av[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int j = j0 + g + u * G;
          const int cj = __shfl_sync(0xffffffffu, c, j & 31);
          av[u] = __shfl_sync(0xffffffffu, a, j & 31);
          xv[u].zero();
          if (g < G && j < nb) {
            xv[u].load(xb + (int64_t)cj * ldxb, keep);
          } else {
            av[u] = 0.f;
          }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) fma_raw<XT, VB>(acc, xv[u].w, av[u]);
      }
    }
    for (int sft = 1; sft < G; sft <<= 1) {  // fixed-order tree over the G lane groups
#pragma unroll
      for (int i = 0; i < E; ++i) {
        const float o = __shfl_down_sync(0xffffffffu, acc[i], sft * L);
        if ((g % (2 * sft)) == 0 && g + sft < G) acc[i] += o;
      }
    }
    if (g == 0) {
      float* zr = z + rs * ldz + f0;
      if (f0 + E <= dim) {
#pragma unroll
        for (int i = 0; i < E; i += 4)
          reinterpret_cast<float4*>(zr)[i / 4] = make_float4(acc[i], acc[i + 1], acc[i + 2], acc[i + 3]);
      } else {
#pragma unroll
        for (int i = 0; i < E; ++i)
          if (f0 + i < dim) zr[i] = acc[i];
      }
    }
  }
}

// K3, small plans with hub rows: the rows kernel above leaves a hub row's 32-entry batches on one
// warp (C1: a degree-168 row is ~6 dependent gather rounds of the 10 us launch).  Here the plan
// cuts every row into pieces of <= 32 entries (HybridPlan.scalar_pieces) and one warp takes one
// piece: a row of one piece is stored directly; the pieces of a longer row write partials, add 1
// to the row's completion counter, and the last one to arrive sums the partials in piece order
// (deterministic), stores the row and resets the counter (the split_arrive scheme of K4).
template <typename XT, typename VT, int VB>
__global__ void __launch_bounds__(256, 1) k_spmm_scalar_pieces(const int32_t* __restrict__ col,
                                                            const VT* __restrict__ val,
                                                            const int32_t* __restrict__ p_row,
                                                            const int64_t* __restrict__ p_k,
                                                            const int32_t* __restrict__ p_first,
                                                            const int32_t* __restrict__ p_count, int64_t npieces,
                                                            const XT* __restrict__ x, int dim, int64_t ldx,
                                                            float* __restrict__ z, int64_t ldz,
                                                            float* __restrict__ slots, int64_t ld_slot,
                                                            unsigned* __restrict__ cnt) {
  constexpr int E = VB / (int)sizeof(XT);
  const int lane = threadIdx.x & 31;
  const int64_t pc = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5);
  if (pc >= npieces) return;
  const int64_t rs = __ldg(p_row + pc);
  const int64_t kb = __ldg(p_k + 2 * pc), ke = __ldg(p_k + 2 * pc + 1);
  const int first = __ldg(p_first + pc), count = __ldg(p_count + pc);
  const uint64_t keep = policy_evict_last();
  const uint64_t strm = stream_policy();
  int c = 0;
  float a = 0.f;
  const int nb = (int)(ke - kb);  // <= 32
  if (lane < nb) {
    c = ld_stream_s32(col + kb + lane, strm);
    a = load_val(val + kb + lane, strm);
  }
  const int nvec_total = (dim + E - 1) / E;
  const int64_t ldxb = ldx * (int64_t)sizeof(XT);
  for (int fs = 0; fs < nvec_total; fs += 32) {
    const int L = min(32, nvec_total - fs);
    const int G = 32 / L;
    const int g = lane / L, v = lane - g * L;
    const int f0 = (fs + v) * E;
    const char* xb = reinterpret_cast<const char*>(x + f0);
    float acc[E];
#pragma unroll
    for (int i = 0; i < E; ++i) acc[i] = 0.f;
    for (int j0 = 0; j0 < nb; j0 += G * 8) {
      XRaw<VB> xv[8];
      float av[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int j = j0 + g + u * G;
        const int cj = __shfl_sync(0xffffffffu, c, j & 31);
        av[u] = __shfl_sync(0xffffffffu, a, j & 31);
        xv[u].zero();
        if (g < G && j < nb) {
          xv[u].load(xb + (int64_t)cj * ldxb, keep);
        } else {
          av[u] = 0.f;
        }
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) fma_raw<XT, VB>(acc, xv[u].w, av[u]);
    }
    for (int sft = 1; sft < G; sft <<= 1) {
#pragma unroll
      for (int i = 0; i < E; ++i) {
        const float o = __shfl_down_sync(0xffffffffu, acc[i], sft * L);
        if ((g % (2 * sft)) == 0 && g + sft < G) acc[i] += o;
      }
    }
    if (g == 0) {
      float* dst = count == 1 ? z + rs * ldz + f0 : slots + pc * ld_slot + f0;
      if (f0 + E <= dim) {
#pragma unroll
        for (int i = 0; i < E; i += 4) {
          if (count == 1)
            reinterpret_cast<float4*>(dst)[i / 4] = make_float4(acc[i], acc[i + 1], acc[i + 2], acc[i + 3]);
          else
            __stcg(reinterpret_cast<float4*>(dst) + i / 4, make_float4(acc[i], acc[i + 1], acc[i + 2], acc[i + 3]));
        }
      } else {
#pragma unroll
        for (int i = 0; i < E; ++i)
          if (f0 + i < dim) {
            if (count == 1) dst[i] = acc[i]; else __stcg(dst + i, acc[i]);
          }
      }
    }
  }
  if (count == 1) return;
  // a row of several pieces: the last piece to finish sums the partials in piece order
  __syncwarp();
  int last = 0;
  if (lane == 0) {
    __threadfence();
    const unsigned old = atomicAdd(cnt + first, 1u);
    if (old + 1u == (unsigned)count) {
      last = 1;
      cnt[first] = 0u;
    }
  }
  last = __shfl_sync(0xffffffffu, last, 0);
  if (!last) return;
  __threadfence();
  for (int f = lane * 4; f < dim; f += 128) {
    float4 sum = __ldcg(reinterpret_cast<const float4*>(slots + (int64_t)first * ld_slot + f));
    for (int q = 1; q < count; ++q) {
      const float4 t = __ldcg(reinterpret_cast<const float4*>(slots + (int64_t)(first + q) * ld_slot + f));
      sum.x += t.x;
      sum.y += t.y;
      sum.z += t.z;
      sum.w += t.w;
    }
    float* zr = z + rs * ldz + f;
    if (f + 4 <= dim) {
      *reinterpret_cast<float4*>(zr) = sum;
    } else {
      const float sv[4] = {sum.x, sum.y, sum.z, sum.w};
      for (int i = 0; i < 4 && f + i < dim; ++i) zr[i] = sv[i];
    }
  }
}

template <typename XT, typename VT>
static int launch_scalar_rows(const int64_t* row_ptr, const int32_t* col, const VT* val, int64_t n_rows, int wh,
                              const int32_t* win_list, int64_t n_list, const XT* x, int dim, int64_t ldx, float* z,
                              int64_t ldz, bool v32, cudaStream_t st) {
  const unsigned grid = (unsigned)((n_list * wh + 7) / 8);
  if (v32)
    k_spmm_scalar_rows<XT, VT, 32, 8><<<grid, 256, 0, st>>>(row_ptr, col, val, n_rows, wh, win_list, n_list, x, dim,
                                                            ldx, z, ldz);
  else
    k_spmm_scalar_rows<XT, VT, 16, 8><<<grid, 256, 0, st>>>(row_ptr, col, val, n_rows, wh, win_list, n_list, x, dim,
                                                            ldx, z, ldz);
  return HCS_OK;
}

// window lists up to this length use the row kernel in auto mode (one warp per row; small graphs)
#ifndef HCS_SCALAR_ROWS_MAX
#define HCS_SCALAR_ROWS_MAX 1024
#endif

// 0 auto (rows kernel for short lists, else warp-per-window), 1 block-per-window kernel, 2 warp kernel with
// 16-B vectors, 3 rows kernel, 4 warp-per-window kernel
static int g_scalar_variant = 0;

template <bool FUSED, typename XT, typename VT>
static int launch_scalar_w(const int64_t* row_ptr, const int32_t* col, const VT* val, int64_t n_rows, int wh,
                           const int32_t* win_list, int64_t n_list, const XT* x, int dim, int64_t ldx, float* z,
                           int64_t ldz, bool v32, cudaStream_t st, const float* mw = nullptr, int d_out = 0,
                           float* out = nullptr, int64_t ldo = 0) {
  // resident blocks only (persistent warps): 4 per SM for the SpMM, 1 for the fused kernel
  const int64_t want = (n_list + kScalarWarps - 1) / kScalarWarps;
  const unsigned grid = (unsigned)std::min<int64_t>(want, (int64_t)num_sms() * (FUSED ? 1 : HCS_SCALAR_MINB));
  const int smem = kScalarWarps * (kScalarCap * 8 + (FUSED ? kFusedMaxRows * kScalarZsLd * 4 : 0));
  auto k = v32 ? k_spmm_scalar_w<XT, VT, 32, HCS_SCALAR_U32, FUSED> : k_spmm_scalar_w<XT, VT, 16, HCS_SCALAR_U16, FUSED>;
  HCS_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  k<<<grid, kScalarWarps * 32, smem, st>>>(row_ptr, col, val, n_rows, wh, win_list, n_list, x, dim, ldx, z, ldz, mw,
                                            d_out, out, ldo);
  return HCS_OK;
}

// 32-byte X vectors when every row slice is 32-byte aligned and padded
static bool scalar_v32(const void* x, int x_dtype, int64_t ldx, int dim) {
  const int xs = x_dtype == HCS_DTYPE_BF16 ? 2 : 4, e32 = 32 / xs;
  return (g_scalar_variant == 0 || g_scalar_variant >= 3) && ((uintptr_t)x & 31) == 0 && (ldx * xs) % 32 == 0 &&
         ldx >= ((dim + e32 - 1) / e32) * e32;
}

}  // namespace hcs

using namespace hcs;

// Scalar-path kernel choice (experiments): 0 auto, 1 block-per-window, 2 warp-per-window with 16-B vectors,
// 3 warp-per-row (the small-list kernel), 4 warp-per-window whatever the list length.
extern "C" int hcs_set_scalar_variant(int variant) {
  HCS_REQUIRE(variant >= 0 && variant <= 4, HCS_EINVAL, "scalar variant must be 0..4 (got %d)", variant);
  g_scalar_variant = variant;
  return HCS_OK;
}

extern "C" int hcs_spmm_scalar(const int64_t* row_ptr, const int32_t* col_idx, const void* values, int values_dtype,
                               int64_t n_rows, int32_t wh, const int32_t* win_list, int64_t n_list, const void* x,
                               int x_dtype, int64_t x_rows, int32_t dim, int64_t ldx, float* z, int64_t ldz,
                               void* stream) {
  HCS_REQUIRE(wh > 0, HCS_EINVAL, "window_height must be positive");
  HCS_REQUIRE(dim > 0, HCS_EINVAL, "dim must be positive");
  HCS_REQUIRE(n_list >= 0 && n_list < (1LL << 31), HCS_EINVAL, "bad window list length");
  const int E = (x_dtype == HCS_DTYPE_BF16) ? 8 : 4;
  HCS_REQUIRE(ldx % E == 0 && ldx >= ((dim + E - 1) / E) * E, HCS_EINVAL,
              "ldx must be a multiple of %d covering dim rounded up to 16 bytes", E);
  HCS_REQUIRE(ldz >= dim, HCS_EINVAL, "ldz < dim");
  HCS_REQUIRE((ldz % 4) == 0, HCS_EINVAL, "ldz must be a multiple of 4");
  HCS_REQUIRE(((uintptr_t)x & 15) == 0 && ((uintptr_t)z & 15) == 0, HCS_EINVAL, "x/z must be 16-byte aligned");
  if (n_list == 0) return HCS_OK;
  cudaStream_t st = as_stream(stream);
  if (g_scalar_variant == 3 || (g_scalar_variant == 0 && n_list <= HCS_SCALAR_ROWS_MAX)) {
    const bool v32 = scalar_v32(x, x_dtype, ldx, dim);
    if (x_dtype == HCS_DTYPE_BF16 && values_dtype == HCS_DTYPE_BF16)
      HCS_TRY(launch_scalar_rows(row_ptr, col_idx, (const __nv_bfloat16*)values, n_rows, wh, win_list, n_list,
                                 (const __nv_bfloat16*)x, dim, ldx, z, ldz, v32, st));
    else if (x_dtype == HCS_DTYPE_BF16 && values_dtype == HCS_DTYPE_F32)
      HCS_TRY(launch_scalar_rows(row_ptr, col_idx, (const float*)values, n_rows, wh, win_list, n_list,
                                 (const __nv_bfloat16*)x, dim, ldx, z, ldz, v32, st));
    else if (x_dtype == HCS_DTYPE_F32 && values_dtype == HCS_DTYPE_F32)
      HCS_TRY(launch_scalar_rows(row_ptr, col_idx, (const float*)values, n_rows, wh, win_list, n_list,
                                 (const float*)x, dim, ldx, z, ldz, v32, st));
    else
      return set_error(HCS_EINVAL, "unsupported dtype combination x=%d values=%d", x_dtype, values_dtype);
    HCS_LAUNCH_CHECK("k_spmm_scalar_rows");
    return HCS_OK;
  }
  if (g_scalar_variant != 1 && wh <= 31) {
    // bf16 X in auto mode: 16-B vectors (16 lanes per 256-B row, 2 rows at a time, 6 entries in
    // flight per lane group) beat 32-B vectors with 3 in flight on C5's 910 K scalar windows:
    // 6.87-6.99 -> 6.17-6.18 ms (tools/exp_c5.py; the 32-B variant stays as "warp", variant 4)
    const bool v32 = scalar_v32(x, x_dtype, ldx, dim) && !(g_scalar_variant == 0 && x_dtype == HCS_DTYPE_BF16);
    if (x_dtype == HCS_DTYPE_BF16 && values_dtype == HCS_DTYPE_BF16)
      HCS_TRY(launch_scalar_w<false>(row_ptr, col_idx, (const __nv_bfloat16*)values, n_rows, wh, win_list, n_list,
                                     (const __nv_bfloat16*)x, dim, ldx, z, ldz, v32, st));
    else if (x_dtype == HCS_DTYPE_BF16 && values_dtype == HCS_DTYPE_F32)
      HCS_TRY(launch_scalar_w<false>(row_ptr, col_idx, (const float*)values, n_rows, wh, win_list, n_list,
                                     (const __nv_bfloat16*)x, dim, ldx, z, ldz, v32, st));
    else if (x_dtype == HCS_DTYPE_F32 && values_dtype == HCS_DTYPE_F32)
      HCS_TRY(launch_scalar_w<false>(row_ptr, col_idx, (const float*)values, n_rows, wh, win_list, n_list,
                                     (const float*)x, dim, ldx, z, ldz, v32, st));
    else
      return set_error(HCS_EINVAL, "unsupported dtype combination x=%d values=%d", x_dtype, values_dtype);
    HCS_LAUNCH_CHECK("k_spmm_scalar_w");
    (void)x_rows;
    return HCS_OK;
  }
  dim3 grid((unsigned)n_list);
  if (x_dtype == HCS_DTYPE_BF16 && values_dtype == HCS_DTYPE_BF16)
    k_spmm_scalar<__nv_bfloat16, __nv_bfloat16, false><<<grid, 256, 0, st>>>(
        row_ptr, col_idx, (const __nv_bfloat16*)values, n_rows, wh, win_list, (const __nv_bfloat16*)x, dim, ldx, z, ldz,
        nullptr, 0, nullptr, 0);
  else if (x_dtype == HCS_DTYPE_BF16 && values_dtype == HCS_DTYPE_F32)
    k_spmm_scalar<__nv_bfloat16, float, false><<<grid, 256, 0, st>>>(
        row_ptr, col_idx, (const float*)values, n_rows, wh, win_list, (const __nv_bfloat16*)x, dim, ldx, z, ldz, nullptr,
        0, nullptr, 0);
  else if (x_dtype == HCS_DTYPE_F32 && values_dtype == HCS_DTYPE_F32)
    k_spmm_scalar<float, float, false><<<grid, 256, 0, st>>>(row_ptr, col_idx, (const float*)values, n_rows, wh,
                                                            win_list, (const float*)x, dim, ldx, z, ldz, nullptr, 0,
                                                            nullptr, 0);
  else
    return set_error(HCS_EINVAL, "unsupported dtype combination x=%d values=%d", x_dtype, values_dtype);
  HCS_LAUNCH_CHECK("k_spmm_scalar");
  (void)x_rows;
  return HCS_OK;
}

// K6/K7 on CUDA cores: scalar windows with the fused GCN epilogue (see k_spmm_scalar).
// z may be NULL (backward: no z_cache).  M: fp32 [dim x d_out] device matrix.
extern "C" int hcs_gcn_scalar(const int64_t* row_ptr, const int32_t* col_idx, const void* values, int values_dtype,
                              int64_t n_rows, int32_t wh, const int32_t* win_list, int64_t n_list, const void* x,
                              int x_dtype, int64_t x_rows, int32_t dim, int64_t ldx, float* z, int64_t ldz,
                              const float* m, int32_t d_out, float* out, int64_t ldo, void* stream) {
  HCS_REQUIRE(wh > 0 && wh <= kFusedMaxRows, HCS_EINVAL, "fused GCN path supports window heights 1..%d",
              kFusedMaxRows);
  HCS_REQUIRE(dim > 0 && dim <= kFusedMaxDim, HCS_EINVAL, "fused GCN path needs 1 <= d_in <= %d (got %d)",
              kFusedMaxDim, dim);
  HCS_REQUIRE(d_out > 0 && d_out <= kFusedMaxDim, HCS_EINVAL, "fused GCN path needs 1 <= d_out <= %d (got %d)",
              kFusedMaxDim, d_out);
  HCS_REQUIRE(n_list >= 0 && n_list < (1LL << 31), HCS_EINVAL, "bad window list length");
  HCS_REQUIRE(m != nullptr && out != nullptr && ldo >= d_out, HCS_EINVAL, "fused GCN: bad M / out arguments");
  const int E = (x_dtype == HCS_DTYPE_BF16) ? 8 : 4;
  HCS_REQUIRE(ldx % E == 0 && ldx >= ((dim + E - 1) / E) * E, HCS_EINVAL,
              "ldx must be a multiple of %d covering dim rounded up to 16 bytes", E);
  HCS_REQUIRE(z == nullptr || (ldz >= dim && (ldz % 4) == 0 && ((uintptr_t)z & 15) == 0), HCS_EINVAL,
              "bad z_cache layout");
  HCS_REQUIRE(((uintptr_t)x & 15) == 0, HCS_EINVAL, "x must be 16-byte aligned");
  if (n_list == 0) return HCS_OK;
  cudaStream_t st = as_stream(stream);
  if (g_scalar_variant != 1) {  // same aggregation kernel (and order) as hcs_spmm_scalar
    const bool v32 = scalar_v32(x, x_dtype, ldx, dim);
    if (x_dtype == HCS_DTYPE_BF16 && values_dtype == HCS_DTYPE_BF16)
      HCS_TRY(launch_scalar_w<true>(row_ptr, col_idx, (const __nv_bfloat16*)values, n_rows, wh, win_list, n_list,
                                    (const __nv_bfloat16*)x, dim, ldx, z, ldz, v32, st, m, d_out, out, ldo));
    else if (x_dtype == HCS_DTYPE_F32 && values_dtype == HCS_DTYPE_F32)
      HCS_TRY(launch_scalar_w<true>(row_ptr, col_idx, (const float*)values, n_rows, wh, win_list, n_list,
                                    (const float*)x, dim, ldx, z, ldz, v32, st, m, d_out, out, ldo));
    else
      return set_error(HCS_EINVAL, "unsupported dtype combination x=%d values=%d", x_dtype, values_dtype);
    HCS_LAUNCH_CHECK("k_spmm_scalar_w<fused>");
    (void)x_rows;
    return HCS_OK;
  }
  dim3 grid((unsigned)n_list);
  if (x_dtype == HCS_DTYPE_BF16 && values_dtype == HCS_DTYPE_BF16)
    k_spmm_scalar<__nv_bfloat16, __nv_bfloat16, true><<<grid, 256, 0, st>>>(
        row_ptr, col_idx, (const __nv_bfloat16*)values, n_rows, wh, win_list, (const __nv_bfloat16*)x, dim, ldx, z, ldz,
        m, d_out, out, ldo);
  else if (x_dtype == HCS_DTYPE_F32 && values_dtype == HCS_DTYPE_F32)
    k_spmm_scalar<float, float, true><<<grid, 256, 0, st>>>(row_ptr, col_idx, (const float*)values, n_rows, wh,
                                                           win_list, (const float*)x, dim, ldx, z, ldz, m, d_out, out,
                                                           ldo);
  else
    return set_error(HCS_EINVAL, "unsupported dtype combination x=%d values=%d", x_dtype, values_dtype);
  HCS_LAUNCH_CHECK("k_spmm_scalar<fused>");
  (void)x_rows;
  return HCS_OK;
}

// K3 for small plans, hub rows split: one warp per piece of <= 32 entries of a row (see
// k_spmm_scalar_pieces).  Pieces of one row are consecutive: p_first[i] = the row's first piece,
// p_count[i] = its number of pieces; p_k = [k0, k1) entry ranges (2 int64 per piece).
// slots: npieces x ld_slot floats (ld_slot >= dim, multiple of 4, 16-B aligned); cnt: npieces
// uint32 completion counters, zero before the first launch (left zero).
#ifndef HCS_PIECES_BF16_V16_MAXDIM
// bf16 rows up to this width use 16-B lane vectors (4 lanes per 64-B row, a 3-step shuffle tree
// instead of 4 over twice the floats): C1 dim 32 piece launch 10.26 -> 8.23 us, bench 10.5 -> 10.3 us
#define HCS_PIECES_BF16_V16_MAXDIM 64
#endif
extern "C" int hcs_spmm_scalar_pieces(const int32_t* col_idx, const void* values, int values_dtype,
                                      const int32_t* p_row, const int64_t* p_k, const int32_t* p_first,
                                      const int32_t* p_count, int64_t npieces, const void* x, int x_dtype,
                                      int32_t dim, int64_t ldx, float* z, int64_t ldz, float* slots, int64_t ld_slot,
                                      unsigned* cnt, void* stream) {
  HCS_REQUIRE(dim > 0 && npieces >= 0, HCS_EINVAL, "dim must be positive");
  HCS_REQUIRE(ld_slot >= dim && ld_slot % 4 == 0 && ((uintptr_t)slots & 15) == 0, HCS_EINVAL,
              "slots: ld_slot must cover dim, be a multiple of 4 and 16-byte aligned");
  HCS_REQUIRE(((uintptr_t)x & 15) == 0 && ((uintptr_t)z & 15) == 0 && ldz % 4 == 0 && ldz >= dim, HCS_EINVAL,
              "x/z must be 16-byte aligned, ldz a multiple of 4 covering dim");
  if (npieces == 0) return HCS_OK;
  cudaStream_t st = as_stream(stream);
  const unsigned grid = (unsigned)((npieces + 7) / 8);
  const bool v32 = ((uintptr_t)x & 31) == 0 && (ldx * (x_dtype == HCS_DTYPE_BF16 ? 2 : 4)) % 32 == 0 &&
                   ldx >= ((dim + (x_dtype == HCS_DTYPE_BF16 ? 15 : 7)) / (x_dtype == HCS_DTYPE_BF16 ? 16 : 8)) *
                              (x_dtype == HCS_DTYPE_BF16 ? 16 : 8) &&
                   !(x_dtype == HCS_DTYPE_BF16 && dim <= HCS_PIECES_BF16_V16_MAXDIM);
#define HCS_PIECES(XT, VT)                                                                                        \
  do {                                                                                                          \
    if (v32)                                                                                                    \
      k_spmm_scalar_pieces<XT, VT, 32><<<grid, 256, 0, st>>>(col_idx, (const VT*)values, p_row, p_k, p_first,  \
                                                             p_count, npieces, (const XT*)x, dim, ldx, z, ldz,  \
                                                             slots, ld_slot, cnt);                              \
    else                                                                                                        \
      k_spmm_scalar_pieces<XT, VT, 16><<<grid, 256, 0, st>>>(col_idx, (const VT*)values, p_row, p_k, p_first,  \
                                                             p_count, npieces, (const XT*)x, dim, ldx, z, ldz,  \
                                                             slots, ld_slot, cnt);                              \
  } while (0)
  if (x_dtype == HCS_DTYPE_BF16 && values_dtype == HCS_DTYPE_BF16)
    HCS_PIECES(__nv_bfloat16, __nv_bfloat16);
  else if (x_dtype == HCS_DTYPE_BF16 && values_dtype == HCS_DTYPE_F32)
    HCS_PIECES(__nv_bfloat16, float);
  else if (x_dtype == HCS_DTYPE_F32 && values_dtype == HCS_DTYPE_F32)
    HCS_PIECES(float, float);
  else
    return set_error(HCS_EINVAL, "unsupported dtype combination x=%d values=%d", x_dtype, values_dtype);
#undef HCS_PIECES
  HCS_LAUNCH_CHECK("k_spmm_scalar_pieces");
  return HCS_OK;
}
