// K3: CUDA-core SpMM path (executors.py:100-108 scalar_window, 191-213 spmm_scalar).
//
// One warp per output row.  Each lane loads 16 bytes of an X row per entry
// (8 bf16 or 4 fp32 features), so a row of X is covered by VEC = dim*s/16 lanes
// and the warp works on G = 32/VEC entries at once.  Partial sums of the G lane
// groups are combined by a fixed shuffle tree, so the result is deterministic.
// CSR indices/values stream with L2::evict_first; X rows are gathered with
// L2::evict_last so the feature table stays resident in L2.
#include "common.cuh"

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

}  // namespace hcs

using namespace hcs;

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
