// K2: pack the TILE windows of an assignment into the tensor-core kernel's
// chunked format (the on-GPU counterpart of executors.py:129-135, where each
// tile window's entries are scattered into a zero-padded condensed slab and
// the matching X rows are gathered).
//
// A chunk is 64 consecutive condensed columns of one window.  Per chunk we keep
//   gidx[64]     : original column (= X row) of each condensed column, -1 = pad
//   entries      : packed (bf16 value << 16 | swizzled slab byte offset of (r, c)),
//                  in (row, column) order
// Entries are in (chunk, row, column) order.  Default builder: k_tile_bucket, one CTA per
// TILE window doing a stable counting sort of the window's CSR-ordered entries by chunk
// (16 x chunks counters in shared memory, rows walked in order), so no global sort and no
// key arrays (C2: 44 ms -> see DESIGN.md).  hcs_set_tile_plan_builder(1) selects the
// original radix sort on (chunk, position); both produce identical plans.
#include <cub/cub.cuh>

#include "common.cuh"
#include "mma_helpers.cuh"

namespace hcs {

static size_t a256(size_t x) { return (x + 255) & ~(size_t)255; }

__global__ void k_tile_nnz(const int64_t* __restrict__ row_ptr, const int32_t* __restrict__ tile_list, int64_t T,
                           int64_t n_rows, int wh, int64_t* __restrict__ out) {
  int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= T) return;
  int64_t w = tile_list[t];
  int64_t rs = w * wh, re = min(rs + wh, n_rows);
  out[t + 1] = row_ptr[re] - row_ptr[rs];
}

__global__ void k_tile_gidx(const int32_t* __restrict__ tile_list, int64_t T, const int64_t* __restrict__ chunk_ptr,
                            const int64_t* __restrict__ win_col_ptr, const int32_t* __restrict__ nonzero_cols,
                            int32_t* __restrict__ gidx) {
  // one block per tile window
  for (int64_t t = blockIdx.x; t < T; t += gridDim.x) {
    int64_t w = tile_list[t];
    int64_t c0 = win_col_ptr[w], nc = win_col_ptr[w + 1] - c0;
    int64_t s0 = chunk_ptr[t] * 64, s1 = chunk_ptr[t + 1] * 64;
    for (int64_t i = threadIdx.x; i < s1 - s0; i += blockDim.x) gidx[s0 + i] = (i < nc) ? nonzero_cols[c0 + i] : -1;
  }
}

template <typename VT>
__global__ void k_tile_keys(const int64_t* __restrict__ row_ptr, const int32_t* __restrict__ cond,
                            const VT* __restrict__ vals, const int32_t* __restrict__ tile_list, int64_t T,
                            const int64_t* __restrict__ chunk_ptr, const int64_t* __restrict__ ent_off, int64_t n_rows,
                            int wh, uint64_t* __restrict__ keys, uint32_t* __restrict__ kv) {
  // one block per tile window, one warp per row
  int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nwarp = blockDim.x >> 5;
  for (int64_t t = blockIdx.x; t < T; t += gridDim.x) {
    int64_t w = tile_list[t];
    int64_t rs = w * wh, re = min(rs + wh, n_rows);
    int64_t base_e = row_ptr[rs];
    uint64_t cbase = (uint64_t)chunk_ptr[t];
    for (int64_t r = rs + warp; r < re; r += nwarp) {
      uint64_t lr = (uint64_t)(r - rs);
      for (int64_t e = row_ptr[r] + lane; e < row_ptr[r + 1]; e += 32) {
        uint64_t c = (uint64_t)cond[e];
        uint64_t key = ((cbase + (c >> 6)) << 10) | (lr << 6) | (c & 63);
        int64_t slot = ent_off[t] + (e - base_e);
        keys[slot] = key;
        kv[slot] = __float_as_uint((float)vals[e]);  // exact for bf16 inputs
      }
    }
  }
}

__global__ void k_tile_emit(const uint64_t* __restrict__ keys, const uint32_t* __restrict__ kv, int64_t n, int ent_dtype,
                            void* __restrict__ ent, int64_t* __restrict__ ent_ptr, int64_t nchunks) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (; i < n; i += stride) {
    uint64_t k = keys[i];
    // slab byte offset of (row r, column c) in the 16 x 64 K-major 128B-swizzled B tile
    const uint32_t rc = (uint32_t)(k & 1023);
    uint32_t pos = sw128_kmajor_off16(rc >> 6, rc & 63u);
    if (ent_dtype == HCS_DTYPE_BF16) {
      uint32_t b = (uint32_t)__bfloat16_as_ushort(__float2bfloat16_rn(__uint_as_float(kv[i])));
      reinterpret_cast<uint32_t*>(ent)[i] = (b << 16) | pos;
    } else {
      // tf32 tile path: byte offset in the 16 x 64 fp32 slab, value RNA-rounded to tf32
      uint32_t t;
      asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(t) : "f"(__uint_as_float(kv[i])));
      reinterpret_cast<uint2*>(ent)[i] = make_uint2(tf32_slab_off(rc >> 6, rc & 63u), t);
    }
    if (i == 0 || (keys[i - 1] >> 10) != (k >> 10)) ent_ptr[k >> 10] = i;
    if (i == n - 1) ent_ptr[nchunks] = n;
  }
}


// Stable per-window bucketing of entries by chunk (see header).  Chunk range [k0, k0 + KR)
// per pass; windows with more chunks take several passes over their entries.
constexpr int kBucketRows = 16;
constexpr int kBucketThreads = 512;  // 16 warps: warp r walks row r
constexpr int kBucketChunks = 1536;  // chunks per pass (16 x 1536 x 4 B = 96 KB of counters: 2 CTAs/SM)

template <typename VT>
__global__ void __launch_bounds__(kBucketThreads, 2)
    k_tile_bucket(const int64_t* __restrict__ row_ptr, const int32_t* __restrict__ cond,
                  const VT* __restrict__ vals, const int32_t* __restrict__ tile_list, int64_t T,
                  const int64_t* __restrict__ chunk_ptr, const int64_t* __restrict__ ent_off, int64_t n_rows, int wh,
                  int ent_dtype, void* __restrict__ ent, int64_t* __restrict__ ent_ptr, int64_t nchunks) {
  extern __shared__ int32_t bcnt[];  // [kBucketRows][kBucketChunks], then tot/start [kBucketChunks]
  int32_t* bstart = bcnt + kBucketRows * kBucketChunks;
  __shared__ int32_t warp_tot[kBucketThreads / 32];
  __shared__ int32_t pass_total;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int64_t t = blockIdx.x; t < T; t += gridDim.x) {
    const int64_t w = tile_list[t];
    const int64_t rs = w * wh;
    const int nr = (int)(n_rows - rs < wh ? n_rows - rs : wh);
    const int64_t cbase = chunk_ptr[t];
    const int nch = (int)(chunk_ptr[t + 1] - cbase);
    const int64_t base_e = row_ptr[rs];
    int64_t out_base = ent_off[t];  // entries of chunks before this pass
    int64_t e0 = 0, e1 = 0;
    if (warp < nr) {
      e0 = row_ptr[rs + warp];
      e1 = row_ptr[rs + warp + 1];
    }
    for (int k0 = 0; k0 < nch; k0 += kBucketChunks) {
      const int kr = min(kBucketChunks, nch - k0);
      // this pass's entries of the row: a row's condensed columns ascend, so chunks
      // [k0, k0 + kr) are one contiguous segment [s0, s1) (binary search; whole row if 1 pass)
      int64_t s0 = e0, s1 = e1;
      if (nch > kBucketChunks && lane == 0 && e1 > e0) {
        auto lower = [&](int key) {
          int64_t lo = e0, hi = e1;
          while (lo < hi) {
            const int64_t mid = (lo + hi) >> 1;
            if (__ldg(cond + mid) < key) lo = mid + 1; else hi = mid;
          }
          return lo;
        };
        s0 = lower(k0 << 6);
        s1 = lower((k0 + kr) << 6);
      }
      s0 = __shfl_sync(0xffffffffu, s0, 0);
      s1 = __shfl_sync(0xffffffffu, s1, 0);
      for (int i = threadIdx.x; i < kBucketRows * kr; i += blockDim.x) bcnt[(i / kr) * kBucketChunks + i % kr] = 0;
      __syncthreads();
      // 1. per (row, chunk) counts (integer atomics: order-free)
      for (int64_t eb = s0 + lane; eb < s1; eb += 128) {  // 4 loads in flight per lane
        int cc[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) cc[u] = eb + 32 * u < s1 ? __ldg(cond + eb + 32 * u) : -1;
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int k = (cc[u] >> 6) - k0;
          if (cc[u] >= 0 && k >= 0 && k < kr) atomicAdd(&bcnt[warp * kBucketChunks + k], 1);
        }
      }
      __syncthreads();
      // 2. exclusive prefix over rows per chunk, chunk totals
      for (int k = threadIdx.x; k < kr; k += blockDim.x) {
        int run = 0;
#pragma unroll
        for (int r = 0; r < kBucketRows; ++r) {
          const int c = bcnt[r * kBucketChunks + k];
          bcnt[r * kBucketChunks + k] = run;
          run += c;
        }
        bstart[k] = run;
      }
      __syncthreads();
      // 3. exclusive scan of chunk totals (each thread a contiguous block of chunks)
      {
        const int per = (kr + blockDim.x - 1) / blockDim.x;
        const int a = threadIdx.x * per, b = min(kr, a + per);
        int run = 0;
        for (int k = a; k < b; ++k) run += bstart[k];
        int incl = run;  // block-wide inclusive scan of the per-thread sums
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const int v = __shfl_up_sync(0xffffffffu, incl, o);
          if (lane >= o) incl += v;
        }
        if (lane == 31) warp_tot[warp] = incl;
        __syncthreads();
        int woff = 0;
        for (int i = 0; i < warp; ++i) woff += warp_tot[i];
        int excl = woff + incl - run;
        for (int k = a; k < b; ++k) {
          const int c = bstart[k];
          bstart[k] = excl;
          excl += c;
        }
        if (threadIdx.x == blockDim.x - 1) pass_total = excl;
        __syncthreads();
      }
      for (int k = threadIdx.x; k < kr; k += blockDim.x) ent_ptr[cbase + k0 + k] = out_base + bstart[k];
      // 4. scatter in (chunk, row, column) order: rank inside a (row, chunk) segment from the
      //    row's sorted condensed columns (segment start = last chunk change at or before e)
      int64_t seg = s0;
      int prev_last = -1;  // condensed column of the entry before this block (row-local)
      int cn = s0 + lane < s1 ? __ldg(cond + s0 + lane) : 0;
      float vn = s0 + lane < s1 ? (float)vals[s0 + lane] : 0.f;
      for (int64_t eb = s0; eb < s1; eb += 32) {
        const int64_t e = eb + lane;
        const bool live = e < s1;
        const int c = cn;
        const float v = vn;
        if (eb + 32 + lane < s1) {  // prefetch the next block
          cn = __ldg(cond + eb + 32 + lane);
          vn = (float)vals[eb + 32 + lane];
        }
        const int k = (c >> 6) - k0;
        int cp = __shfl_up_sync(0xffffffffu, c, 1);
        if (lane == 0) cp = prev_last;
        prev_last = __shfl_sync(0xffffffffu, c, 31);
        const bool head = live && (e == s0 || (cp >> 6) != (c >> 6));
        const uint32_t hm = __ballot_sync(0xffffffffu, head) & (0xffffffffu >> (31 - lane));
        const int64_t st = hm ? eb + (31 - __clz(hm)) : seg;
        seg = __shfl_sync(0xffffffffu, st, 31);
        if (live && k >= 0 && k < kr) {
          const int64_t pos = out_base + bstart[k] + bcnt[warp * kBucketChunks + k] + (e - st);
          const uint32_t lr = (uint32_t)warp, cc = (uint32_t)(c & 63);
          if (ent_dtype == HCS_DTYPE_BF16) {
            const uint32_t bv = (uint32_t)__bfloat16_as_ushort(__float2bfloat16_rn(v));
            reinterpret_cast<uint32_t*>(ent)[pos] = (bv << 16) | sw128_kmajor_off16(lr, cc);
          } else {
            uint32_t tv;
            asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(tv) : "f"(v));
            reinterpret_cast<uint2*>(ent)[pos] = make_uint2(tf32_slab_off(lr, cc), tv);
          }
        }
      }
      // entries of this pass's chunks precede the next pass's
      __syncthreads();
      out_base += pass_total;
      __syncthreads();
    }
    (void)base_e;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) ent_ptr[nchunks] = ent_off[T];
}

static int g_plan_builder = 0;  // 0 = per-window bucketing (default), 1 = global radix sort

static int key_bits_for(int64_t nchunks) {
  int b = 1;
  while ((1LL << b) < nchunks + 1) ++b;
  return 10 + b;
}

static size_t cub_bytes(int64_t n, int64_t nchunks, int64_t T) {
  size_t a = 0, b = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, a, (uint64_t*)nullptr, (uint64_t*)nullptr, (uint32_t*)nullptr,
                                  (uint32_t*)nullptr, (int)std::max<int64_t>(n, 1), 0, key_bits_for(nchunks));
  cub::DeviceScan::InclusiveSum(nullptr, b, (int64_t*)nullptr, (int64_t*)nullptr, (int)(T + 1));
  return std::max(a, b);
}

}  // namespace hcs

using namespace hcs;

extern "C" {

int hcs_tile_plan_workspace_bytes(int64_t nnz_tile, int64_t nchunks, size_t* bytes) {
  HCS_REQUIRE(bytes != nullptr, HCS_EINVAL, "bytes is NULL");
  int64_t n = std::max<int64_t>(nnz_tile, 1);
  // T <= nchunks; the bucketing builder needs only the window offsets and the scan scratch
  const size_t sort_keys = g_plan_builder == 1 ? a256(n * 8) * 2 + a256(n * 4) * 2 : 0;
  *bytes = a256((nchunks + 2) * 8) + sort_keys + a256(cub_bytes(g_plan_builder == 1 ? n : 1, nchunks, nchunks));
  return HCS_OK;
}

int hcs_tile_plan(const int64_t* row_ptr, const int32_t* cond_cols, const void* values, int values_dtype,
                  const int64_t* win_col_ptr, const int32_t* nonzero_cols, int64_t n_rows, int64_t n_cols, int32_t wh,
                  const int32_t* tile_list, int64_t n_tile, const int64_t* chunk_ptr, int64_t nchunks, int32_t* gidx,
                  int64_t* ent_ptr, void* ent, int ent_dtype, int64_t nnz_tile, void* workspace, size_t ws_bytes,
                  void* stream) {
  HCS_REQUIRE(wh > 0 && wh <= 16, HCS_EINVAL, "tile path supports window heights 1..16 (got %d)", wh);
  HCS_REQUIRE(nnz_tile < (1LL << 31), HCS_EINVAL, "too many tile entries");
  size_t need = 0;
  hcs_tile_plan_workspace_bytes(nnz_tile, nchunks, &need);
  HCS_REQUIRE(ws_bytes >= need, HCS_EINVAL, "workspace too small (%zu < %zu)", ws_bytes, need);
  if (n_tile == 0) return HCS_OK;
  cudaStream_t st = as_stream(stream);
  const bool sorted_builder = g_plan_builder == 1;
  int64_t n = std::max<int64_t>(nnz_tile, 1);
  char* p = (char*)workspace;
  int64_t* ent_off = (int64_t*)p; p += a256((nchunks + 2) * 8);
  uint64_t *keys_a = nullptr, *keys_b = nullptr;
  uint32_t *kv_a = nullptr, *kv_b = nullptr;
  if (sorted_builder) {
    keys_a = (uint64_t*)p; p += a256(n * 8);
    keys_b = (uint64_t*)p; p += a256(n * 8);
    kv_a = (uint32_t*)p; p += a256(n * 4);
    kv_b = (uint32_t*)p; p += a256(n * 4);
  }
  void* tmp = p;
  size_t tmp_bytes = cub_bytes(sorted_builder ? n : 1, nchunks, n_tile);

  HCS_CUDA(cudaMemsetAsync(ent_off, 0, sizeof(int64_t) * (n_tile + 1), st));
  k_tile_nnz<<<(int)((n_tile + 255) / 256), 256, 0, st>>>(row_ptr, tile_list, n_tile, n_rows, wh, ent_off);
  HCS_LAUNCH_CHECK("k_tile_nnz");
  size_t tb = tmp_bytes;
  HCS_CUDA(cub::DeviceScan::InclusiveSum(tmp, tb, ent_off, ent_off, (int)(n_tile + 1), st));
  int grid = (int)std::min<int64_t>(n_tile, (int64_t)num_sms() * 8);
  k_tile_gidx<<<grid, 256, 0, st>>>(tile_list, n_tile, chunk_ptr, win_col_ptr, nonzero_cols, gidx);
  HCS_LAUNCH_CHECK("k_tile_gidx");
  if (!sorted_builder) {
    const int smem = (kBucketRows + 1) * kBucketChunks * (int)sizeof(int32_t);
    const int bgrid = (int)std::min<int64_t>(n_tile, (int64_t)num_sms() * 4);
    if (values_dtype == HCS_DTYPE_BF16) {
      HCS_CUDA(cudaFuncSetAttribute(k_tile_bucket<__nv_bfloat16>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
      k_tile_bucket<__nv_bfloat16><<<bgrid, kBucketThreads, smem, st>>>(
          row_ptr, cond_cols, (const __nv_bfloat16*)values, tile_list, n_tile, chunk_ptr, ent_off, n_rows, wh,
          ent_dtype, ent, ent_ptr, nchunks);
    } else {
      HCS_CUDA(cudaFuncSetAttribute(k_tile_bucket<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
      k_tile_bucket<float><<<bgrid, kBucketThreads, smem, st>>>(row_ptr, cond_cols, (const float*)values, tile_list,
                                                               n_tile, chunk_ptr, ent_off, n_rows, wh, ent_dtype, ent,
                                                               ent_ptr, nchunks);
    }
    HCS_LAUNCH_CHECK("k_tile_bucket");
    (void)n_cols;
    return HCS_OK;
  }
  if (values_dtype == HCS_DTYPE_BF16)
    k_tile_keys<__nv_bfloat16><<<grid, 512, 0, st>>>(row_ptr, cond_cols, (const __nv_bfloat16*)values, tile_list,
                                                      n_tile, chunk_ptr, ent_off, n_rows, wh, keys_a, kv_a);
  else
    k_tile_keys<float><<<grid, 512, 0, st>>>(row_ptr, cond_cols, (const float*)values, tile_list, n_tile, chunk_ptr,
                                             ent_off, n_rows, wh, keys_a, kv_a);
  HCS_LAUNCH_CHECK("k_tile_keys");
  if (nnz_tile == 0) return HCS_OK;
  tb = tmp_bytes;
  HCS_CUDA(cub::DeviceRadixSort::SortPairs(tmp, tb, keys_a, keys_b, kv_a, kv_b, (int)nnz_tile, 0,
                                           key_bits_for(nchunks), st));
  int g2 = (int)std::min<int64_t>((nnz_tile + 255) / 256, (int64_t)num_sms() * 16);
  k_tile_emit<<<g2, 256, 0, st>>>(keys_b, kv_b, nnz_tile, ent_dtype, ent, ent_ptr, nchunks);
  HCS_LAUNCH_CHECK("k_tile_emit");
  (void)n_cols;
  return HCS_OK;
}

// Plan builder: 0 = per-window bucketing (default), 1 = global radix sort (identical plans).
int hcs_set_tile_plan_builder(int builder) {
  HCS_REQUIRE(builder == 0 || builder == 1, HCS_EINVAL, "builder must be 0 or 1 (got %d)", builder);
  hcs::g_plan_builder = builder;
  return HCS_OK;
}

}  // extern "C"
