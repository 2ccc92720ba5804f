// K2: pack the TILE windows of an assignment into the tensor-core kernel's
// chunked format (the on-GPU counterpart of executors.py:129-135, where each
// tile window's entries are scattered into a zero-padded condensed slab and
// the matching X rows are gathered).
//
// A chunk is 64 consecutive condensed columns of one window.  Per chunk we keep
//   gidx[64]     : original column (= X row) of each condensed column, -1 = pad
//   entries      : packed (bf16 value << 16 | swizzled slab byte offset of (r, c)),
//                  in (row, column) order
// Entries are ordered deterministically by a radix sort on (chunk, position).
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
  // T <= nchunks
  *bytes = a256(n * 8) * 2 + a256(n * 4) * 2 + a256((nchunks + 2) * 8) + a256(cub_bytes(n, nchunks, nchunks));
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
  int64_t n = std::max<int64_t>(nnz_tile, 1);
  char* p = (char*)workspace;
  uint64_t* keys_a = (uint64_t*)p; p += a256(n * 8);
  uint64_t* keys_b = (uint64_t*)p; p += a256(n * 8);
  uint32_t* kv_a = (uint32_t*)p; p += a256(n * 4);
  uint32_t* kv_b = (uint32_t*)p; p += a256(n * 4);
  int64_t* ent_off = (int64_t*)p; p += a256((nchunks + 2) * 8);
  void* tmp = p;
  size_t tmp_bytes = cub_bytes(n, nchunks, n_tile);

  HCS_CUDA(cudaMemsetAsync(ent_off, 0, sizeof(int64_t) * (n_tile + 1), st));
  k_tile_nnz<<<(int)((n_tile + 255) / 256), 256, 0, st>>>(row_ptr, tile_list, n_tile, n_rows, wh, ent_off);
  HCS_LAUNCH_CHECK("k_tile_nnz");
  size_t tb = tmp_bytes;
  HCS_CUDA(cub::DeviceScan::InclusiveSum(tmp, tb, ent_off, ent_off, (int)(n_tile + 1), st));
  int grid = (int)std::min<int64_t>(n_tile, (int64_t)num_sms() * 8);
  k_tile_gidx<<<grid, 256, 0, st>>>(tile_list, n_tile, chunk_ptr, win_col_ptr, nonzero_cols, gidx);
  HCS_LAUNCH_CHECK("k_tile_gidx");
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

}  // extern "C"
