// K1: row-window partition + column condensation + features + selector.
//
// Restates, bit-exactly, /root/reference/pkg/src/rowwin/windows.py:81-106
// (partition: per-window np.unique(cols, return_inverse=True)), windows.py:109-123
// (features) and selector.py:48-56 (logistic decision), on the GPU.
//
// Two strategies produce identical integers:
//  * bitmap (n_cols <= kBitmapMaxCols): one CTA per window (grid-strided), the
//    window's distinct columns marked in a shared-memory bitmap; ncols counted from
//    atomicOr return values; ranks (cond_cols) from per-8-word popcount prefixes.
//  * sort (larger n_cols): CUB radix sort of (window, col) keys, run heads give the
//    ascending unique columns and the inverse index.
#include <cub/cub.cuh>

#include "common.cuh"

namespace hcs {

constexpr int64_t kBitmapMaxCols = 1400000;  // bitmap + prefix fit in 227 KB of smem
constexpr int kPartThreads = 1024;

struct Selector {
  double w_ncols, w_density, bias, mean0, mean1, scale0, scale1;
  int enabled;
};

static inline size_t bitmap_smem_bytes(int64_t n_cols) {
  int64_t nw = (n_cols + 31) / 32;
  int64_t ng = (nw + 7) / 8;
  return (size_t)(nw + ng + 64) * 4;
}

__device__ __forceinline__ int block_reduce_sum(int v, int* red) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  __syncthreads();
  if (lane == 0) red[warp] = v;
  __syncthreads();
  int nw = blockDim.x >> 5;
  int t = (threadIdx.x < nw) ? red[threadIdx.x] : 0;
  if (warp == 0) {
    for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
    if (lane == 0) red[32] = t;
  }
  __syncthreads();
  return red[32];
}

// ---- count: ncols per window (bitmap)
__global__ void __launch_bounds__(kPartThreads) k_count_bitmap(const int64_t* __restrict__ row_ptr,
                                                               const int32_t* __restrict__ col, int64_t n_rows,
                                                               int64_t n_cols, int wh, int64_t W,
                                                               int64_t* __restrict__ ncols_out) {
  extern __shared__ uint32_t sm[];
  int64_t nw = (n_cols + 31) / 32;
  uint32_t* bm = sm;
  int* red = reinterpret_cast<int*>(sm + nw + ((nw + 7) / 8));
  for (int64_t i = threadIdx.x; i < nw; i += blockDim.x) bm[i] = 0;
  __syncthreads();
  for (int64_t w = blockIdx.x; w < W; w += gridDim.x) {
    int64_t rs = w * wh, re = min(rs + wh, n_rows);
    int64_t e0 = row_ptr[rs], e1 = row_ptr[re];
    int cnt = 0;
    for (int64_t e = e0 + threadIdx.x; e < e1; e += blockDim.x) {
      uint32_t c = (uint32_t)col[e];
      uint32_t bit = 1u << (c & 31);
      uint32_t old = atomicOr(&bm[c >> 5], bit);
      cnt += (old & bit) ? 0 : 1;
    }
    int total = block_reduce_sum(cnt, red);
    for (int64_t e = e0 + threadIdx.x; e < e1; e += blockDim.x) bm[(uint32_t)col[e] >> 5] = 0;
    if (threadIdx.x == 0) ncols_out[w] = total;
    __syncthreads();
  }
}

// ---- fill: nonzero_cols + cond_cols (bitmap)
__global__ void __launch_bounds__(kPartThreads) k_fill_bitmap(const int64_t* __restrict__ row_ptr,
                                                              const int32_t* __restrict__ col, int64_t n_rows,
                                                              int64_t n_cols, int wh, int64_t W,
                                                              const int64_t* __restrict__ win_col_ptr,
                                                              int32_t* __restrict__ nonzero_cols,
                                                              int32_t* __restrict__ cond) {
  extern __shared__ uint32_t sm[];
  const int64_t nw = (n_cols + 31) / 32;
  const int64_t ng = (nw + 7) / 8;
  uint32_t* bm = sm;
  uint32_t* gpre = sm + nw;           // exclusive popcount prefix per 8-word group
  int* scan = reinterpret_cast<int*>(sm + nw + ng);  // 33 ints
  for (int64_t i = threadIdx.x; i < nw; i += blockDim.x) bm[i] = 0;
  __syncthreads();
  const int T = blockDim.x;
  const int64_t seg = (ng + T - 1) / T;
  for (int64_t w = blockIdx.x; w < W; w += gridDim.x) {
    int64_t rs = w * wh, re = min(rs + wh, n_rows);
    int64_t e0 = row_ptr[rs], e1 = row_ptr[re];
    if (e1 == e0) continue;  // uniform across the block
    for (int64_t e = e0 + threadIdx.x; e < e1; e += T) {
      uint32_t c = (uint32_t)col[e];
      atomicOr(&bm[c >> 5], 1u << (c & 31));
    }
    __syncthreads();
    // per-thread contiguous segment of groups: local sums
    int64_t g0 = threadIdx.x * seg, g1 = min(g0 + seg, ng);
    uint32_t local = 0;
    for (int64_t g = g0; g < g1; ++g) {
      uint32_t s = 0;
      int64_t w0 = g * 8, w1 = min(w0 + 8, nw);
      for (int64_t k = w0; k < w1; ++k) s += __popc(bm[k]);
      gpre[g] = s;
      local += s;
    }
    // block exclusive scan of `local`
    uint32_t incl = local;
    int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int o = 1; o < 32; o <<= 1) {
      uint32_t t = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += t;
    }
    if (lane == 31) scan[warp] = (int)incl;
    __syncthreads();
    if (warp == 0) {
      int v = (lane < (T >> 5)) ? scan[lane] : 0;
      int inc = v;
      for (int o = 1; o < 32; o <<= 1) {
        int t = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += t;
      }
      if (lane < (T >> 5)) scan[lane] = inc - v;  // exclusive warp offsets
    }
    __syncthreads();
    uint32_t run = (uint32_t)scan[warp] + incl - local;
    for (int64_t g = g0; g < g1; ++g) {
      uint32_t s = gpre[g];
      gpre[g] = run;
      run += s;
    }
    __syncthreads();
    // emit ascending nonzero columns
    int64_t base = win_col_ptr[w];
    for (int64_t k = threadIdx.x; k < nw; k += T) {
      uint32_t bits = bm[k];
      if (!bits) continue;
      uint32_t r = gpre[k >> 3];
      for (int64_t j = k & ~7LL; j < k; ++j) r += __popc(bm[j]);
      while (bits) {
        int b = __ffs(bits) - 1;
        bits &= bits - 1;
        nonzero_cols[base + r] = (int32_t)(k * 32 + b);
        ++r;
      }
    }
    // inverse index per entry
    for (int64_t e = e0 + threadIdx.x; e < e1; e += T) {
      uint32_t c = (uint32_t)col[e];
      uint32_t k = c >> 5;
      uint32_t r = gpre[k >> 3];
      for (uint32_t j = k & ~7u; j < k; ++j) r += __popc(bm[j]);
      r += __popc(bm[k] & ((1u << (c & 31)) - 1u));
      cond[e] = (int32_t)r;
    }
    __syncthreads();
    for (int64_t e = e0 + threadIdx.x; e < e1; e += T) bm[(uint32_t)col[e] >> 5] = 0;
    __syncthreads();
  }
}

// ---- sort path
__global__ void k_make_keys(const int64_t* __restrict__ row_ptr, const int32_t* __restrict__ col, int64_t n_rows,
                            int wh, uint64_t* __restrict__ keys, int32_t* __restrict__ vals) {
  int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  int lane = threadIdx.x & 31;
  for (int64_t r = warp; r < n_rows; r += nwarps) {
    uint64_t win = (uint64_t)(r / wh);
    for (int64_t e = row_ptr[r] + lane; e < row_ptr[r + 1]; e += 32) {
      keys[e] = (win << 32) | (uint32_t)col[e];
      vals[e] = (int32_t)e;
    }
  }
}

__global__ void k_count_heads(const uint64_t* __restrict__ keys, int64_t nnz, int64_t* __restrict__ ncols) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (; i < nnz; i += stride) {
    uint64_t k = keys[i];
    if (i == 0 || keys[i - 1] != k) atomicAdd(reinterpret_cast<unsigned long long*>(&ncols[k >> 32]), 1ull);
  }
}

__global__ void k_flags(const uint64_t* __restrict__ keys, int64_t nnz, int32_t* __restrict__ flags) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (; i < nnz; i += stride) flags[i] = (i == 0 || keys[i - 1] != keys[i]) ? 1 : 0;
}

__global__ void k_fill_sorted(const uint64_t* __restrict__ keys, const int32_t* __restrict__ pos,
                              const int32_t* __restrict__ uid_incl, int64_t nnz,
                              const int64_t* __restrict__ win_col_ptr, int32_t* __restrict__ nonzero_cols,
                              int32_t* __restrict__ cond) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (; i < nnz; i += stride) {
    uint64_t k = keys[i];
    int64_t g = (int64_t)uid_incl[i] - 1;  // global unique index
    int64_t win = (int64_t)(k >> 32);
    int64_t r = g - win_col_ptr[win];
    if (i == 0 || keys[i - 1] != k) nonzero_cols[g] = (int32_t)(uint32_t)(k & 0xffffffffu);
    cond[pos[i]] = (int32_t)r;
  }
}

// ---- features + selector (windows.py:109-123, selector.py:48-56)
__global__ void k_features(const int64_t* __restrict__ row_ptr, int64_t n_rows, int wh, int64_t W,
                           const int64_t* __restrict__ win_col_ptr, Selector sel, double* __restrict__ density,
                           double* __restrict__ ci, uint8_t* __restrict__ codes) {
  int64_t w = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (w >= W) return;
  int64_t rs = w * wh, re = min(rs + wh, n_rows);
  int64_t nnz = row_ptr[re] - row_ptr[rs];
  int64_t nc = win_col_ptr[w + 1] - win_col_ptr[w];
  int64_t rc = re - rs;
  double d = 0.0, c = 0.0;
  if (nc > 0) {
    // Python int/int true division of exact integers (< 2**53): one IEEE rn division
    d = __ddiv_rn((double)nnz, (double)(rc * nc));
    c = __ddiv_rn((double)nnz, (double)nc);
  }
  if (density) density[w] = d;
  if (ci) ci[w] = c;
  if (codes && sel.enabled) {
    uint8_t code = 0;  // SCALAR
    if (nc > 0) {
      double zn = __ddiv_rn(__dsub_rn((double)nc, sel.mean0), sel.scale0);
      double zd = __ddiv_rn(__dsub_rn(d, sel.mean1), sel.scale1);
      double s = __dadd_rn(__dadd_rn(__dmul_rn(sel.w_ncols, zn), __dmul_rn(sel.w_density, zd)), sel.bias);
      code = (s > 0.0) ? 0 : 1;  // selector.py:56: score > 0 -> SCALAR, else TILE
    }
    codes[w] = code;
  }
}

__global__ void k_classify(const int64_t* __restrict__ wcp, const double* __restrict__ dens, int64_t W, Selector s,
                           uint8_t* __restrict__ out) {
  int64_t w = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (w >= W) return;
  int64_t nc = wcp[w + 1] - wcp[w];
  uint8_t code = 0;
  if (nc > 0) {
    double zn = __ddiv_rn(__dsub_rn((double)nc, s.mean0), s.scale0);
    double zd = __ddiv_rn(__dsub_rn(dens[w], s.mean1), s.scale1);
    double sc = __dadd_rn(__dadd_rn(__dmul_rn(s.w_ncols, zn), __dmul_rn(s.w_density, zd)), s.bias);
    code = (sc > 0.0) ? 0 : 1;
  }
  out[w] = code;
}

static Selector make_selector(const double* s) {
  Selector sel{};
  if (s) {
    sel.w_ncols = s[0]; sel.w_density = s[1]; sel.bias = s[2];
    sel.mean0 = s[3]; sel.mean1 = s[4]; sel.scale0 = s[5]; sel.scale1 = s[6];
    sel.enabled = 1;
  }
  return sel;
}

struct SortWs {
  uint64_t* keys_a; uint64_t* keys_b; int32_t* vals_a; int32_t* vals_b; void* cub_tmp; size_t cub_bytes;
};

static int key_bits(int64_t W) {
  int b = 1;
  while ((1LL << b) < W) ++b;
  return 32 + b;
}

static size_t cub_sort_bytes(int64_t nnz, int64_t W) {
  size_t sort_bytes = 0, scan_bytes = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, sort_bytes, (uint64_t*)nullptr, (uint64_t*)nullptr, (int32_t*)nullptr,
                                  (int32_t*)nullptr, (int)nnz, 0, key_bits(W));
  cub::DeviceScan::InclusiveSum(nullptr, scan_bytes, (int32_t*)nullptr, (int32_t*)nullptr, (int)nnz);
  size_t s2 = 0;
  cub::DeviceScan::InclusiveSum(nullptr, s2, (int64_t*)nullptr, (int64_t*)nullptr, (int)(W + 1));
  return std::max(std::max(sort_bytes, scan_bytes), s2);
}

static size_t align_up(size_t x) { return (x + 255) & ~(size_t)255; }

static size_t sort_ws_bytes(int64_t nnz, int64_t W) {
  return align_up(nnz * 8) * 2 + align_up(nnz * 4) * 2 + align_up(cub_sort_bytes(nnz, W));
}

static SortWs carve(void* ws, int64_t nnz, int64_t W) {
  SortWs s{};
  char* p = (char*)ws;
  s.keys_a = (uint64_t*)p; p += align_up(nnz * 8);
  s.keys_b = (uint64_t*)p; p += align_up(nnz * 8);
  s.vals_a = (int32_t*)p; p += align_up(nnz * 4);
  s.vals_b = (int32_t*)p; p += align_up(nnz * 4);
  s.cub_tmp = p;
  s.cub_bytes = cub_sort_bytes(nnz, W);
  return s;
}

static size_t scan_ws_bytes(int64_t W) {
  size_t s = 0;
  cub::DeviceScan::InclusiveSum(nullptr, s, (int64_t*)nullptr, (int64_t*)nullptr, (int)(W + 1));
  return align_up(s);
}

static int check_common(const int64_t* row_ptr, const int32_t* col_idx, int64_t n_rows, int64_t n_cols,
                        int64_t nnz, int32_t wh) {
  HCS_REQUIRE(wh > 0, HCS_EINVAL, "window_height must be positive");
  HCS_REQUIRE(n_rows >= 0 && n_cols >= 0 && nnz >= 0, HCS_EINVAL, "negative dimensions");
  HCS_REQUIRE(nnz < (1LL << 31), HCS_EINVAL, "nnz %lld exceeds the int32 entry index range; shard the matrix",
              (long long)nnz);
  HCS_REQUIRE(n_cols < (1LL << 31), HCS_EINVAL, "n_cols exceeds int32 range");
  HCS_REQUIRE(n_rows == 0 || row_ptr != nullptr, HCS_EINVAL, "row_ptr is NULL");
  HCS_REQUIRE(nnz == 0 || col_idx != nullptr, HCS_EINVAL, "col_idx is NULL");
  return HCS_OK;
}

}  // namespace hcs

using namespace hcs;

extern "C" {

int hcs_partition_workspace_bytes(int64_t n_rows, int64_t n_cols, int64_t nnz, int32_t wh, size_t* bytes) {
  HCS_REQUIRE(bytes != nullptr, HCS_EINVAL, "bytes is NULL");
  HCS_REQUIRE(wh > 0, HCS_EINVAL, "window_height must be positive");
  int64_t W = (n_rows + wh - 1) / wh;
  size_t b = scan_ws_bytes(W);
  if (n_cols > kBitmapMaxCols && nnz > 0) b += sort_ws_bytes(nnz, W);
  *bytes = b;
  return HCS_OK;
}

int hcs_partition_count(const int64_t* row_ptr, const int32_t* col_idx, int64_t n_rows, int64_t n_cols, int64_t nnz,
                        int32_t wh, const double* selector, int64_t* win_col_ptr, double* density, double* ci,
                        uint8_t* codes, void* workspace, size_t ws_bytes, void* stream) {
  int rc = check_common(row_ptr, col_idx, n_rows, n_cols, nnz, wh);
  if (rc) return rc;
  cudaStream_t st = as_stream(stream);
  int64_t W = (n_rows + wh - 1) / wh;
  HCS_REQUIRE(win_col_ptr != nullptr, HCS_EINVAL, "win_col_ptr is NULL");
  size_t need = 0;
  hcs_partition_workspace_bytes(n_rows, n_cols, nnz, wh, &need);
  HCS_REQUIRE(ws_bytes >= need, HCS_EINVAL, "workspace too small (%zu < %zu)", ws_bytes, need);
  HCS_CUDA(cudaMemsetAsync(win_col_ptr, 0, sizeof(int64_t) * (W + 1), st));
  if (W == 0) return HCS_OK;
  size_t scan_bytes = scan_ws_bytes(W);
  if (nnz > 0) {
    if (n_cols <= kBitmapMaxCols) {
      size_t smem = bitmap_smem_bytes(n_cols) + 33 * 4;
      HCS_CUDA(cudaFuncSetAttribute(k_count_bitmap, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      int per_sm = smem > 100000 ? 1 : (smem > 50000 ? 2 : 4);
      int64_t grid = std::min<int64_t>(W, (int64_t)num_sms() * per_sm);
      k_count_bitmap<<<(int)grid, kPartThreads, smem, st>>>(row_ptr, col_idx, n_rows, n_cols, wh, W, win_col_ptr + 1);
      HCS_LAUNCH_CHECK("k_count_bitmap");
    } else {
      SortWs s = carve((char*)workspace + scan_bytes, nnz, W);
      int grid = std::min<int64_t>((n_rows + 7) / 8, (int64_t)num_sms() * 16);
      k_make_keys<<<grid, 256, 0, st>>>(row_ptr, col_idx, n_rows, wh, s.keys_a, s.vals_a);
      HCS_LAUNCH_CHECK("k_make_keys");
      size_t tb = s.cub_bytes;
      HCS_CUDA(cub::DeviceRadixSort::SortPairs(s.cub_tmp, tb, s.keys_a, s.keys_b, s.vals_a, s.vals_b, (int)nnz, 0,
                                               key_bits(W), st));
      int g2 = std::min<int64_t>((nnz + 255) / 256, (int64_t)num_sms() * 16);
      k_count_heads<<<g2, 256, 0, st>>>(s.keys_b, nnz, win_col_ptr + 1);
      HCS_LAUNCH_CHECK("k_count_heads");
    }
  }
  size_t sb = scan_bytes;
  HCS_CUDA(cub::DeviceScan::InclusiveSum(workspace, sb, win_col_ptr, win_col_ptr, (int)(W + 1), st));
  Selector sel = make_selector(selector);
  k_features<<<(int)((W + 255) / 256), 256, 0, st>>>(row_ptr, n_rows, wh, W, win_col_ptr, sel, density, ci, codes);
  HCS_LAUNCH_CHECK("k_features");
  return HCS_OK;
}

int hcs_partition_fill(const int64_t* row_ptr, const int32_t* col_idx, int64_t n_rows, int64_t n_cols, int64_t nnz,
                       int32_t wh, const int64_t* win_col_ptr, int32_t* nonzero_cols, int32_t* cond_cols,
                       void* workspace, size_t ws_bytes, void* stream) {
  int rc = check_common(row_ptr, col_idx, n_rows, n_cols, nnz, wh);
  if (rc) return rc;
  cudaStream_t st = as_stream(stream);
  int64_t W = (n_rows + wh - 1) / wh;
  if (W == 0 || nnz == 0) return HCS_OK;
  size_t need = 0;
  hcs_partition_workspace_bytes(n_rows, n_cols, nnz, wh, &need);
  HCS_REQUIRE(ws_bytes >= need, HCS_EINVAL, "workspace too small (%zu < %zu)", ws_bytes, need);
  if (n_cols <= kBitmapMaxCols) {
    size_t smem = bitmap_smem_bytes(n_cols) + 33 * 4;
    HCS_CUDA(cudaFuncSetAttribute(k_fill_bitmap, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    int per_sm = smem > 100000 ? 1 : (smem > 50000 ? 2 : 4);
    int64_t grid = std::min<int64_t>(W, (int64_t)num_sms() * per_sm);
    k_fill_bitmap<<<(int)grid, kPartThreads, smem, st>>>(row_ptr, col_idx, n_rows, n_cols, wh, W, win_col_ptr,
                                                          nonzero_cols, cond_cols);
    HCS_LAUNCH_CHECK("k_fill_bitmap");
  } else {
    size_t scan_bytes = scan_ws_bytes(W);
    SortWs s = carve((char*)workspace + scan_bytes, nnz, W);
    int g2 = std::min<int64_t>((nnz + 255) / 256, (int64_t)num_sms() * 16);
    int32_t* flags = s.vals_a;  // vals_a is free after the sort (sorted positions live in vals_b)
    k_flags<<<g2, 256, 0, st>>>(s.keys_b, nnz, flags);
    HCS_LAUNCH_CHECK("k_flags");
    size_t tb = s.cub_bytes;
    HCS_CUDA(cub::DeviceScan::InclusiveSum(s.cub_tmp, tb, flags, flags, (int)nnz, st));
    k_fill_sorted<<<g2, 256, 0, st>>>(s.keys_b, s.vals_b, flags, nnz, win_col_ptr, nonzero_cols, cond_cols);
    HCS_LAUNCH_CHECK("k_fill_sorted");
  }
  return HCS_OK;
}

int hcs_classify(const int64_t* win_col_ptr, const double* density, int64_t n_windows, const double* selector,
                 uint8_t* codes, void* stream) {
  HCS_REQUIRE(selector != nullptr, HCS_EINVAL, "selector is NULL");
  if (n_windows == 0) return HCS_OK;
  Selector sel = make_selector(selector);
  k_classify<<<(int)((n_windows + 255) / 256), 256, 0, as_stream(stream)>>>(win_col_ptr, density, n_windows, sel, codes);
  HCS_LAUNCH_CHECK("hcs_classify");
  return HCS_OK;
}

}  // extern "C"
