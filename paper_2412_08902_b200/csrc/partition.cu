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
//  * sort (larger n_cols): windows of <= 1024 entries sort their (col, entry) pairs inside one
//    CTA, larger ones go through one CUB segmented radix sort (the windows are contiguous
//    segments of the CSR); run heads -> ascending unique columns, scan of the flags -> ranks.
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

// ---- sort path.  Windows are contiguous in the CSR, so each is one segment of col_idx.
//  * windows of <= kCtaSortMax entries: one CTA sorts the (col, local entry) pairs in shared
//    memory (cub::BlockRadixSort, size classes 128 / 512 / 1024), then the run heads give the
//    ascending unique columns and a block scan of the head flags the inverse index;
//  * larger windows: one segmented radix sort (their segments only, column bits only), then a
//    CTA per window walks its sorted segment the same way.
// Both stage ranks (per entry) and unique columns (at the window's first entry offset), so
// hcs_partition_fill only copies them once win_col_ptr is known.
constexpr int kCtaSortMax = 1024;

__global__ void k_win_offsets(const int64_t* __restrict__ row_ptr, int64_t n_rows, int wh, int64_t W,
                              int32_t* __restrict__ woff, int32_t* __restrict__ iota, int64_t nnz) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t w = i; w <= W; w += stride) woff[w] = (int32_t)row_ptr[min(w * wh, n_rows)];
  for (int64_t e = i; e < nnz; e += stride) iota[e] = (int32_t)e;
}

template <int TH, int IT>
__global__ void __launch_bounds__(TH) k_win_sort(int64_t W, const int32_t* __restrict__ woff,
                                                 const int32_t* __restrict__ col, int lo, int end_bit,
                                                 int64_t* __restrict__ ncols_out, int32_t* __restrict__ stage_rank,
                                                 int32_t* __restrict__ stage_uniq) {
  using Sort = cub::BlockRadixSort<uint32_t, TH, IT, int32_t>;
  using Scan = cub::BlockScan<int, TH>;
  __shared__ union {
    typename Sort::TempStorage sort;
    typename Scan::TempStorage scan;
  } ts;
  __shared__ uint32_t last[TH];
  const int tid = threadIdx.x;
  for (int64_t w = blockIdx.x; w < W; w += gridDim.x) {
    const int32_t e0 = woff[w];
    const int n = woff[w + 1] - e0;
    if (n <= lo || n > TH * IT) continue;  // uniform across the block
    uint32_t k[IT];
    int32_t v[IT];
#pragma unroll
    for (int i = 0; i < IT; ++i) {  // striped load (the input order does not matter to the sort)
      const int idx = i * TH + tid;
      k[i] = idx < n ? (uint32_t)col[e0 + idx] : 0xFFFFFFFFu;  // pads sort after every column
      v[i] = idx;
    }
    Sort(ts.sort).Sort(k, v, 0, end_bit);  // blocked: thread tid holds sorted [tid*IT, tid*IT+IT)
    last[tid] = k[IT - 1];
    __syncthreads();
    int f[IT], r[IT];
    uint32_t prev = tid ? last[tid - 1] : 0u;
#pragma unroll
    for (int i = 0; i < IT; ++i) {
      const int p = tid * IT + i;
      f[i] = (p < n && (p == 0 || k[i] != prev)) ? 1 : 0;
      prev = k[i];
    }
    int total;
    Scan(ts.scan).ExclusiveSum(f, r, total);
#pragma unroll
    for (int i = 0; i < IT; ++i) {
      if (tid * IT + i < n) {
        const int rk = r[i] + f[i] - 1;
        if (f[i]) stage_uniq[e0 + rk] = (int32_t)k[i];
        stage_rank[e0 + v[i]] = rk;
      }
    }
    if (tid == 0) ncols_out[w] = total;
    __syncthreads();  // shared memory is reused by the next window
  }
}

template <int TH, int IT>
static int launch_win_sort(int64_t W, const int32_t* woff, const int32_t* col, int lo, int end_bit, int64_t* ncols,
                           int32_t* rank, int32_t* uniq, cudaStream_t st) {
  auto kern = k_win_sort<TH, IT>;
  int per_sm = 0;
  HCS_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, TH, 0));
  const int64_t grid = std::min<int64_t>(W, (int64_t)num_sms() * std::max(per_sm, 1));
  kern<<<(int)grid, TH, 0, st>>>(W, woff, col, lo, end_bit, ncols, rank, uniq);
  HCS_LAUNCH_CHECK("k_win_sort");
  return HCS_OK;
}

// windows above kCtaSortMax entries: list + segment bounds for the segmented sort
__global__ void k_big_flags(int64_t W, const int32_t* __restrict__ woff, int64_t* __restrict__ bidx) {
  const int64_t w = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (w >= W) return;
  bidx[w + 1] = (woff[w + 1] - woff[w]) > kCtaSortMax ? 1 : 0;
  if (w == 0) bidx[0] = 0;
}

// after the inclusive scan bidx[w] = number of big windows before w
__global__ void k_big_list(int64_t W, const int32_t* __restrict__ woff, const int64_t* __restrict__ bidx,
                           int32_t* __restrict__ big_w, int32_t* __restrict__ seg_b, int32_t* __restrict__ seg_e) {
  const int64_t w = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (w >= W || bidx[w + 1] == bidx[w]) return;
  const int64_t j = bidx[w];
  big_w[j] = (int32_t)w;
  seg_b[j] = woff[w];
  seg_e[j] = woff[w + 1];
}

constexpr int kWalkThreads = 256, kWalkItems = 4;
__global__ void __launch_bounds__(kWalkThreads) k_big_walk(int64_t nbig, const int32_t* __restrict__ big_w,
                                                           const int32_t* __restrict__ woff,
                                                           const uint32_t* __restrict__ keys,
                                                           const int32_t* __restrict__ vals,
                                                           int64_t* __restrict__ ncols_out,
                                                           int32_t* __restrict__ stage_rank,
                                                           int32_t* __restrict__ stage_uniq) {
  using Scan = cub::BlockScan<int, kWalkThreads>;
  __shared__ typename Scan::TempStorage ts;
  for (int64_t j = blockIdx.x; j < nbig; j += gridDim.x) {
    const int64_t w = big_w[j];
    const int32_t s0 = woff[w], s1 = woff[w + 1];
    int running = 0;
    for (int32_t c = s0; c < s1; c += kWalkThreads * kWalkItems) {
      uint32_t k[kWalkItems];
      int f[kWalkItems], r[kWalkItems];
      const int32_t p0 = c + threadIdx.x * kWalkItems;
      uint32_t prev = (p0 > s0 && p0 < s1) ? keys[p0 - 1] : 0u;
#pragma unroll
      for (int i = 0; i < kWalkItems; ++i) {
        const int32_t p = p0 + i;
        k[i] = p < s1 ? keys[p] : 0u;
        f[i] = (p < s1 && (p == s0 || k[i] != prev)) ? 1 : 0;
        prev = k[i];
      }
      int agg;
      Scan(ts).ExclusiveSum(f, r, agg);
#pragma unroll
      for (int i = 0; i < kWalkItems; ++i) {
        const int32_t p = p0 + i;
        if (p < s1) {
          const int rk = running + r[i] + f[i] - 1;
          if (f[i]) stage_uniq[s0 + rk] = (int32_t)k[i];
          stage_rank[vals[p]] = rk;
        }
      }
      running += agg;
      __syncthreads();  // scan storage reuse
    }
    if (threadIdx.x == 0) ncols_out[w] = running;
  }
}

// nonzero_cols of window w = its staged unique columns (one CTA per window, 4 loads in flight)
__global__ void __launch_bounds__(256) k_win_emit(int64_t W, const int32_t* __restrict__ woff,
                                                  const int64_t* __restrict__ wcp,
                                                  const int32_t* __restrict__ stage_uniq,
                                                  int32_t* __restrict__ nonzero_cols) {
  for (int64_t w = blockIdx.x; w < W; w += gridDim.x) {
    const int64_t b = wcp[w], n = wcp[w + 1] - b;
    const int32_t* src = stage_uniq + woff[w];
    for (int64_t i0 = 0; i0 < n; i0 += 4 * 256) {
      int32_t t[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int64_t i = i0 + u * 256 + threadIdx.x;
        t[u] = i < n ? src[i] : 0;
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int64_t i = i0 + u * 256 + threadIdx.x;
        if (i < n) nonzero_cols[b + i] = t[u];
      }
    }
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

// sort-path workspace (after the scan temp storage): key/value double buffers of the
// segmented sort, the staged ranks / unique columns, window offsets, big-window list,
// CUB temp storage
struct SortWs {
  uint32_t* keys_a; uint32_t* keys_b; int32_t* vals_a; int32_t* vals_b; int32_t* rank; int32_t* uniq;
  int32_t* woff; int64_t* bidx; int32_t* big_w; int32_t* seg_b; int32_t* seg_e; void* cub_tmp; size_t cub_bytes;
};

static size_t align_up(size_t x) { return (x + 255) & ~(size_t)255; }

static size_t cub_seg_bytes(int64_t nnz, int64_t W) {
  size_t b = 0, c = 0;
  cub::DoubleBuffer<uint32_t> k(nullptr, nullptr);
  cub::DoubleBuffer<int32_t> v(nullptr, nullptr);
  cub::DeviceSegmentedRadixSort::SortPairs(nullptr, b, k, v, (int)nnz, (int)W, (const int32_t*)nullptr,
                                           (const int32_t*)nullptr, 0, 32);
  cub::DeviceScan::InclusiveSum(nullptr, c, (int64_t*)nullptr, (int64_t*)nullptr, (int)(W + 1));
  return std::max(b, c);
}

static size_t sort_ws_bytes(int64_t nnz, int64_t W) {
  return align_up(nnz * 4) * 6 + align_up((W + 1) * 4) * 4 + align_up((W + 1) * 8) + align_up(cub_seg_bytes(nnz, W));
}

static SortWs carve(void* ws, int64_t nnz, int64_t W) {
  SortWs s{};
  char* p = (char*)ws;
  s.keys_a = (uint32_t*)p; p += align_up(nnz * 4);
  s.keys_b = (uint32_t*)p; p += align_up(nnz * 4);
  s.vals_a = (int32_t*)p; p += align_up(nnz * 4);
  s.vals_b = (int32_t*)p; p += align_up(nnz * 4);
  s.rank = (int32_t*)p; p += align_up(nnz * 4);
  s.uniq = (int32_t*)p; p += align_up(nnz * 4);
  s.woff = (int32_t*)p; p += align_up((W + 1) * 4);
  s.big_w = (int32_t*)p; p += align_up((W + 1) * 4);
  s.seg_b = (int32_t*)p; p += align_up((W + 1) * 4);
  s.seg_e = (int32_t*)p; p += align_up((W + 1) * 4);
  s.bidx = (int64_t*)p; p += align_up((W + 1) * 8);
  s.cub_tmp = p;
  s.cub_bytes = cub_seg_bytes(nnz, W);
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
      const int g = (int)std::min<int64_t>((std::max(nnz, W + 1) + 255) / 256, (int64_t)num_sms() * 16);
      k_win_offsets<<<g, 256, 0, st>>>(row_ptr, n_rows, wh, W, s.woff, s.vals_a, nnz);
      HCS_LAUNCH_CHECK("k_win_offsets");
      int end_bit = 1;
      while ((1LL << end_bit) <= n_cols) ++end_bit;  // every column < 2^end_bit - 1 = the pad key's bits
      int64_t* ncols = win_col_ptr + 1;
      rc = launch_win_sort<32, 4>(W, s.woff, col_idx, 0, end_bit, ncols, s.rank, s.uniq, st);
      if (rc == HCS_OK) rc = launch_win_sort<64, 8>(W, s.woff, col_idx, 128, end_bit, ncols, s.rank, s.uniq, st);
      if (rc == HCS_OK) rc = launch_win_sort<128, 8>(W, s.woff, col_idx, 512, end_bit, ncols, s.rank, s.uniq, st);
      if (rc != HCS_OK) return rc;
      const int g1 = (int)((W + 255) / 256);
      k_big_flags<<<g1, 256, 0, st>>>(W, s.woff, s.bidx);
      HCS_LAUNCH_CHECK("k_big_flags");
      size_t tb = s.cub_bytes;
      HCS_CUDA(cub::DeviceScan::InclusiveSum(s.cub_tmp, tb, s.bidx, s.bidx, (int)(W + 1), st));
      k_big_list<<<g1, 256, 0, st>>>(W, s.woff, s.bidx, s.big_w, s.seg_b, s.seg_e);
      HCS_LAUNCH_CHECK("k_big_list");
      int64_t nbig = 0;
      HCS_CUDA(cudaMemcpyAsync(&nbig, s.bidx + W, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
      HCS_CUDA(cudaStreamSynchronize(st));  // CUB's segment count is a host argument
      if (nbig > 0) {
        HCS_CUDA(cudaMemcpyAsync(s.keys_a, col_idx, nnz * 4, cudaMemcpyDeviceToDevice, st));
        cub::DoubleBuffer<uint32_t> keys(s.keys_a, s.keys_b);
        cub::DoubleBuffer<int32_t> vals(s.vals_a, s.vals_b);
        tb = s.cub_bytes;
        HCS_CUDA(cub::DeviceSegmentedRadixSort::SortPairs(s.cub_tmp, tb, keys, vals, (int)nnz, (int)nbig, s.seg_b,
                                                          s.seg_e, 0, end_bit, st));
        const int gw = (int)std::min<int64_t>(nbig, (int64_t)num_sms() * 8);
        k_big_walk<<<gw, kWalkThreads, 0, st>>>(nbig, s.big_w, s.woff, keys.Current(), vals.Current(), ncols, s.rank,
                                                s.uniq);
        HCS_LAUNCH_CHECK("k_big_walk");
      }
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
    SortWs s = carve((char*)workspace + scan_ws_bytes(W), nnz, W);  // staged by hcs_partition_count
    HCS_CUDA(cudaMemcpyAsync(cond_cols, s.rank, nnz * 4, cudaMemcpyDeviceToDevice, st));
    const int g = (int)std::min<int64_t>(W, (int64_t)num_sms() * 8);
    k_win_emit<<<g, 256, 0, st>>>(W, s.woff, win_col_ptr, s.uniq, nonzero_cols);
    HCS_LAUNCH_CHECK("k_win_emit");
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
