// K4: tensor-core tile path (executors.py:111-141 tile_window) on sm_100a.
//
// Per row window the condensed columns are processed in chunks of 64.  The
// reference multiplies a zero-padded row_count x 8*ceil(ncols/8) slab by the
// gathered X rows; here each chunk is one K=64 step of
//     D[f][r] += sum_k Xg[k][f] * S[r][k]            (D = Z^T of the window)
// issued as 4 x tcgen05.mma.kind::f16 (M=128 features, N=16 window rows, K=16):
//   A = gathered X rows, MN-major, 128B-swizzled, staged by cp.async (LDGSTS)
//   B = the window's 16 x 64 slab, K-major, 128B-swizzled, built in smem
//   D = fp32 accumulator in TMEM (two 16-column buffers: MMA of window i+1
//       overlaps the epilogue of window i).
// Warp roles (persistent CTA per SM):
//   w0-w1 producers  : cp.async 16B gathers of X rows + staged packed entries
//   w2    builder    : zero + scatter the chunk's entries into the B slab
//   w3    MMA issuer : one elected lane issues tcgen05.mma, commits to mbarriers
//   w4-w7 epilogue   : tcgen05.ld -> fp32 Z rows (coalesced 128B stores)
// Gathering with cp.async instead of TMA tile::gather4: measured on B200,
// gather4 sustains ~2.3 TB/s of 128B rows, LDG/LDGSTS row gathers ~13 TB/s
// from L2 (tools/probe, profiles/r01_probe.md).
#include "common.cuh"

namespace hcs {

constexpr int kTileThreads = 256;
constexpr int kEntCap = 512;  // staged packed entries per chunk (2 KB); rest read from global

struct TileSmem {
  int stages;
  uint32_t a_bytes;     // per stage
  uint32_t off_a, off_slab, off_ent, off_bar, total;
};

__host__ __device__ inline TileSmem tile_smem_layout(int nblk, int stages) {
  TileSmem L;
  L.stages = stages;
  L.a_bytes = (uint32_t)nblk * 64 * 128;
  L.off_a = 0;
  L.off_slab = L.off_a + stages * L.a_bytes;
  L.off_ent = L.off_slab + stages * 2048;
  L.off_bar = L.off_ent + stages * kEntCap * 4;
  L.total = L.off_bar + (3 * stages + 4) * 8 + 16;
  return L;
}

__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src, uint32_t src_bytes, uint64_t pol) {
  asm volatile("cp.async.cg.shared.global.L2::cache_hint [%0], [%1], 16, %2, %3;" ::"r"(dst), "l"(src),
               "r"(src_bytes), "l"(pol)
               : "memory");
}
__device__ __forceinline__ void cp_async4(uint32_t dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(dst), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_arrive_noinc(uint64_t* bar) {
  asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(bar)) : "memory");
}


// first t in [0, n] with a[t] >= v  (a non-decreasing, length n+1)
__device__ __forceinline__ int64_t lower_bound_i64(const int64_t* __restrict__ a, int64_t n, int64_t v) {
  int64_t lo = 0, hi = n;
  while (lo < hi) {
    int64_t mid = (lo + hi) >> 1;
    if (a[mid] < v) lo = mid + 1; else hi = mid;
  }
  return lo;
}

// warp-cooperative prefetching reader of a monotone int64 array (e.g. ent_ptr):
// lanes hold a[base .. base+63]; get(i) for base <= i < base+64.
struct I64Window {
  const int64_t* p;
  int64_t base, lim;  // valid indices < lim
  int64_t a, b;
  __device__ __forceinline__ void init(const int64_t* p_, int64_t base_, int64_t lim_, int lane) {
    p = p_; base = base_; lim = lim_;
    a = (base + lane < lim) ? p[base + lane] : 0;
    b = (base + 32 + lane < lim) ? p[base + 32 + lane] : 0;
  }
  __device__ __forceinline__ void advance(int64_t i, int lane) {
    while (i >= base + 32) {
      a = b;
      base += 32;
      b = (base + 32 + lane < lim) ? p[base + 32 + lane] : 0;
    }
  }
  __device__ __forceinline__ int64_t get(int64_t i) const {
    int d = (int)(i - base);
    int64_t va = __shfl_sync(0xffffffffu, a, d & 31);
    int64_t vb = __shfl_sync(0xffffffffu, b, d & 31);
    return d < 32 ? va : vb;
  }
};

template <int NBLK>
__global__ void __launch_bounds__(kTileThreads, 1)
    k_spmm_tile_bf16(const int32_t* __restrict__ tile_list, int64_t T, const int64_t* __restrict__ chunk_ptr,
                     const int32_t* __restrict__ gidx, const int64_t* __restrict__ ent_ptr,
                     const uint32_t* __restrict__ ent, int64_t n_rows, int wh, const __nv_bfloat16* __restrict__ x,
                     int64_t ldx, int vec, int dim, float* __restrict__ z, int64_t ldz, int stages) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  const TileSmem L = tile_smem_layout(NBLK, stages);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L.off_bar);
  uint64_t* full = bars;
  uint64_t* built = bars + stages;
  uint64_t* empty = bars + 2 * stages;
  uint64_t* accf = bars + 3 * stages;
  uint64_t* acce = accf + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acce + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < stages; ++s) {
      mbar_init(&full[s], 64);
      mbar_init(&built[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&accf[b], 1);
      mbar_init(&acce[b], 4);
    }
    fence_barrier_init();
  }
  if (warp == 0) tmem_alloc<32>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t sbase = smem_u32(smem);
  // contiguous, chunk-balanced range of tile windows for this CTA
  const int64_t C = chunk_ptr[T];
  const int64_t G = gridDim.x;
  const int64_t tb0 = lower_bound_i64(chunk_ptr, T, (C * (int64_t)blockIdx.x) / G);
  const int64_t tb1 = lower_bound_i64(chunk_ptr, T, (C * ((int64_t)blockIdx.x + 1)) / G);
  const int64_t cb0 = chunk_ptr[tb0], cb1 = chunk_ptr[tb1];

  if (warp < 2) {
    // ------------------------------------------------------------ producers
    const uint64_t keep = policy_evict_last();
    const uint64_t strm = stream_policy();
    const int p = warp;
    int stage = 0;
    uint32_t phase = 0;
    const int32_t* gp = gidx + 32 * p + lane;
    // gather-index prefetch ring, distance 4 chunks
    int i0 = (cb0 + 0 < cb1) ? ld_stream_s32(gp + (cb0 + 0) * 64, strm) : -1;
    int i1 = (cb0 + 1 < cb1) ? ld_stream_s32(gp + (cb0 + 1) * 64, strm) : -1;
    int i2 = (cb0 + 2 < cb1) ? ld_stream_s32(gp + (cb0 + 2) * 64, strm) : -1;
    int i3 = (cb0 + 3 < cb1) ? ld_stream_s32(gp + (cb0 + 3) * 64, strm) : -1;
    I64Window ep;
    ep.init(ent_ptr, cb0, cb1 + 1, lane);
    for (int64_t ch = cb0; ch < cb1; ++ch) {
      const int cur_idx = i0;
      i0 = i1; i1 = i2; i2 = i3;
      i3 = (ch + 4 < cb1) ? ld_stream_s32(gp + (ch + 4) * 64, strm) : -1;
      ep.advance(ch, lane);
      const int64_t e_lo = ep.get(ch), e_hi = ep.get(ch + 1);
      mbar_wait(&empty[stage], phase ^ 1);
      const uint32_t a_st = sbase + L.off_a + stage * L.a_bytes;
      for (int o = lane; o < 32 * vec; o += 32) {
        const int r = o / vec, v = o - r * vec;
        const int gi = __shfl_sync(__activemask(), cur_idx, r);
        const int row = 32 * p + r;
        const uint32_t dst = a_st + (uint32_t)(v >> 3) * 8192u + (uint32_t)row * 128u +
                             ((uint32_t)((v & 7) ^ (row & 7)) << 4);
        const __nv_bfloat16* src = (gi >= 0) ? x + (int64_t)gi * ldx + v * 8 : x;
        cp_async16(dst, src, gi >= 0 ? 16u : 0u, keep);
      }
      if (p == 0) {
        const int ne = (int)(e_hi - e_lo < kEntCap ? e_hi - e_lo : kEntCap);
        const uint32_t e_st = sbase + L.off_ent + stage * kEntCap * 4;
        for (int i = lane; i < ne; i += 32) cp_async4(e_st + i * 4, ent + e_lo + i);
      }
      cp_async_arrive_noinc(&full[stage]);
      if (++stage == stages) { stage = 0; phase ^= 1; }
    }
  } else if (warp == 2) {
    // ------------------------------------------------------------ slab builder
    int stage = 0;
    uint32_t phase = 0;
    I64Window ep;
    ep.init(ent_ptr, cb0, cb1 + 1, lane);
    for (int64_t ch = cb0; ch < cb1; ++ch) {
      ep.advance(ch, lane);
      const int64_t e_lo = ep.get(ch), e_hi = ep.get(ch + 1);
      mbar_wait(&full[stage], phase);
      uint8_t* slab = smem + L.off_slab + stage * 2048;
      const int4 zero4 = make_int4(0, 0, 0, 0);
#pragma unroll
      for (int i = 0; i < 4; ++i) reinterpret_cast<int4*>(slab)[lane + 32 * i] = zero4;
      __syncwarp();
      const uint32_t* es = reinterpret_cast<const uint32_t*>(smem + L.off_ent + stage * kEntCap * 4);
      const int ne = (int)(e_hi - e_lo);
      for (int i = lane; i < ne; i += 32) {
        const uint32_t w = (i < kEntCap) ? es[i] : ent[e_lo + i];
        const uint32_t pos = w & 1023u;
        *reinterpret_cast<uint16_t*>(slab + sw128_kmajor_off16(pos >> 6, pos & 63u)) = (uint16_t)(w >> 16);
      }
      fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) mbar_arrive(&built[stage]);
      if (++stage == stages) { stage = 0; phase ^= 1; }
    }
  } else if (warp == 3) {
    // ------------------------------------------------------------ MMA issuer
    constexpr uint32_t idesc = umma_idesc(128, 16, 1, 1, 1, 0);
    const uint32_t lbo = (NBLK == 2) ? 8192u : 0u;  // NBLK==1: features 64..127 alias 0..63 (discarded)
    int stage = 0;
    uint32_t phase = 0;
    int acc = 0;
    uint32_t acc_phase = 0;
    for (int64_t t = tb0; t < tb1; ++t) {
      const int64_t c0 = chunk_ptr[t], c1 = chunk_ptr[t + 1];
      mbar_wait(&acce[acc], acc_phase ^ 1);
      tc_fence_after();
      for (int64_t ch = c0; ch < c1; ++ch) {
        mbar_wait(&built[stage], phase);
        fence_proxy_async_smem();
        tc_fence_after();
        if (lane == 0) {
          const uint32_t a_st = sbase + L.off_a + stage * L.a_bytes;
          const uint32_t b_st = sbase + L.off_slab + stage * 2048;
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            const uint64_t ad = umma_sdesc(a_st + k * 2048, lbo, 1024);
            const uint64_t bd = umma_sdesc(b_st + k * 32, 0, 1024);
            umma_f16(tmem + acc * 16, ad, bd, idesc, (ch > c0 || k > 0) ? 1u : 0u);
          }
          umma_commit(&empty[stage]);
        }
        __syncwarp();
        if (++stage == stages) { stage = 0; phase ^= 1; }
      }
      if (lane == 0) umma_commit(&accf[acc]);
      __syncwarp();
      if (++acc == 2) { acc = 0; acc_phase ^= 1; }
    }
  } else {
    // ------------------------------------------------------------ epilogue
    const int q = warp & 3;  // TMEM lane quadrant accessible to this warp
    int acc = 0;
    uint32_t acc_phase = 0;
    const int f = 32 * q + lane;
    for (int64_t t = tb0; t < tb1; ++t) {
      const int64_t w = tile_list[t];
      const int64_t rs = w * wh;
      const int rows = (int)(n_rows - rs < wh ? n_rows - rs : wh);
      mbar_wait(&accf[acc], acc_phase);
      tc_fence_after();
      uint32_t r[16];
      tmem_ld16(tmem + ((uint32_t)(32 * q) << 16) + acc * 16, r);
      tmem_ld_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&acce[acc]);
      if (f < dim) {
        float* zp = z + rs * ldz + f;
#pragma unroll
        for (int n = 0; n < 16; ++n)
          if (n < rows) __stcs(zp + (int64_t)n * ldz, __uint_as_float(r[n]));
      }
      if (++acc == 2) { acc = 0; acc_phase ^= 1; }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc<32>(tmem);
}

}  // namespace hcs

using namespace hcs;

extern "C" int hcs_spmm_tile(const int32_t* tile_list, int64_t n_tile, const int64_t* chunk_ptr, const int32_t* gidx,
                             const int64_t* ent_ptr, const void* ent, int ent_dtype, int64_t n_rows, int32_t wh,
                             const void* x, int x_dtype, int64_t x_rows, int32_t dim, int64_t ldx, float* z,
                             int64_t ldz, void* stream) {
  HCS_REQUIRE(wh > 0 && wh <= 16, HCS_EINVAL, "tile path supports window heights 1..16 (got %d)", wh);
  HCS_REQUIRE(dim > 0, HCS_EINVAL, "dim must be positive");
  HCS_REQUIRE(x_dtype == HCS_DTYPE_BF16 && ent_dtype == HCS_DTYPE_BF16, HCS_EINVAL,
              "tile path: only bf16 operands are implemented in this build");
  HCS_REQUIRE(ldx % 8 == 0 && ldx >= ((dim + 7) / 8) * 8, HCS_EINVAL, "ldx must be a multiple of 8 covering dim");
  HCS_REQUIRE(((uintptr_t)x & 15) == 0, HCS_EINVAL, "x must be 16-byte aligned");
  if (n_tile == 0) return HCS_OK;
  cudaStream_t st = as_stream(stream);
  const int grid = (int)std::min<int64_t>(n_tile, num_sms());
  for (int f0 = 0; f0 < dim; f0 += 128) {
    const int d = std::min(128, dim - f0);
    const int vec = (d + 7) / 8;
    const int nblk = vec > 8 ? 2 : 1;
    int stages = nblk == 2 ? 10 : 16;
    TileSmem L = tile_smem_layout(nblk, stages);
    size_t smem = L.total + 1024;
    const __nv_bfloat16* xs = reinterpret_cast<const __nv_bfloat16*>(x) + f0;
    float* zs = z + f0;
    if (nblk == 2) {
      HCS_CUDA(cudaFuncSetAttribute(k_spmm_tile_bf16<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      k_spmm_tile_bf16<2><<<grid, kTileThreads, smem, st>>>(tile_list, n_tile, chunk_ptr, gidx, ent_ptr,
                                                            (const uint32_t*)ent, n_rows, wh, xs, ldx, vec, d, zs, ldz,
                                                            stages);
    } else {
      HCS_CUDA(cudaFuncSetAttribute(k_spmm_tile_bf16<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      k_spmm_tile_bf16<1><<<grid, kTileThreads, smem, st>>>(tile_list, n_tile, chunk_ptr, gidx, ent_ptr,
                                                            (const uint32_t*)ent, n_rows, wh, xs, ldx, vec, d, zs, ldz,
                                                            stages);
    }
    HCS_LAUNCH_CHECK("k_spmm_tile_bf16");
  }
  (void)x_rows;
  return HCS_OK;
}
