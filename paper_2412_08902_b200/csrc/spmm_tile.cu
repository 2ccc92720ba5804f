// K4: tensor-core tile path (executors.py:111-141 tile_window) on sm_100a.
//
// Per row window the condensed columns are processed in chunks of 64.  The
// reference multiplies a zero-padded row_count x 8*ceil(ncols/8) slab by the
// gathered X rows; here each chunk is one K=64 step of
//     D[f][r] += sum_k Xg[k][f] * S[r][k]            (D = Z^T of the window)
// issued as 4 x tcgen05.mma.kind::f16 (M=128 features, N=16 window rows, K=16):
//   A = gathered X rows, MN-major, 64B/128B-swizzled, staged by cp.async (LDGSTS)
//   B = the window's 16 x 64 slab, K-major, 128B-swizzled, built in smem
//   D = fp32 accumulator in TMEM (two 16-column buffers: the MMAs of window i+1
//       overlap the epilogue of window i).
// A pipeline stage holds G chunks (16 KB of gathered rows): G = 1 for dim <= 128,
// 2 for dim <= 64, 4 for dim <= 32, so per-stage overheads are amortised evenly.
//
// Warp roles (persistent CTA per SM, 12 warps):
//   w0-w3  producers : gather-index prefetch (cp.async into an index ring, D stages
//                      ahead) + 16-byte cp.async row gathers + packed-entry staging;
//                      completion tracked per thread with commit/wait_group, then
//                      published on an mbarrier.
//   w4-w5  builders  : zero + scatter a stage's entries into its B slabs (alternating)
//   w6     MMA       : one lane issues tcgen05.mma and commits to mbarriers
//   w8-w11 epilogue  : tcgen05.ld -> fp32 Z rows (coalesced 128B stores)
// Why cp.async and not TMA tile::gather4: on B200 gather4 sustains ~2.3 TB/s of
// 128B rows (one row per ~18 cycles per SM) while LDG/LDGSTS row gathers reach
// ~13 TB/s from L2 (tools/probe, profiles/).  Control data (indices, entry
// pointers) is prefetched far ahead because loads complete in issue order behind
// the gathers in the SM's L1TEX queue.
#include "common.cuh"
#include "mma_helpers.cuh"

namespace hcs {

// Warp roles (NP producer warps; NP in {4, 8, 16}):
//   [0, NP)        producers: X-row gathers (cp.async)
//   NP             gather-index ring loader (TMA bulk copies)
//   NP+1           packed-entry loader (TMA bulk copies) + stage records
//   NP+2, NP+3     B-slab builders (round-robin stages)
//   NP+4 .. NP+7   tcgen05 epilogue (TMEM lane quadrants 0-3) | mma.sync compute warps
//   NP+8           tcgen05.mma issuer (tcgen05 engine only)
// Gather throughput from L2 scales with the number of issuing warps
// (profiles/r01_probe_gather_smem.txt), hence NP > 4.
template <int NP, int ENGINE>
struct Roles {
  static constexpr int kProducers = NP;
  static constexpr int kIdxWarp = NP;
  static constexpr int kEntWarp = NP + 1;
  static constexpr int kBuilder0 = NP + 2;
  static constexpr int kBuilders = 2;
  static constexpr int kEpiWarp0 = NP + 4;
  static constexpr int kMmaWarp = NP + 8;
  static constexpr int kThreads = (NP + 8 + (ENGINE == 0 ? 1 : 0)) * 32;
  static_assert(kEpiWarp0 % 4 == 0, "epilogue warps must form an aligned warpgroup");
};
constexpr int kEntCapPerChunk = 128;
#ifndef HCS_TILE_NOINC
#define HCS_TILE_NOINC 1  // 1: cp.async.mbarrier.arrive.noinc completion, 0: commit/wait_group publish
#endif  // staged packed entries per chunk; the rest is read from global

// first t in [0, n] with a[t] >= v  (a non-decreasing, length n+1)
__device__ __forceinline__ int64_t lower_bound_i64(const int64_t* __restrict__ a, int64_t n, int64_t v) {
  int64_t lo = 0, hi = n;
  while (lo < hi) {
    int64_t mid = (lo + hi) >> 1;
    if (a[mid] < v) lo = mid + 1; else hi = mid;
  }
  return lo;
}

// Warp-cooperative prefetching reader of a monotone int64 array: lanes hold
// a[base .. base+95] in three registers; get(i) for base <= i < base+64.  The
// third block is requested 32+ steps before it is read.
struct I64Window {
  const int64_t* p;
  int64_t base, lim;
  int64_t a, b, c;
  __device__ __forceinline__ int64_t ld(int64_t i) const { return i < lim ? p[i] : 0; }
  __device__ __forceinline__ void init(const int64_t* p_, int64_t base_, int64_t lim_, int lane) {
    p = p_; base = base_; lim = lim_;
    a = ld(base + lane);
    b = ld(base + 32 + lane);
    c = ld(base + 64 + lane);
  }
  __device__ __forceinline__ void advance(int64_t i, int lane) {
    while (i >= base + 32) {
      a = b;
      b = c;
      base += 32;
      c = ld(base + 64 + lane);
    }
  }
  __device__ __forceinline__ int64_t get(int64_t i) const {
    const int d = (int)(i - base);  // warp-uniform
    return d < 32 ? __shfl_sync(0xffffffffu, a, d) : __shfl_sync(0xffffffffu, b, d - 32);
  }
};

// Deterministic stage sequence shared by every role: windows t in [tb0, tb1),
// each split into stages of up to G consecutive chunks.
template <int G>
struct StageIter {
  I64Window cp;  // chunk_ptr
  int64_t t, tb1, c, c_end;
  __device__ __forceinline__ void init(const int64_t* chunk_ptr, int64_t tb0, int64_t tb1_, int lane) {
    cp.init(chunk_ptr, tb0, tb1_ + 1, lane);
    t = tb0;
    tb1 = tb1_;
    if (t < tb1) {
      c = cp.get(t);
      c_end = cp.get(t + 1);
    }
  }
  __device__ __forceinline__ bool valid() const { return t < tb1; }
  __device__ __forceinline__ int g() const { return (int)(c_end - c < G ? c_end - c : G); }
  __device__ __forceinline__ bool first(int64_t c0) const { return c == c0; }
  __device__ __forceinline__ bool last() const { return c + G >= c_end; }
  __device__ __forceinline__ void next(int lane) {
    c += G;
    if (c >= c_end) {
      ++t;
      if (t < tb1) {
        cp.advance(t, lane);
        c = cp.get(t);
        c_end = cp.get(t + 1);
      }
    }
  }
};

// Optional wait-time instrumentation (hcs_debug_tile_profile): cycles spent in each
// wait, accumulated per CTA into prof[blockIdx.x * 16 + slot].
#define TPROF(slot, stmt)                                                        \
  do {                                                                           \
    if (prof) {                                                                  \
      const long long _t0 = clock64();                                           \
      stmt;                                                                      \
      if (lane == 0) atomicAdd(&prof[blockIdx.x * 16 + (slot)], (unsigned long long)(clock64() - _t0)); \
    } else {                                                                     \
      stmt;                                                                      \
    }                                                                            \
  } while (0)

// Fused GCN epilogue (K6/K7): the window's aggregated 16 x d_in tile is multiplied
// on chip by a d_in x d_out matrix M (W forward, W^T backward).  M^T is kept in
// shared memory as bf16 [kMaxOut][kLdw]; partial products of the feature-slice
// warps are summed in a fixed order through a 16 x kMaxOut fp32 buffer.
constexpr int kMaxOut = 128;
constexpr int kLdw = 128 + 8;  // bf16 elements per M^T row (padding breaks bank conflicts)

template <int VEC, bool FUSED = false>
struct TileCfg {
  // VEC: 16-byte vectors per gathered row (dim <= 8*VEC)
  static constexpr int ROWB = VEC <= 4 ? 64 : 128;             // smem bytes per gathered row per MN block
  static constexpr int NBLK = VEC > 8 ? 2 : 1;                 // MN (feature) blocks of 64 bf16
  static constexpr int G = VEC <= 4 ? 4 : (VEC <= 8 ? 2 : 1);  // chunks per stage
  static constexpr int LAYOUT = ROWB == 64 ? 4 : 2;             // UMMA SWIZZLE_64B / SWIZZLE_128B
  static constexpr int SBO = 8 * ROWB;                          // 8-row swizzle atom
  static constexpr int CHUNK_A = 64 * ROWB;                     // bytes of one chunk in one MN block
  static constexpr int STAGE_A = G * CHUNK_A * NBLK;            // 16 KB
  static constexpr int STAGE_SLAB = G * 2048;
  static constexpr int STAGE_ENT = G * kEntCapPerChunk * 4;
  static constexpr int STAGE_BYTES = STAGE_A + STAGE_SLAB + STAGE_ENT;
  static constexpr int IDX_SLOT = G * 64 * 4;
  static constexpr int IDX_SLOTS = 16;           // gather-index ring (TMA loader runs up to 16 stages ahead)
  static constexpr int RED_BYTES = 4 * 16 * 32 * 4;  // mma.sync K-split partial sums
  static constexpr int W_BYTES = FUSED ? kMaxOut * kLdw * 2 : 0;  // M^T, bf16
  static constexpr int REDF_BYTES = FUSED ? 16 * kMaxOut * 4 : 0;  // fused partial sums
  static constexpr int STAGES = (223 * 1024 - IDX_SLOTS * IDX_SLOT - RED_BYTES - W_BYTES - REDF_BYTES) / STAGE_BYTES;
  static constexpr int INFLIGHT = STAGES - 2;    // stages of gathers in flight per producer thread
  static constexpr int OFF_A = 0;
  static constexpr int OFF_SLAB = OFF_A + STAGES * STAGE_A;
  static constexpr int OFF_ENT = OFF_SLAB + STAGES * STAGE_SLAB;
  static constexpr int OFF_IDX = OFF_ENT + STAGES * STAGE_ENT;
  static constexpr int OFF_INFO = OFF_IDX + IDX_SLOTS * IDX_SLOT;
  static constexpr int OFF_RED = OFF_INFO + STAGES * 64;
  static constexpr int OFF_W = OFF_RED + RED_BYTES;
  static constexpr int OFF_REDF = OFF_W + W_BYTES;
  static constexpr int OFF_IDXG = OFF_REDF + REDF_BYTES;   // int g per index slot
  static constexpr int OFF_BAR = OFF_IDXG + IDX_SLOTS * 4;
  static constexpr int NBAR = 3 * STAGES + 4 + 2 * IDX_SLOTS;
  static constexpr int SMEM = OFF_BAR + NBAR * 8 + 16 + 1024;  // + alignment slack
  static_assert(SMEM <= 227 * 1024, "tile kernel shared memory budget");
  static_assert(STAGES >= 4, "pipeline too shallow");
};

// Per-stage record written by producer warp 0 (visible to consumers through the
// full -> built mbarrier chain): entry pointers of the stage's chunks and flags.
struct StageInfo {
  int64_t ep[5];  // ent_ptr[c .. c+g]
  int32_t g;
  int16_t flags;  // bit0: first stage of a window, bit1: last stage of a window
  int16_t skew;   // staged entry i lives at ent_stage[skew + i] (16-byte aligned bulk copy)
};

// number of stages of windows [tb0, tb1) (warp-cooperative)
template <int G>
__device__ __forceinline__ int64_t count_stages(const int64_t* __restrict__ chunk_ptr, int64_t tb0, int64_t tb1,
                                                int lane) {
  int64_t n = 0;
  for (int64_t t = tb0 + lane; t < tb1; t += 32) n += (chunk_ptr[t + 1] - chunk_ptr[t] + G - 1) / G;
  for (int o = 16; o > 0; o >>= 1) n += __shfl_xor_sync(0xffffffffu, n, o);
  return n;
}

// ENGINE 0: tcgen05.mma (M=128 features x N=16 rows, TMEM accumulators, epilogue warps)
// ENGINE 1: mma.sync m16n8k16 (ldmatrix-fed from the same smem stages; up to 4 compute
//           warps own 32 features each, fp32 accumulators in registers).
// Measured on B200 (tools/probe/mma_rate, hmma_rate): a tcgen05.mma has a ~45-cycle
// floor per instruction for N <= 64, so the 16-row window shape runs ~8x below the
// tensor-core peak, while HMMA.16816 sustains ~2 cycles per instruction per SM.

template <int VEC, int ENGINE, int NP, bool FUSED>
__global__ void __launch_bounds__(Roles<NP, ENGINE>::kThreads, 1)
    k_spmm_tile_bf16(const int32_t* __restrict__ tile_list, int64_t T, const int64_t* __restrict__ chunk_ptr,
                     const int32_t* __restrict__ gidx, const int64_t* __restrict__ ent_ptr,
                     const uint32_t* __restrict__ ent, int64_t n_rows, int wh, const __nv_bfloat16* __restrict__ x,
                     int64_t ldx, int vec, int dim, float* __restrict__ z, int64_t ldz,
                     unsigned long long* __restrict__ prof, const float* __restrict__ mw, int d_out,
                     float* __restrict__ out, int64_t ldo, int dbg) {
  using C = TileCfg<VEC, FUSED>;
  using R = Roles<NP, ENGINE>;
  constexpr int kProducers = R::kProducers, kIdxWarp = R::kIdxWarp, kEntWarp = R::kEntWarp;
  constexpr int kBuilder0 = R::kBuilder0, kEpiWarp0 = R::kEpiWarp0, kMmaWarp = R::kMmaWarp;
  constexpr int S = C::STAGES, G = C::G;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::OFF_BAR);
  uint64_t* full = bars;           // S: gathers + staged entries landed (kProducers arrivals)
  uint64_t* built = bars + S;      // S: B slabs built (1 arrival)
  uint64_t* empty = bars + 2 * S;  // S: MMAs of the stage done (tcgen05.commit)
  uint64_t* accf = bars + 3 * S;   // 2: accumulator ready for the epilogue
  uint64_t* acce = accf + 2;       // 2: accumulator drained (4 epilogue warps)
  uint64_t* idx_full = acce + 2;                 // IDX_SLOTS: index slot loaded (TMA tx)
  uint64_t* idx_empty = idx_full + C::IDX_SLOTS;  // IDX_SLOTS: index slot read by all producers
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(idx_empty + C::IDX_SLOTS);
  StageInfo* info = reinterpret_cast<StageInfo*>(smem + C::OFF_INFO);
  int32_t* idx_g = reinterpret_cast<int32_t*>(smem + C::OFF_IDXG);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const long long t_start = clock64();
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      // producers (per-lane cp.async arrivals, or one publish per warp) + entry loader (arrive.expect_tx)
      mbar_init(&full[s], (HCS_TILE_NOINC ? kProducers * 32 : kProducers) + 1);
      mbar_init(&built[s], 1);
      // tcgen05.commit | all mma.sync compute warps (FS feature slices x KS K-splits)
      mbar_init(&empty[s], ENGINE == 0 ? 1 : ((dim + 31) / 32) * ((dim + 31) / 32 >= 3 ? 1 : ((dim + 31) / 32 == 2 ? 2 : 4)));
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&accf[b], 1);
      mbar_init(&acce[b], 4);
    }
    for (int i = 0; i < C::IDX_SLOTS; ++i) {
      mbar_init(&idx_full[i], 1);
      mbar_init(&idx_empty[i], kProducers);
    }
    fence_barrier_init();
  }
  if (ENGINE == 0 && warp == 0) tmem_alloc<32>(tmem_slot);
  if (FUSED) {
    // M is [dim x d_out] fp32 row-major; smem holds M^T as bf16 [kMaxOut][kLdw], zero-padded
    __nv_bfloat16* wt = reinterpret_cast<__nv_bfloat16*>(smem + C::OFF_W);
    for (int i = threadIdx.x; i < kMaxOut * kLdw; i += blockDim.x) {
      const int n = i / kLdw, k = i % kLdw;
      wt[i] = __float2bfloat16_rn((n < d_out && k < dim) ? mw[(int64_t)k * d_out + n] : 0.f);
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = ENGINE == 0 ? *tmem_slot : 0u;
  const uint32_t sbase = smem_u32(smem);
  // contiguous, chunk-balanced range of tile windows for this CTA
  const int64_t Ctot = chunk_ptr[T];
  const int64_t Gd = gridDim.x;
  const int64_t tb0 = lower_bound_i64(chunk_ptr, T, (Ctot * (int64_t)blockIdx.x) / Gd);
  const int64_t tb1 = lower_bound_i64(chunk_ptr, T, (Ctot * ((int64_t)blockIdx.x + 1)) / Gd);

  if (warp < kProducers) {
    // ================================================================ producers
    const uint64_t keep = policy_evict_last();
    const int p = warp;
    constexpr int ROWS_W = 64 * G / kProducers;  // rows of a stage gathered by this warp
    constexpr int RPI = 32 / VEC;                // rows per warp instruction
    constexpr int ITERS = ROWS_W * VEC / 32;
    static_assert(ITERS >= 1 && ROWS_W % RPI == 0, "producer row split");
    const int lrow = lane / VEC, v = lane % VEC;
    const int row0 = ROWS_W * p;  // first stage row of this warp
    const char* xl = reinterpret_cast<const char*>(x + v * 8);
    const int64_t ldxb = ldx * 2;
    const uint32_t vbytes = (v < vec) ? 16u : 0u;  // lanes past dim zero-fill
    uint32_t dofs[ITERS];  // per-iteration smem destination offsets (relative to the stage's A base)
#pragma unroll
    for (int it = 0; it < ITERS; ++it) {
      const int row = row0 + it * RPI + lrow;
      const int jch = row >> 6, r = row & 63, vchunk = v & 7;
      uint32_t d = (uint32_t)(v >> 3) * (uint32_t)(G * C::CHUNK_A) + (uint32_t)jch * C::CHUNK_A;
      if (C::ROWB == 128) d += (uint32_t)r * 128u + ((uint32_t)(vchunk ^ (r & 7)) << 4);
      else d += (uint32_t)(r >> 3) * 512u + (uint32_t)(r & 7) * 64u + ((uint32_t)((vchunk ^ ((r & 7) >> 1)) & 3) << 4);
      dofs[it] = d;
    }
    const int nst = (int)count_stages<G>(chunk_ptr, tb0, tb1, lane);
    int stage = 0, sig = 0, pending = 0, islot = 0;
    uint32_t phase = 0, iphase = 0;
    for (int n = 0; n < nst; ++n) {
      TPROF(0, mbar_wait(&idx_full[islot], iphase));
      const int g = idx_g[islot];
      const int32_t* idx_s =
          reinterpret_cast<const int32_t*>(smem + C::OFF_IDX + islot * C::IDX_SLOT) + row0 + lrow;
      int gi[ITERS];
#pragma unroll
      for (int it = 0; it < ITERS; ++it) gi[it] = idx_s[it * RPI];
      __syncwarp();
      if (lane == 0) mbar_arrive(&idx_empty[islot]);
      if (++islot == C::IDX_SLOTS) { islot = 0; iphase ^= 1; }
      TPROF(1, mbar_wait(&empty[stage], phase ^ 1));
      const uint32_t a_st = sbase + C::OFF_A + stage * C::STAGE_A;
      const int lim = g * 64 - row0 - lrow;  // rows it*RPI < lim are valid
#pragma unroll
      for (int it = 0; it < ITERS; ++it) {
        if (G == 1 || it * RPI < lim) {
          if (!(dbg & 4))
            cp_async16(a_st + dofs[it], xl + (int64_t)max(gi[it], 0) * ldxb, gi[it] >= 0 ? vbytes : 0u, keep);
        }
      }
#if HCS_TILE_NOINC
      // each lane arrives on the stage's barrier once all its prior cp.async copies landed
      cp_async_arrive_noinc(&full[stage]);
#else
      cp_async_commit();
      if (++pending > C::INFLIGHT) {  // oldest in-flight stage has landed -> publish it
        TPROF(2, cp_async_wait<C::INFLIGHT>());
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) mbar_arrive(&full[sig]);
        if (++sig == S) sig = 0;
        --pending;
      }
#endif
      if (++stage == S) { stage = 0; phase ^= 1; }
    }
#if !HCS_TILE_NOINC
    cp_async_wait<0>();
    fence_proxy_async_smem();
    __syncwarp();
    for (; pending > 0; --pending) {
      if (lane == 0) mbar_arrive(&full[sig]);
      if (++sig == S) sig = 0;
    }
#endif
  } else if (warp == kIdxWarp) {
    // ================================================================ gather-index loader (TMA)
    const uint64_t strm = policy_evict_first();
    StageIter<G> cur;
    cur.init(chunk_ptr, tb0, tb1, lane);
    int islot = 0;
    uint32_t iphase = 0;
    for (; cur.valid(); cur.next(lane)) {
      const int g = cur.g();
      TPROF(3, mbar_wait(&idx_empty[islot], iphase ^ 1));
      if (lane == 0) {
        idx_g[islot] = g;
        if (dbg & 16) {
          mbar_arrive(&idx_full[islot]);
        } else {
        mbar_expect_tx(&idx_full[islot], (uint32_t)g * 256u);
        tma_bulk_g2s(sbase + C::OFF_IDX + islot * C::IDX_SLOT, gidx + cur.c * 64, (uint32_t)g * 256u,
                     &idx_full[islot], strm);
        }
      }
      __syncwarp();
      if (++islot == C::IDX_SLOTS) { islot = 0; iphase ^= 1; }
    }
  } else if (warp == kEntWarp) {
    // ================================================================ entry loader (TMA) + stage records
    const uint64_t strm = policy_evict_first();
    const char* entb = reinterpret_cast<const char*>(ent);
    StageIter<G> cur;
    cur.init(chunk_ptr, tb0, tb1, lane);
    I64Window ep;
    ep.init(ent_ptr, tb0 < tb1 ? chunk_ptr[tb0] : 0, chunk_ptr[tb1] + 1, lane);
    int stage = 0;
    uint32_t phase = 0;
    int64_t c0w = cur.valid() ? cur.c : 0;  // first chunk of the current window
    for (; cur.valid(); cur.next(lane)) {
      const int g = cur.g();
      ep.advance(cur.c, lane);
      int64_t epj[G + 1];
#pragma unroll
      for (int j = 0; j <= G; ++j) epj[j] = ep.get(cur.c + (j <= g ? j : g));
      const bool first = cur.c == c0w, last = cur.last();
      if (last) c0w = cur.c_end;
      // 16-byte aligned superset of the stage's entries, capped to the staging buffer
      const int64_t b0 = (epj[0] * 4) & ~(int64_t)15;
      const int64_t b1 = (epj[G] * 4 + 15) & ~(int64_t)15;
      const uint32_t bytes = (uint32_t)(b1 - b0 < C::STAGE_ENT ? b1 - b0 : C::STAGE_ENT);
      TPROF(4, mbar_wait(&empty[stage], phase ^ 1));
      if (lane == 0) {
#pragma unroll
        for (int j = 0; j <= G; ++j) info[stage].ep[j] = epj[j];
        info[stage].g = g;
        info[stage].flags = (int16_t)((first ? 1 : 0) | (last ? 2 : 0));
        info[stage].skew = (int16_t)((epj[0] * 4 - b0) >> 2);
        if (dbg & 8) mbar_arrive(&full[stage]);
        else mbar_expect_tx(&full[stage], bytes);
        if (bytes && !(dbg & 8)) tma_bulk_g2s(sbase + C::OFF_ENT + stage * C::STAGE_ENT, entb + b0, bytes, &full[stage], strm);
      }
      __syncwarp();
      if (++stage == S) { stage = 0; phase ^= 1; }
    }
  } else if (warp >= kBuilder0 && warp < kBuilder0 + R::kBuilders) {
    // ================================================================ slab builders (round-robin stages)
    constexpr int NB = R::kBuilders;
    const int b = warp - kBuilder0;
    const int64_t nst = count_stages<G>(chunk_ptr, tb0, tb1, lane);
    for (int64_t n = b; n < nst; n += NB) {
      const int stage = (int)(n % S);
      const uint32_t phase = (uint32_t)((n / S) & 1);
      TPROF(5, mbar_wait(&full[stage], phase));
      const StageInfo& inf = info[stage];
      const int g = inf.g;
      const int64_t e0 = inf.ep[0];
      const long long t_b0 = prof ? clock64() : 0;
      uint8_t* slab = smem + C::OFF_SLAB + stage * C::STAGE_SLAB;
      const int4 zero4 = make_int4(0, 0, 0, 0);
#pragma unroll
      for (int i = 0; i < G * 4; ++i) reinterpret_cast<int4*>(slab)[lane + 32 * i] = zero4;
      __syncwarp();
      const int skew = inf.skew;
      const uint32_t* es = reinterpret_cast<const uint32_t*>(smem + C::OFF_ENT + stage * C::STAGE_ENT) + skew;
      const int cap = G * kEntCapPerChunk - skew;  // entries available in the staged copy
      // entry = bf16 value << 16 | byte offset in its chunk's swizzled slab (precomputed by the plan)
      const int ne = (int)(inf.ep[g] - e0);
      if (dbg & 2) {
      } else if (ne <= cap) {
        // fast path: all entries staged; chunk j's slab starts 2 KB after chunk j-1's
        int bq[G];  // first entry of chunk q (q >= g: past the end)
#pragma unroll
        for (int q = 0; q < G; ++q) bq[q] = q < g ? (int)(inf.ep[q] - e0) : ne;
        for (int i0 = 0; i0 < ne; i0 += 128) {
          uint32_t w[4];
          int ii[4];
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            ii[u] = i0 + u * 32 + lane;
            w[u] = ii[u] < ne ? es[ii[u]] : 0u;
          }
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            if (ii[u] < ne) {
              int j = 0;  // chunk of entry ii[u]: ep boundaries (g <= 4)
#pragma unroll
              for (int q = 1; q < G; ++q) j += ii[u] >= bq[q] ? 1 : 0;
              *reinterpret_cast<uint16_t*>(slab + j * 2048 + (w[u] & 0x7FFu)) = (uint16_t)(w[u] >> 16);
            }
          }
        }
      } else {
        for (int j = 0; j < g; ++j) {
          const int lo = (int)(inf.ep[j] - e0), hi = (int)(inf.ep[j + 1] - e0);
          uint8_t* sl = slab + j * 2048;
          for (int i = lo + lane; i < hi; i += 32) {
            const uint32_t w = (i < cap) ? es[i] : ent[e0 + i];
            *reinterpret_cast<uint16_t*>(sl + (w & 0x7FFu)) = (uint16_t)(w >> 16);
          }
        }
      }
      fence_proxy_async_smem();
      __syncwarp();
      if (prof && lane == 0) atomicAdd(&prof[blockIdx.x * 16 + 14], (unsigned long long)(clock64() - t_b0));
      if (lane == 0) mbar_arrive(&built[stage]);
    }
  } else if (ENGINE == 1 && warp >= kEpiWarp0) {
    // ================================================================ HMMA compute warps
    // Warp cw owns feature slice fs = cw % FS (32 features) and the stage's chunks
    // j == kp (mod KS), kp = cw / FS; with KS > 1 the partial window sums are reduced
    // through shared memory in a fixed order (deterministic).
    const int FS = (dim + 31) / 32;                  // 1..4 feature slices
    const int KS = FS >= 3 ? 1 : (FS == 2 ? 2 : 4);  // K-split factor
    const int cw = warp - kEpiWarp0;
    const int fs = cw % FS, kp = cw / FS;
    const int ncw = FS * KS;
    if (cw < ncw) {
      const int f0 = fs * 32;
      const int64_t nst = count_stages<G>(chunk_ptr, tb0, tb1, lane);
      // lane-constant parts of the ldmatrix addresses
      const int ar = lane & 15, akc = lane >> 4;                           // A: row, k-chunk offset
      const int bk = (lane & 7) + ((lane >> 3) & 1) * 8, bfc = lane >> 4;  // B: k row, feature-chunk offset
      auto a_tile_off = [&](int row, int fchunk) -> uint32_t {  // gathered-row layout (see producers)
        const int jch = row >> 6, r = row & 63;
        if (C::ROWB == 128)
          return (uint32_t)(fchunk >> 3) * (uint32_t)(G * C::CHUNK_A) + (uint32_t)jch * C::CHUNK_A +
                 (uint32_t)r * 128u + ((uint32_t)((fchunk & 7) ^ (r & 7)) << 4);
        return (uint32_t)jch * C::CHUNK_A + (uint32_t)(r >> 3) * 512u + (uint32_t)(r & 7) * 64u +
               ((uint32_t)((fchunk ^ ((r & 7) >> 1)) & 3) << 4);
      };
      float* red = reinterpret_cast<float*>(smem + C::OFF_RED);  // [KS][FS][16][32]
      float acc[4][4];
#pragma unroll
      for (int i = 0; i < 4; ++i) acc[i][0] = acc[i][1] = acc[i][2] = acc[i][3] = 0.f;
      int64_t t = tb0;
      int64_t wid_next = (t < tb1) ? tile_list[t] : 0;
      int stage = 0;
      uint32_t phase = 0;
      for (int64_t n = 0; n < nst; ++n) {
        TPROF(6, mbar_wait(&built[stage], phase));
        const int g = info[stage].g, flags = info[stage].flags;
        const uint32_t a_st = sbase + C::OFF_A + stage * C::STAGE_A;
        const uint32_t b_st = sbase + C::OFF_SLAB + stage * C::STAGE_SLAB;
        // steps (j, ks) of this warp, software-pipelined: fragments of step s+1 load during the MMAs of s
        const int nsteps = ((g - kp + KS - 1) / KS) * 4;  // chunks kp, kp+KS, ... below g, 4 K-steps each
        (void)nsteps;
        for (int j = kp; j < ((dbg & 1) ? 0 : g); j += KS) {
          const uint32_t sl = b_st + j * 2048;
          // the 4 K-steps' fragments are all loaded before the MMAs (latency overlap)
          uint32_t a[4][4], b0[4][4], b1[4][4];
#pragma unroll
          for (int ks = 0; ks < 4; ++ks) {
            const int kc = 2 * ks + akc;
            ldsm_x4(a[ks], sl + ar * 128 + (((kc ^ ar) & 7) << 4));
            const int row = j * 64 + ks * 16 + bk;
            ldsm_x4_trans(b0[ks], a_st + a_tile_off(row, (f0 >> 3) + bfc));
            ldsm_x4_trans(b1[ks], a_st + a_tile_off(row, (f0 >> 3) + 2 + bfc));
          }
#pragma unroll
          for (int ks = 0; ks < 4; ++ks) {
            hmma_16816(acc[0], a[ks], b0[ks][0], b0[ks][1]);
            hmma_16816(acc[1], a[ks], b0[ks][2], b0[ks][3]);
            hmma_16816(acc[2], a[ks], b1[ks][0], b1[ks][1]);
            hmma_16816(acc[3], a[ks], b1[ks][2], b1[ks][3]);
          }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[stage]);
        if (flags & 2) {  // window done: (reduce partials) rows -> Z, reset accumulators
          const int64_t rs = wid_next * wh;
          const int rows = (int)(n_rows - rs < wh ? n_rows - rs : wh);
          ++t;
          wid_next = (t < tb1) ? tile_list[t] : 0;
          const int r0 = lane >> 2, cc = (lane & 3) * 2;
          if (KS > 1) {
            float* my = red + ((kp * FS + fs) * 16) * 32;
#pragma unroll
            for (int nt = 0; nt < 4; ++nt) {
              *reinterpret_cast<float2*>(my + r0 * 32 + nt * 8 + cc) = make_float2(acc[nt][0], acc[nt][1]);
              *reinterpret_cast<float2*>(my + (r0 + 8) * 32 + nt * 8 + cc) = make_float2(acc[nt][2], acc[nt][3]);
            }
            named_bar_sync(2, ncw * 32);
            if (kp == 0) {
#pragma unroll
              for (int nt = 0; nt < 4; ++nt) {
                for (int k = 1; k < KS; ++k) {
                  const float* o = red + ((k * FS + fs) * 16) * 32;
                  const float2 u = *reinterpret_cast<const float2*>(o + r0 * 32 + nt * 8 + cc);
                  const float2 w = *reinterpret_cast<const float2*>(o + (r0 + 8) * 32 + nt * 8 + cc);
                  acc[nt][0] += u.x; acc[nt][1] += u.y; acc[nt][2] += w.x; acc[nt][3] += w.y;
                }
              }
            }
          }
          if (kp == 0 && z != nullptr) {
#pragma unroll
            for (int nt = 0; nt < 4; ++nt) {
              const int f = f0 + nt * 8 + cc;
              if (f < dim) {
                if (r0 < rows)
                  *reinterpret_cast<float2*>(z + (rs + r0) * ldz + f) = make_float2(acc[nt][0], acc[nt][1]);
                if (r0 + 8 < rows)
                  *reinterpret_cast<float2*>(z + (rs + r0 + 8) * ldz + f) = make_float2(acc[nt][2], acc[nt][3]);
              }
            }
          }
          if (FUSED && kp == 0) {
            // out[16 x d_out] = Zw[16 x dim] . M: this warp's 32 features are two k16 steps whose
            // A fragments are exactly its accumulator fragments (n-tiles 2j, 2j+1); partials of
            // the FS feature-slice warps are summed in slice order 0..FS-1 (deterministic).
            uint32_t af[2][4];
#pragma unroll
            for (int j = 0; j < 2; ++j) {
              af[j][0] = pack_bf16(acc[2 * j][0], acc[2 * j][1]);
              af[j][1] = pack_bf16(acc[2 * j][2], acc[2 * j][3]);
              af[j][2] = pack_bf16(acc[2 * j + 1][0], acc[2 * j + 1][1]);
              af[j][3] = pack_bf16(acc[2 * j + 1][2], acc[2 * j + 1][3]);
            }
            const uint32_t* wt = reinterpret_cast<const uint32_t*>(smem + C::OFF_W);
            float* redf = reinterpret_cast<float*>(smem + C::OFF_REDF);  // [16][kMaxOut]
            const int g8 = lane >> 2, t4 = lane & 3;
            const int ntiles = (d_out + 7) >> 3;
            for (int ph = 0; ph < FS; ++ph) {
              if (ph == fs) {
                for (int n8 = 0; n8 < ntiles; ++n8) {
                  float c[4] = {0.f, 0.f, 0.f, 0.f};
                  const uint32_t* wrow = wt + ((n8 * 8 + g8) * kLdw + f0) / 2 + t4;
                  hmma_16816(c, af[0], wrow[0], wrow[4]);
                  hmma_16816(c, af[1], wrow[8], wrow[12]);
                  float2* p0 = reinterpret_cast<float2*>(redf + g8 * kMaxOut + n8 * 8 + 2 * t4);
                  float2* p1 = reinterpret_cast<float2*>(redf + (g8 + 8) * kMaxOut + n8 * 8 + 2 * t4);
                  if (ph == 0) {
                    *p0 = make_float2(c[0], c[1]);
                    *p1 = make_float2(c[2], c[3]);
                  } else {
                    const float2 u = *p0, w = *p1;
                    *p0 = make_float2(u.x + c[0], u.y + c[1]);
                    *p1 = make_float2(w.x + c[2], w.y + c[3]);
                  }
                }
              }
              named_bar_sync(3, FS * 32);
            }
            for (int i = fs * 32 + lane; i < rows * d_out; i += FS * 32) {
              const int r = i / d_out, j = i - r * d_out;
              out[(rs + r) * ldo + j] = redf[r * kMaxOut + j];
            }
            named_bar_sync(3, FS * 32);  // redf consumed before the next window overwrites it
          }
#pragma unroll
          for (int nt = 0; nt < 4; ++nt) acc[nt][0] = acc[nt][1] = acc[nt][2] = acc[nt][3] = 0.f;
          if (KS > 1) named_bar_sync(2, ncw * 32);  // partials consumed before the next window reuses them
        }
        if (++stage == S) { stage = 0; phase ^= 1; }
      }
    }
  } else if (ENGINE == 0 && warp == kMmaWarp) {
    // ================================================================ MMA issuer
    constexpr uint32_t idesc = umma_idesc(128, 16, 1, 1, 1, 0);
    // A: MN-major; NBLK == 2 -> second 64-feature block G*CHUNK_A bytes away.
    // NBLK == 1 (dim <= 64): LBO = 0 makes feature rows 64..127 alias 0..63 (discarded).
    const uint32_t lbo = (C::NBLK == 2) ? (uint32_t)(G * C::CHUNK_A) : 0u;
    constexpr uint32_t KSTEP_A = 16 * C::ROWB;  // 16 gathered rows per K=16 MMA
    const int64_t nst = count_stages<G>(chunk_ptr, tb0, tb1, lane);
    int stage = 0, acc = 0;
    uint32_t phase = 0, acc_phase = 0;
    for (int64_t n = 0; n < nst; ++n) {
      TPROF(6, mbar_wait(&built[stage], phase));
      const int g = info[stage].g, flags = info[stage].flags;
      const bool first = flags & 1, last = flags & 2;
      if (first) TPROF(7, mbar_wait(&acce[acc], acc_phase ^ 1));
      fence_proxy_async_smem();
      tc_fence_after();
      const long long t_mma0 = prof ? clock64() : 0;
      if (lane == 0) {
        const uint32_t a_st = sbase + C::OFF_A + stage * C::STAGE_A;
        const uint32_t b_st = sbase + C::OFF_SLAB + stage * C::STAGE_SLAB;
        for (int j = 0; j < g; ++j) {
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            const uint64_t ad = umma_sdesc(a_st + j * C::CHUNK_A + k * KSTEP_A, lbo, C::SBO, C::LAYOUT);
            const uint64_t bd = umma_sdesc(b_st + j * 2048 + k * 32, 0, 1024, 2);
            umma_f16(tmem + acc * 16, ad, bd, idesc, (first && j == 0 && k == 0) ? 0u : 1u);
          }
        }
        umma_commit(&empty[stage]);
        if (last) umma_commit(&accf[acc]);
      }
      __syncwarp();
      if (prof && lane == 0) atomicAdd(&prof[blockIdx.x * 16 + 9], (unsigned long long)(clock64() - t_mma0));
      if (last && ++acc == 2) { acc = 0; acc_phase ^= 1; }
      if (++stage == S) { stage = 0; phase ^= 1; }
    }
  } else if (ENGINE == 0 && warp >= kEpiWarp0) {
    // ================================================================ epilogue
    const int q = warp & 3;  // TMEM lane quadrant accessible to this warp
    int acc = 0;
    uint32_t acc_phase = 0;
    const int f = 32 * q + lane;
    for (int64_t t = tb0; t < tb1; ++t) {
      const int64_t w = tile_list[t];
      const int64_t rs = w * wh;
      const int rows = (int)(n_rows - rs < wh ? n_rows - rs : wh);
      // one warp polls the mbarrier; the other three block on a named barrier (no spinning)
      if (q == 0) TPROF(8, mbar_wait(&accf[acc], acc_phase));
      named_bar_sync(1, 128);
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
        for (int nr = 0; nr < 16; ++nr)
          if (nr < rows) __stcs(zp + (int64_t)nr * ldz, __uint_as_float(r[nr]));
      }
      if (++acc == 2) { acc = 0; acc_phase ^= 1; }
    }
  }
  if (prof && lane == 0) {
    atomicAdd(&prof[blockIdx.x * 16 + 10 + (warp < kProducers ? 0 : warp < kBuilder0 ? 1 : warp < kEpiWarp0 ? 2 : 3)],
              (unsigned long long)(clock64() - t_start));
  }
  tc_fence_before();
  __syncthreads();
  if (ENGINE == 0 && warp == 0) tmem_dealloc<32>(tmem);
  if (prof && threadIdx.x == 0) atomicAdd(&prof[blockIdx.x * 16 + 15], (unsigned long long)(clock64() - t_start));
}

static unsigned long long* g_tile_prof = nullptr;  // debug wait-time counters (nullptr = off)
static int g_tile_engine = -1;                     // -1 auto, 0 tcgen05, 1 mma.sync
static int g_tile_debug = 0;                       // experiment switches (bit0 no MMA, bit1 no build, bit2 no gather)
static int g_tile_producers = 4;                   // producer warps per CTA: 4, 8 or 16

template <int VEC, int ENGINE, int NP, bool FUSED = false>
static int launch_tile(int grid, cudaStream_t st, const int32_t* tile_list, int64_t n_tile, const int64_t* chunk_ptr,
                       const int32_t* gidx, const int64_t* ent_ptr, const uint32_t* ent, int64_t n_rows, int wh,
                       const __nv_bfloat16* x, int64_t ldx, int vec, int d, float* z, int64_t ldz,
                       const float* mw = nullptr, int d_out = 0, float* out = nullptr, int64_t ldo = 0) {
  using C = TileCfg<VEC, FUSED>;
  auto kern = k_spmm_tile_bf16<VEC, ENGINE, NP, FUSED>;
  HCS_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM));
  kern<<<grid, Roles<NP, ENGINE>::kThreads, C::SMEM, st>>>(tile_list, n_tile, chunk_ptr, gidx, ent_ptr, ent, n_rows, wh, x, ldx, vec,
                                            d, z, ldz, g_tile_prof, mw, d_out, out, ldo, g_tile_debug);
  HCS_LAUNCH_CHECK("k_spmm_tile_bf16");
  return HCS_OK;
}

}  // namespace hcs

using namespace hcs;

namespace hcs {
int spmm_tile_warp(const int32_t* tile_list, int64_t n_tile, const int64_t* chunk_ptr, const int32_t* gidx,
                   const int64_t* ent_ptr, const uint32_t* ent, int64_t n_rows, int wh, const __nv_bfloat16* x,
                   int64_t x_rows, int64_t ldx, int dim, float* z, int64_t ldz, float* scratch, int64_t scratch_floats,
                   cudaStream_t st);
int spmm_tile_warp_tf32(const int32_t* tile_list, int64_t n_tile, const int64_t* chunk_ptr, const int32_t* gidx,
                        const int64_t* ent_ptr, const uint2* ent, int64_t n_rows, int wh, const float* x, int64_t ldx,
                        int dim, float* z, int64_t ldz, float* scratch, int64_t scratch_floats, cudaStream_t st);
int gcn_tile_warp(const int32_t* tile_list, int64_t n_tile, const int64_t* chunk_ptr, const int32_t* gidx,
                  const int64_t* ent_ptr, const uint32_t* ent, int64_t n_rows, int wh, const __nv_bfloat16* x,
                  int64_t ldx, int dim, float* z, int64_t ldz, const float* m, int d_out, float* out, int64_t ldo,
                  float* scratch, int64_t scratch_floats, cudaStream_t st);
}  // namespace hcs

extern "C" int hcs_spmm_tile(const int32_t* tile_list, int64_t n_tile, const int64_t* chunk_ptr, const int32_t* gidx,
                             const int64_t* ent_ptr, const void* ent, int ent_dtype, int64_t n_rows, int32_t wh,
                             const void* x, int x_dtype, int64_t x_rows, int32_t dim, int64_t ldx, float* z,
                             int64_t ldz, void* workspace, size_t ws_bytes, void* stream) {
  HCS_REQUIRE(wh > 0 && wh <= 16, HCS_EINVAL, "tile path supports window heights 1..16 (got %d)", wh);
  HCS_REQUIRE(dim > 0, HCS_EINVAL, "dim must be positive");
  HCS_REQUIRE(((uintptr_t)x & 15) == 0, HCS_EINVAL, "x must be 16-byte aligned");
  HCS_REQUIRE(x_dtype == ent_dtype, HCS_EINVAL, "x and plan dtypes differ (%d vs %d)", x_dtype, ent_dtype);
  if (x_dtype == HCS_DTYPE_F32) {
    // tf32 tensor-core path (warp-independent kernel only)
    HCS_REQUIRE(ldx % 4 == 0 && ldx >= ((dim + 3) / 4) * 4, HCS_EINVAL, "ldx must be a multiple of 4 covering dim");
    HCS_REQUIRE(((uintptr_t)z & 7) == 0 && ldz % 2 == 0, HCS_EINVAL, "z must be 8-byte aligned with even ldz");
    if (n_tile == 0) return HCS_OK;
    return spmm_tile_warp_tf32(tile_list, n_tile, chunk_ptr, gidx, ent_ptr, (const uint2*)ent, n_rows, wh,
                               (const float*)x, ldx, dim, z, ldz, (float*)workspace,
                               (int64_t)(ws_bytes / sizeof(float)), as_stream(stream));
  }
  HCS_REQUIRE(x_dtype == HCS_DTYPE_BF16, HCS_EINVAL, "tile path: x dtype must be bf16 or f32 (tf32)");
  HCS_REQUIRE(ldx % 8 == 0 && ldx >= ((dim + 7) / 8) * 8, HCS_EINVAL, "ldx must be a multiple of 8 covering dim");
  if (n_tile == 0) return HCS_OK;
  cudaStream_t st = as_stream(stream);
  const int grid = (int)std::min<int64_t>(n_tile, num_sms());
  const uint32_t* e = (const uint32_t*)ent;
  const int eng = g_tile_engine >= 0 ? g_tile_engine : 2;  // auto: warp-independent kernel
  if (eng == 2) {
    HCS_REQUIRE(((uintptr_t)z & 7) == 0 && ldz % 2 == 0, HCS_EINVAL, "z must be 8-byte aligned with even ldz");
    return spmm_tile_warp(tile_list, n_tile, chunk_ptr, gidx, ent_ptr, (const uint32_t*)ent, n_rows, wh,
                          (const __nv_bfloat16*)x, x_rows, ldx, dim, z, ldz, (float*)workspace,
                          (int64_t)(ws_bytes / sizeof(float)), st);
  }
  for (int f0 = 0; f0 < dim; f0 += 128) {
    const int d = std::min(128, dim - f0);
    const int vec = (d + 7) / 8;
    const __nv_bfloat16* xs = reinterpret_cast<const __nv_bfloat16*>(x) + f0;
    float* zs = z + f0;
    const int engine = eng;
    int rc;
#define HCS_TILE_ARGS grid, st, tile_list, n_tile, chunk_ptr, gidx, ent_ptr, e, n_rows, wh, xs, ldx, vec, d, zs, ldz
#define HCS_TILE_NP(V, E)                                                         \
    (g_tile_producers == 4 ? launch_tile<V, E, 4>(HCS_TILE_ARGS)                  \
     : g_tile_producers == 16 ? launch_tile<V, E, 16>(HCS_TILE_ARGS)              \
                              : launch_tile<V, E, 8>(HCS_TILE_ARGS))
    if (engine == 0) {
      if (vec > 8) rc = HCS_TILE_NP(16, 0);
      else if (vec > 4) rc = HCS_TILE_NP(8, 0);
      else rc = HCS_TILE_NP(4, 0);
    } else {
      if (vec > 8) rc = HCS_TILE_NP(16, 1);
      else if (vec > 4) rc = HCS_TILE_NP(8, 1);
      else rc = HCS_TILE_NP(4, 1);
    }
#undef HCS_TILE_NP
#undef HCS_TILE_ARGS
    if (rc) return rc;
  }
  (void)x_rows;
  return HCS_OK;
}

// K6/K7: tile path with the fused GCN epilogue: out = (A_w X) M per TILE window, plus
// z = A_w X when z != NULL (the forward z_cache).  M: fp32 [dim x d_out] row-major device
// matrix (W forward, W^T backward); dim <= 128, d_out <= 128.  mma.sync engine.
extern "C" int hcs_gcn_tile(const int32_t* tile_list, int64_t n_tile, const int64_t* chunk_ptr, const int32_t* gidx,
                            const int64_t* ent_ptr, const void* ent, int ent_dtype, int64_t n_rows, int32_t wh,
                            const void* x, int x_dtype, int64_t x_rows, int32_t dim, int64_t ldx, float* z,
                            int64_t ldz, const float* m, int32_t d_out, float* out, int64_t ldo, void* workspace,
                            size_t ws_bytes, void* stream) {
  HCS_REQUIRE(wh > 0 && wh <= 16, HCS_EINVAL, "tile path supports window heights 1..16 (got %d)", wh);
  HCS_REQUIRE(dim > 0 && dim <= kMaxOut, HCS_EINVAL, "fused GCN tile path needs 1 <= d_in <= %d (got %d)", kMaxOut,
              dim);
  HCS_REQUIRE(d_out > 0 && d_out <= kMaxOut, HCS_EINVAL, "fused GCN tile path needs 1 <= d_out <= %d (got %d)",
              kMaxOut, d_out);
  HCS_REQUIRE(x_dtype == HCS_DTYPE_BF16 && ent_dtype == HCS_DTYPE_BF16, HCS_EINVAL,
              "tile path: only bf16 operands are implemented in this build");
  HCS_REQUIRE(ldx % 8 == 0 && ldx >= ((dim + 7) / 8) * 8, HCS_EINVAL, "ldx must be a multiple of 8 covering dim");
  HCS_REQUIRE(((uintptr_t)x & 15) == 0, HCS_EINVAL, "x must be 16-byte aligned");
  HCS_REQUIRE(m != nullptr && out != nullptr && ldo >= d_out, HCS_EINVAL, "fused GCN: bad M / out arguments");
  if (n_tile == 0) return HCS_OK;
  cudaStream_t st = as_stream(stream);
  const int grid = (int)std::min<int64_t>(n_tile, num_sms());
  const uint32_t* e = (const uint32_t*)ent;
  if (d_out <= 64 && (g_tile_engine < 0 || g_tile_engine == 2)) {
    HCS_REQUIRE(z == nullptr || (((uintptr_t)z & 7) == 0 && ldz % 2 == 0), HCS_EINVAL,
                "z must be 8-byte aligned with even ldz");
    return gcn_tile_warp(tile_list, n_tile, chunk_ptr, gidx, ent_ptr, e, n_rows, wh, (const __nv_bfloat16*)x, ldx, dim,
                         z, ldz, m, d_out, out, ldo, (float*)workspace, (int64_t)(ws_bytes / sizeof(float)), st);
  }
  const int vec = (dim + 7) / 8;
  const __nv_bfloat16* xs = reinterpret_cast<const __nv_bfloat16*>(x);
  float* zs = z;
  const int d = dim;
#define HCS_GCN_ARGS grid, st, tile_list, n_tile, chunk_ptr, gidx, ent_ptr, e, n_rows, wh, xs, ldx, vec, d, zs, ldz, \
                     m, d_out, out, ldo
  int rc;
  if (vec > 8) rc = launch_tile<16, 1, 4, true>(HCS_GCN_ARGS);
  else if (vec > 4) rc = launch_tile<8, 1, 4, true>(HCS_GCN_ARGS);
  else rc = launch_tile<4, 1, 4, true>(HCS_GCN_ARGS);
#undef HCS_GCN_ARGS
  (void)x_rows;
  return rc;
}

// Debug: enable (1) / disable (0) the tile kernel's wait-time counters, or read
// them (host_out != NULL: copies n counters, 16 per CTA, then clears them).
extern "C" int hcs_debug_tile_profile(int enable, unsigned long long* host_out, int n) {
  const int total = 16 * 1024;
  if (enable && !hcs::g_tile_prof) {
    HCS_CUDA(cudaMalloc(&hcs::g_tile_prof, total * sizeof(unsigned long long)));
    HCS_CUDA(cudaMemset(hcs::g_tile_prof, 0, total * sizeof(unsigned long long)));
  }
  if (host_out && hcs::g_tile_prof) {
    HCS_CUDA(cudaDeviceSynchronize());
    HCS_CUDA(cudaMemcpy(host_out, hcs::g_tile_prof, std::min(n, total) * sizeof(unsigned long long),
                        cudaMemcpyDeviceToHost));
    HCS_CUDA(cudaMemset(hcs::g_tile_prof, 0, total * sizeof(unsigned long long)));
  }
  if (!enable && hcs::g_tile_prof) {
    cudaFree(hcs::g_tile_prof);
    hcs::g_tile_prof = nullptr;
  }
  return HCS_OK;
}

// Experiment switches of the tile kernel (results are wrong when set): bit0 skip MMAs,
// bit1 skip slab builds, bit2 skip X-row gathers.  0 = normal operation.
extern "C" int hcs_debug_tile_switches(int bits) {
  hcs::g_tile_debug = bits;
  return HCS_OK;
}

// Producer (X-row gather) warps per CTA of the tile kernel: 4, 8 or 16.
extern "C" int hcs_set_tile_producers(int np) {
  HCS_REQUIRE(np == 4 || np == 8 || np == 16, HCS_EINVAL, "producer warps must be 4, 8 or 16 (got %d)", np);
  hcs::g_tile_producers = np;
  return HCS_OK;
}

// Select the tile-path MMA engine: -1 auto (default), 0 tcgen05.mma, 1 mma.sync m16n8k16.
extern "C" int hcs_set_tile_engine(int engine) {
  HCS_REQUIRE(engine >= -1 && engine <= 2, HCS_EINVAL,
              "engine must be -1 (auto), 0 (tcgen05), 1 (mma.sync pipeline) or 2 (warp-independent mma.sync)");
  hcs::g_tile_engine = engine;
  return HCS_OK;
}
