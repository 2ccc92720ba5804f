// K4 (default engine): warp-independent tensor-core tile path (executors.py:111-141
// tile_window) on sm_100a.
//
// Measured on B200 (profiles/r01_tile_switches_pipeline_engine_c2.txt): the warp-specialised
// producer/builder/MMA pipeline of round 1's first engine (cp.async/TMA producers, tcgen05.mma
// or mma.sync consumer; removed in round 2, in git history as csrc/spmm_tile.cu) spent ~3.8 ms of
// its 5.0 ms (C2, N = 128) in per-chunk cross-warp hand-offs alone.  Here every warp is an independent worker with
// its own cp.async ring, so no barrier is shared between warps on the per-chunk path:
//
//   unit  = (TILE window t, feature slice f) with 32- or 64-feature slices (SWV = 4 / 8
//           16-B vectors per row slice); a window's condensed columns are processed in the
//           K2 plan's 64-column chunks (tile_plan.cu);
//   warp  = a contiguous, exactly balanced range [a, b) of the flattened (unit, chunk)
//           sequence -- or, with paired slices (default for FS > 1), the FS warps of a
//           group walk one balanced range of (window, chunk) positions, one slice each, so
//           a chunk's plan is read once and an X row's slices are fetched together;
//           ranges may cut a unit, whose partial sums then go to two scratch slots per
//           warp; the last warp of the unit to finish adds them in range order
//           (deterministic, no float atomics; split_arrive below);
//   chunk = gather 64 X-row slices (cp.async 16 B, L2 evict_last, 3-stage ring per warp,
//           XOR-swizzled for conflict-free ldmatrix.trans), build the 16 x 64 bf16 slab
//           from the packed entries (prefetched into registers one chunk ahead; the slab is
//           kept zero by undoing each chunk's scatter), then 4 k16 steps x (2 SWV) n8 tiles
//           of mma.sync m16n8k16 with fp32 accumulators in registers;
//   store = the window's 16 x (8 SWV) fp32 slice straight to Z.
// The bound is the LSU: 8 + 4 SM cycles per 512 B gathered (cp.async + ldmatrix), see
// DESIGN.md section 4 and profiles/r01_probe_*.
#include "common.cuh"
#include "mma_helpers.cuh"

namespace hcs {

// warps per CTA of the 32- / 64-feature-slice kernels (overridable for tuning sweeps:
// tools/exp_tile_warps.sh); the 3-stage ring below is structural (P0..P3 rotation)
#ifndef HCS_TILE_WARPS4
#define HCS_TILE_WARPS4 16  // 12 -> 16: N <= 32 0.79 -> 0.77 ms (tools/exp_tile_warps.sh)
#endif
#ifndef HCS_TILE_WARPS8
#define HCS_TILE_WARPS8 8
#endif
// 128-B lines of packed entries past the chunk being loaded that are pulled into L2 one step
// early, 64-feature slices only (C2 N = 128 2.441 -> 2.404 ms, N = 64 1.200 -> 1.195; N = 32
// 0.815 -> 0.834, so not there; the tf32 kernel +1 %; prefetching the gather indices ahead instead
// cost +30 %: profiles/r02_exp_c5_tile.txt)
#ifndef HCS_PLAN_PF_ENTL
#define HCS_PLAN_PF_ENTL 4
#endif
constexpr int kWarpTileStages = 3;   // cp.async ring depth per warp
constexpr int kWarpSlabBytes = 16 * 64 * 2;
constexpr int kWarpEntRegs = 4;      // packed entries per lane held in registers (128 per chunk)

// SWV = 16-byte vectors per gathered row slice: 4 (32 features) or 8 (64 features).
template <int SWV>
struct WarpCfg {
  static constexpr int kFeat = 8 * SWV;                  // features per slice
  static constexpr int kRowBytes = 16 * SWV;             // bytes per gathered row slice
  static constexpr int kStageBytes = 64 * kRowBytes;     // 64 rows (one chunk)
  static constexpr int kWarps = SWV == 4 ? HCS_TILE_WARPS4 : (SWV == 8 ? HCS_TILE_WARPS8 : 4);  // warps per CTA (smem / register limited)
  static constexpr int kPerWarp = kWarpTileStages * kStageBytes + kWarpSlabBytes;
  static constexpr int kSmem = kWarps * kPerWarp + 128;
  static constexpr int kIssue = 2 * SWV;                 // cp.async instructions per chunk
  static constexpr int kSlot = 16 * kFeat;               // floats of one 16 x kFeat partial
  static constexpr int kOffW = kWarps * kPerWarp;        // fused GCN: M^T (bf16) after the warp regions
  static_assert(kSmem <= 227 * 1024, "smem");
  static_assert(SWV != 8 || kSmem + 64 * (128 + 8) * 2 <= 227 * 1024, "fused smem");
  // XOR swizzle of 16-B vector v of row r (conflict-free ldmatrix.trans over 8 consecutive rows)
  // (SWV = 4: two 64-B rows per 128-B line, bit 2 of the position alternates with r>>3 so the
  // 8 rows {8q + it} written by one cp.async instruction also spread over all banks)
  __device__ static __forceinline__ uint32_t off(int r, int v) {
    if (SWV == 4)
      return (uint32_t)(r >> 1) * 128u +
             ((uint32_t)(((r & 1) * 4 + v) ^ (((r >> 1) & 3) | (((r >> 3) & 1) << 2))) << 4);
    if (SWV == 16) return (uint32_t)r * 256u + ((uint32_t)((v & 8) | ((v ^ r) & 7)) << 4);
    return (uint32_t)r * 128u + ((uint32_t)(v ^ (r & 7)) << 4);
  }
};

// read-once plan data: L2 evict_first so it does not displace the X rows
__device__ __forceinline__ int32_t ld_plan_s32(const int32_t* p, uint64_t pol) {
  int32_t r;
  asm volatile("ld.global.nc.L2::cache_hint.s32 %0, [%1], %2;" : "=r"(r) : "l"(p), "l"(pol));
  return r;
}
__device__ __forceinline__ uint32_t ld_plan_u32(const uint32_t* p, uint64_t pol) {
  uint32_t r;
  asm volatile("ld.global.nc.L2::cache_hint.u32 %0, [%1], %2;" : "=r"(r) : "l"(p), "l"(pol));
  return r;
}
__device__ __forceinline__ int64_t ld_plan_s64(const int64_t* p, uint64_t pol) {
  int64_t r;
  asm volatile("ld.global.nc.L2::cache_hint.s64 %0, [%1], %2;" : "=l"(r) : "l"(p), "l"(pol));
  return r;
}

// Position in the flattened (unit, chunk) sequence of one warp.
struct ChunkPos {
  int64_t t;     // index into tile_list
  int64_t base;  // chunk_ptr[t]
  int64_t fi;    // flattened index
  int32_t f, j, nj;
};

__device__ __forceinline__ int64_t ldg64(const int64_t* p) { return __ldg(p); }

// unit containing flattened chunk index v (0 <= v < FS * (chunk_ptr[T] - chunk_ptr[0])).
// chunk_ptr may be a view into a larger plan (sub-range launches): flattened indices are
// relative to chunk_ptr[0], plan arrays (gidx, ent_ptr) are addressed with absolute chunks.
__device__ __forceinline__ ChunkPos locate(const int64_t* __restrict__ chunk_ptr, int64_t T, int FS, int64_t v) {
  const int64_t c0 = ldg64(chunk_ptr);
  int64_t lo = 0, hi = T;  // largest t with FS*(chunk_ptr[t]-c0) <= v
  while (hi - lo > 1) {
    const int64_t mid = (lo + hi) >> 1;
    if (FS * (ldg64(chunk_ptr + mid) - c0) <= v) lo = mid; else hi = mid;
  }
  ChunkPos p;
  p.t = lo;
  p.base = ldg64(chunk_ptr + lo);
  p.nj = (int32_t)(ldg64(chunk_ptr + lo + 1) - p.base);
  const int64_t rem = v - FS * (p.base - c0);
  p.f = (int32_t)(rem / p.nj);
  p.j = (int32_t)(rem - (int64_t)p.f * p.nj);
  p.fi = v;
  return p;
}

__device__ __forceinline__ void advance(ChunkPos& p, const int64_t* __restrict__ chunk_ptr, int64_t T, int FS) {
  ++p.fi;
  if (++p.j < p.nj) return;
  p.j = 0;
  if (++p.f < FS) return;
  p.f = 0;
  ++p.t;
  p.base += p.nj;
  p.nj = p.t < T ? (int32_t)(ldg64(chunk_ptr + p.t + 1) - p.base) : 1;  // past the end: never used
}

__device__ __forceinline__ void warp_range(int64_t total, int64_t nwarps, int64_t gw, int64_t& a, int64_t& b,
                                           const int64_t* __restrict__ wb = nullptr) {
  if (wb != nullptr) {  // cost-weighted bounds (k_tile_bounds): range g = [wb[g], wb[g + 1])
    a = __ldg(wb + gw);
    b = __ldg(wb + gw + 1);
    return;
  }
  a = (total * gw) / nwarps;
  b = (total * (gw + 1)) / nwarps;
}

// ---------------------------------------------------------------- split units, in-kernel
// A unit (or, for the fused out partials, a window) cut by warp-range boundaries is finished
// by the LAST of its warps to arrive: every participant writes its partial slot, fences and
// adds the number of positions it covered to the unit's counter (indexed by the opening
// warp); the one that completes the count sums the slots in range order (opener's tail slot
// 1, then each later warp's head slot 0) -- the same order whichever warp arrives last, so
// results are deterministic -- writes Z and resets the counter to zero for the next launch.
// Replaces round 1's fix-up launch (O(nwarps) scan per warp; 10 us on a 2 K-node graph).

// workspace layout: [z counters | out counters] (kCntWords u32 each) then the partial slots
constexpr int kMaxWarpsPerCta = 16;
inline int64_t tile_cnt_words() { return ((int64_t)num_sms() * kMaxWarpsPerCta + 31) / 32 * 32; }

// group of a balanced split of `total` positions over `ng` ranges that owns position v
// (largest g with floor(total * g / ng) <= v; see warp_range)
__device__ __forceinline__ int64_t range_owner(int64_t total, int64_t ng, int64_t v,
                                               const int64_t* __restrict__ wb = nullptr) {
  if (wb != nullptr) {  // largest g < ng with wb[g] <= v (empty ranges have wb[g] == wb[g + 1])
    int64_t lo = 0, hi = ng - 1;
    while (lo < hi) {
      const int64_t mid = (lo + hi + 1) >> 1;
      if (__ldg(wb + mid) <= v) lo = mid; else hi = mid - 1;
    }
    return lo;
  }
  return ((v + 1) * ng - 1) / total;
}

// all lanes: after writing this warp's slot for the split unit [us, ue); (a, b) = our range.
// Returns true in the warp that must reduce (the last to arrive).
__device__ __forceinline__ bool split_arrive(unsigned* cnt, int64_t us, int64_t ue, int64_t a, int64_t b, int lane) {
  __syncwarp();
  int last = 0;
  if (lane == 0) {
    const unsigned mine = (unsigned)((b < ue ? b : ue) - (a > us ? a : us));
    __threadfence();
    const unsigned old = atomicAdd(cnt, mine);
    if (old + mine == (unsigned)(ue - us)) {
      last = 1;
      *cnt = 0u;
    }
  }
  last = __shfl_sync(0xffffffffu, last, 0);
  if (last) __threadfence();
  return last != 0;
}

// acc = sum of the split unit's partial slots in range order. Slots of warp w: slots + (2w + s) *
// SLOT floats (s = 1: the unit it opened, s = 0: the unit it continued); warp of group k = k * FSm + fw.
template <int NT, int SLOT>
__device__ __forceinline__ void split_reduce(const float* __restrict__ slots, int64_t total, int64_t ng, int64_t g_o,
                                             int FSm, int fw, int64_t ue, float (&acc)[NT][4], int lane,
                                             const int64_t* __restrict__ wb = nullptr) {
  const float* s = slots + ((g_o * FSm + fw) * 2 + 1) * (int64_t)SLOT;
#pragma unroll
  for (int nt = 0; nt < NT; ++nt)
#pragma unroll
    for (int q = 0; q < 4; ++q) acc[nt][q] = __ldcg(s + (nt * 4 + q) * 32 + lane);
  // range bounds floor(total * k / ng) stepped incrementally (no 64-bit division in the loop)
  const int64_t tq = total / ng, tr = total - tq * ng;
  int64_t bk = (total * (g_o + 1)) / ng, br = total * (g_o + 1) - bk * ng;
  if (wb != nullptr) bk = __ldg(wb + g_o + 1);
  for (int64_t k = g_o + 1; k < ng; ++k) {
    const int64_t ak = bk;
    if (wb != nullptr) {
      bk = __ldg(wb + k + 1);
    } else {
      bk += tq;
      br += tr;
      if (br >= ng) {
        ++bk;
        br -= ng;
      }
    }
    if (ak >= bk) continue;
    const float* sk = slots + ((k * FSm + fw) * 2 + 0) * (int64_t)SLOT;
#pragma unroll
    for (int nt = 0; nt < NT; ++nt)
#pragma unroll
      for (int q = 0; q < 4; ++q) acc[nt][q] += __ldcg(sk + (nt * 4 + q) * 32 + lane);
    if (ue <= bk) break;
  }
}

// the out counters follow the z counters (grid = num_sms() for every tile launch)
__device__ __forceinline__ int64_t tile_cnt_words_dev() {
  return ((int64_t)gridDim.x * kMaxWarpsPerCta + 31) / 32 * 32;
}

template <int NT>
__device__ __forceinline__ void write_slot(float* __restrict__ slot, const float (&acc)[NT][4], int lane) {
#pragma unroll
  for (int nt = 0; nt < NT; ++nt)
#pragma unroll
    for (int q = 0; q < 4; ++q) __stcg(slot + (nt * 4 + q) * 32 + lane, acc[nt][q]);
}

template <int SWV>
__device__ __forceinline__ void store_slice(float* __restrict__ z, int64_t ldz, int64_t rs, int rows, int dim, int f,
                                            const float (&acc)[SWV][4], int lane) {
  const int r0 = lane >> 2, cc = (lane & 3) * 2;
#pragma unroll
  for (int nt = 0; nt < SWV; ++nt) {
    const int col = f * (8 * SWV) + nt * 8 + cc;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int r = r0 + 8 * h;
      if (r < rows) {
        float* zp = z + (rs + r) * ldz + col;
        if (col + 1 < dim) {
          *reinterpret_cast<float2*>(zp) = make_float2(acc[nt][2 * h], acc[nt][2 * h + 1]);
        } else if (col < dim) {
          zp[0] = acc[nt][2 * h];
        }
      }
    }
  }
}

// tf32 kernel's slice (permuted n8 tiles): lane (g, t) holds features 8t..8t+7 of rows g, g+8 as
// acc[0..3][0], acc[0..3][1] (row g) and acc[0..3][2], acc[0..3][3] (row g+8)
__device__ __forceinline__ void store_slice_tf32p(float* __restrict__ z, int64_t ldz, int64_t rs, int rows, int dim,
                                                  int f, const float (&acc)[4][4], int lane) {
  const int r0 = lane >> 2, c0 = f * 32 + (lane & 3) * 8;
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int r = r0 + 8 * h;
    if (r >= rows) continue;
    float* zp = z + (rs + r) * ldz + c0;
#pragma unroll
    for (int q = 0; q < 4; ++q) {  // features c0 + 2q, c0 + 2q + 1
      const int j0 = 2 * q, j1 = 2 * q + 1;
      const float v0 = acc[j0 & 3][2 * h + (j0 >> 2)], v1 = acc[j1 & 3][2 * h + (j1 >> 2)];
      if (c0 + j1 < dim) {
        *reinterpret_cast<float2*>(zp + j0) = make_float2(v0, v1);
      } else if (c0 + j0 < dim) {
        zp[j0] = v0;
      }
    }
  }
}

constexpr int kFusedOutMax = 64;        // d_out of the warp kernel's fused epilogue
constexpr int kFusedLdw = 128 + 8;      // bf16 per M^T row (d_in <= 128)
constexpr int kOutSlot = 16 * kFusedOutMax;

// fused epilogue: a window's 16 x d_out out rows (accumulator layout of m16n8 tiles)
template <int NO>
__device__ __forceinline__ void store_out(float* __restrict__ out, int64_t ldo, int64_t rs, int rows, int d_out,
                                          const float (&oacc)[NO][4], int lane) {
  const int r0 = lane >> 2, cc = (lane & 3) * 2;
#pragma unroll
  for (int n8 = 0; n8 < NO; ++n8)
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int r = r0 + 8 * (q >> 1), col = n8 * 8 + cc + (q & 1);
      if (r < rows && col < d_out) out[(rs + r) * ldo + col] = oacc[n8][q];
    }
}

// Split-unit finish for Z: arrive on the unit's counter; the last warp sums the slots and stores.
// Everything that locates the unit in the balanced split is recomputed here from kernel
// parameters (rare path), so none of it stays live across the gather/MMA loop (the 32-feature
// kernel runs at its 128-register cap).  unit = (window chunk base, slice f) of a sequence of
// FSr = (paired ? 1 : FS) slices per window; warp of group k = k * FSm + fw (FSm = paired ? FS : 1).
template <int SWV, int SLOT, bool PERM = false>
__device__ __forceinline__ void finish_split_z(const int64_t* __restrict__ chunk_ptr, int64_t T, int FS, int paired,
                                               int warps_per_cta, unsigned* __restrict__ cnt,
                                               const float* __restrict__ slots, float* __restrict__ z, int64_t ldz,
                                               int64_t base, int f, int nj, int64_t rs, int rows, int dim,
                                               const int64_t* __restrict__ wb = nullptr) {
  const int lane = threadIdx.x & 31;
  const int64_t gw = (int64_t)blockIdx.x * warps_per_cta + (threadIdx.x >> 5);
  const int64_t nwarps = (int64_t)gridDim.x * warps_per_cta;
  const int FSr = paired ? 1 : FS, FSm = paired ? FS : 1;
  const int fw = paired ? (int)(gw % FS) : 0;
  const int64_t ng = nwarps / FSm, gi = gw / FSm;
  const int64_t c0 = __ldg(chunk_ptr);
  const int64_t total = (int64_t)FSr * (__ldg(chunk_ptr + T) - c0);
  int64_t a, b;
  warp_range(total, ng, gi, a, b, wb);
  const int64_t us = (int64_t)FSr * (base - c0) + (int64_t)f * nj;
  const int64_t g_o = range_owner(total, ng, us, wb);
  if (!split_arrive(cnt + g_o * FSm + fw, us, us + nj, a, b, lane)) return;
  float acc[SWV][4];
  split_reduce<SWV, SLOT>(slots, total, ng, g_o, FSm, fw, us + nj, acc, lane, wb);
  if constexpr (PERM) {
    store_slice_tf32p(z, ldz, rs, rows, dim, f + fw, acc, lane);
  } else {
    store_slice<SWV>(z, ldz, rs, rows, dim, f + fw, acc, lane);
  }
}

// the same for a window's fused out rows (window = positions [FSr (base - c0), + FSr nj) of the
// group sequence; one out partial per group, slot 2g + s; counters follow the z counters)
__device__ __forceinline__ void finish_split_out(const int64_t* __restrict__ chunk_ptr, int64_t T, int FS,
                                                 int paired, int warps_per_cta, unsigned* __restrict__ cnt,
                                                 const float* __restrict__ oslots, float* __restrict__ out,
                                                 int64_t ldo, int64_t base, int nj, int64_t rs, int rows, int d_out,
                                                 const int64_t* __restrict__ wb = nullptr) {
  const int lane = threadIdx.x & 31;
  const int FSr = paired ? 1 : FS, FSm = paired ? FS : 1;
  const int64_t gw = (int64_t)blockIdx.x * warps_per_cta + (threadIdx.x >> 5);
  const int64_t ng = (int64_t)gridDim.x * warps_per_cta / FSm;
  const int64_t c0 = __ldg(chunk_ptr);
  const int64_t total = (int64_t)FSr * (__ldg(chunk_ptr + T) - c0);
  int64_t a, b;
  warp_range(total, ng, gw / FSm, a, b, wb);
  const int64_t ws = (int64_t)FSr * (base - c0), we = ws + (int64_t)FSr * nj;
  const int64_t g_o = range_owner(total, ng, ws, wb);
  if (!split_arrive(cnt + tile_cnt_words_dev() + g_o, ws, we, a, b, lane)) return;
  float oacc[kFusedOutMax / 8][4];
  split_reduce<kFusedOutMax / 8, kOutSlot>(oslots, total, ng, g_o, 1, 0, we, oacc, lane, wb);
  store_out(out, ldo, rs, rows, d_out, oacc, lane);
}

// Fused GCN epilogue (K6/K7) of the warp kernel: after each (window, slice) unit the
// warp multiplies its 16 x 64 aggregated slice (bf16 A fragments taken straight from the
// accumulators) by the matching 64 x d_out block of M (bf16 M^T resident in shared
// memory) into an out accumulator; a window's out rows are written when its last slice
// is done, or summed in warp order by the last of its warps to finish when a warp boundary cuts it.

// NPR = 16-feature groups of a slice that hold features (compile time, so the unrolled
// ldmatrix/mma schedule is kept): SWV/2, or 3 for a single 33..48-feature slice (the 41-wide
// GCN gradient), whose last group is neither gathered nor multiplied.
template <int SWV, bool FUSED, int NPR = SWV / 2, bool WB = false>
__global__ void __launch_bounds__(WarpCfg<SWV>::kWarps * 32, 1)
    k_tile_warp(const int32_t* __restrict__ tile_list, int64_t T, const int64_t* __restrict__ chunk_ptr,
                const int32_t* __restrict__ gidx, const int64_t* __restrict__ ent_ptr,
                const uint32_t* __restrict__ ent, int64_t n_rows, int wh, const __nv_bfloat16* __restrict__ x,
                int64_t ldx, int dim, int FS, float* __restrict__ z, int64_t ldz, float* __restrict__ scratch,
                const float* __restrict__ mw, int d_out, float* __restrict__ out, int64_t ldo,
                float* __restrict__ oscratch, int paired, unsigned* __restrict__ cnt,
                const int64_t* __restrict__ wb_arg) {
  using C = WarpCfg<SWV>;
  // WB: cost-weighted warp ranges from k_tile_bounds (a separate instantiation, so the uniform
  // kernel's code is unchanged by the weighted path: +6 % on C2 when both shared one body)
  const int64_t* wb = WB ? wb_arg : nullptr;
  constexpr int kWarpTileWarps = C::kWarps, kWarpStageBytes = C::kStageBytes, kWarpSmemPerWarp = C::kPerWarp;
  constexpr int NI = C::kIssue;
  extern __shared__ uint8_t wsmem_raw[];
  uint8_t* wsmem = (uint8_t*)(((uintptr_t)wsmem_raw + 127) & ~(uintptr_t)127);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t nwarps = (int64_t)gridDim.x * kWarpTileWarps;
  const int64_t gw = (int64_t)blockIdx.x * kWarpTileWarps + warp;
  const int64_t c0 = chunk_ptr[0];
  // paired slices (FS > 1, not FUSED): warps gw = g*FS + f of a group g walk the same balanced
  // range of (window, chunk) positions, warp f doing feature slice f, so a window's slices run
  // side by side (the plan is read once from DRAM, an X row's slices are fetched together).
  // Otherwise one warp walks the flattened (window, slice, chunk) sequence.
  const int FSr = paired ? 1 : FS;
  const int fw = paired ? (int)(gw % FS) : 0;
  const int64_t ngroups = paired ? nwarps / FS : nwarps;
  const int64_t total = (int64_t)FSr * (chunk_ptr[T] - c0);
  int64_t a = 0, b = 0;
  if (!paired || gw < ngroups * FS) warp_range(total, ngroups, paired ? gw / FS : gw, a, b, wb);
  if (FUSED) {
    __nv_bfloat16* wt = reinterpret_cast<__nv_bfloat16*>(wsmem + C::kOffW);
    for (int i = threadIdx.x; i < kFusedOutMax * kFusedLdw; i += blockDim.x) {
      const int n = i / kFusedLdw, k = i - n * kFusedLdw;
      wt[i] = __float2bfloat16_rn((n < d_out && k < dim) ? mw[(int64_t)k * d_out + n] : 0.f);
    }
    __syncthreads();
  }
  if (a >= b) return;

  const uint32_t stage0 = smem_u32(wsmem + warp * kWarpSmemPerWarp);
  const uint32_t slab = stage0 + kWarpTileStages * kWarpStageBytes;
  const uint64_t keep = policy_evict_last();
#if HCS_PLAN_PF_ENTL > 0
  const int64_t ent_end = SWV == 8 ? __ldg(ent_ptr + chunk_ptr[T]) : 0;  // entries of this launch end here
#endif
  // plan data (indices, entries) is read once per feature slice: keep it for the window's
  // other slice-warps (FS > 1), stream it otherwise
  // (paired slice-warps read each chunk's plan together: stream it)
  const uint64_t once = (FS > 1 && !paired) ? policy_evict_normal() : policy_evict_first();
  // gather lane mapping: lane (rg, v) copies 16-B vector v of rows rg*NI + it, it < NI, so its
  // NI gather indices are contiguous (NI/4 x 128-bit loads)
  const int gv = lane % SWV, rg = lane / SWV;
  uint32_t dofs[NI];  // smem destination of each of the lane's copies (constant per lane)
#pragma unroll
  for (int it = 0; it < NI; ++it) dofs[it] = C::off(rg * NI + it, gv);
  const int featv = gv * 8;  // feature offset of the lane's vector inside a slice
  const uint32_t vb_full = 16u;
  const char* xb = reinterpret_cast<const char*>(x);
  const uint32_t ldxb = (uint32_t)(ldx * 2);
  // ldmatrix lane mapping (A: slab rows, B: gathered rows k, 8-feature chunks)
  const int ar = lane & 15, akc = lane >> 4;
  const int bk = (lane & 7) + ((lane >> 3) & 1) * 8, bfc = lane >> 4;

  struct Pos {
    int64_t base;   // chunk_ptr[t]
    int32_t t, f, j, nj, rem;  // rem = b - flattened index (valid while > 0)
  };
  auto mk = [&](const ChunkPos& c) {
    Pos p;
    p.base = c.base;
    p.t = (int32_t)c.t;
    p.f = c.f;
    p.j = c.j;
    p.nj = c.nj;
    p.rem = (int32_t)(b - c.fi);
    return p;
  };
  auto adv = [&](Pos& p) {
    --p.rem;
    if (++p.j < p.nj) return;
    p.j = 0;
    if (++p.f < FSr) return;
    p.f = 0;
    ++p.t;
    p.base += p.nj;
    p.nj = (p.t < T && p.rem > 0) ? (int32_t)(ldg64(chunk_ptr + p.t + 1) - p.base) : 1;
  };
  auto load_gidx = [&](const Pos& p, int (&g)[NI]) {
    if (p.rem > 0) {
      const int4* gp = reinterpret_cast<const int4*>(gidx + (p.base + p.j) * 64 + rg * NI);
#pragma unroll
      for (int q = 0; q < NI / 4; ++q) {
        int4 v;
        asm volatile("ld.global.nc.L2::cache_hint.v4.s32 {%0,%1,%2,%3}, [%4], %5;"
                     : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                     : "l"(gp + q), "l"(once));
        g[4 * q] = v.x;
        g[4 * q + 1] = v.y;
        g[4 * q + 2] = v.z;
        g[4 * q + 3] = v.w;
      }
    }
  };
  auto issue = [&](const Pos& p, const int (&g)[NI], int slot) {
    if (p.rem > 0 && (NPR == SWV / 2 || gv < 2 * NPR)) {
      const int feat = (p.f + fw) * C::kFeat + featv;
      // X rows are padded with zeros to whole slices (executors.stage_operand), so every lane of
      // a slice inside the row copies 16 B: zero-fill lanes (src-size 0) mixed into a cp.async
      // instruction cost more than the bytes they save (N = 24: 1.13 vs 0.79 ms at N = 32)
      const uint32_t vb = feat < ldx ? vb_full : 0u;
      const char* src = xb + (int64_t)feat * 2;
      const uint32_t dst = stage0 + slot * kWarpStageBytes;
      if (p.j + 1 < p.nj) {  // full chunk: every slot holds a column
#pragma unroll
        for (int it = 0; it < NI; ++it) cp_async16(dst + dofs[it], src + (uint64_t)(uint32_t)g[it] * ldxb, vb, keep);
      } else {  // the window's last chunk: pad slots (-1) are zero-filled
#pragma unroll
        for (int it = 0; it < NI; ++it) {
          const int gi = g[it];
          cp_async16(dst + dofs[it], src + (uint64_t)(uint32_t)max(gi, 0) * ldxb, gi >= 0 ? vb : 0u, keep);
        }
      }
    }
    cp_async_commit();
  };
  auto load_ep = [&](const Pos& p, int64_t& e0, int64_t& e1) {
    if (p.rem > 0) {
      const int64_t c = p.base + p.j;
      e0 = ld_plan_s64(ent_ptr + c, once);
      e1 = ld_plan_s64(ent_ptr + c + 1, once);
    } else {
      e0 = e1 = 0;
    }
  };
  auto load_ent = [&](int64_t e0, int64_t e1, uint32_t (&e)[kWarpEntRegs]) {
#pragma unroll
    for (int q = 0; q < kWarpEntRegs; ++q) {
      const int64_t i = e0 + lane + 32 * q;
      e[q] = i < e1 ? ld_plan_u32(ent + i, once) : 0u;
    }
    // a dense chunk's remaining entries: pull them into L2 one chunk ahead (lane = 128-B line)
    const int64_t ov = e0 + 32 * kWarpEntRegs + 32 * lane;
    if (ov < e1) asm volatile("prefetch.global.L2::evict_last [%0];" ::"l"(ent + ov));
#if HCS_PLAN_PF_ENTL > 0
    // the entries of the following chunks are contiguous after e1: pull their lines into L2
    // a step before their loads
    {
      const int64_t pv = (e1 & ~(int64_t)31) + 32 * lane;
      if (SWV == 8 && lane < HCS_PLAN_PF_ENTL && pv < ent_end) asm volatile("prefetch.global.L2 [%0];" ::"l"(ent + pv));
    }
#endif
  };

  float acc[SWV][4];
#pragma unroll
  for (int i = 0; i < SWV; ++i) acc[i][0] = acc[i][1] = acc[i][2] = acc[i][3] = 0.f;
  float oacc[FUSED ? kFusedOutMax / 8 : 1][4];
#pragma unroll
  for (int i = 0; i < (FUSED ? kFusedOutMax / 8 : 1); ++i) oacc[i][0] = oacc[i][1] = oacc[i][2] = oacc[i][3] = 0.f;
  bool in_head;  // our first unit (t, f) began in an earlier warp's range
  int s0 = 0;    // ring slot of the chunk being computed

  // one pipeline step: compute P0 while P1, P2 are in flight; gathers of P2, indices of P3,
  // entries of P1, entry pointers of P2.  Register sets rotate by renaming (loop unrolled 4x),
  // so no in-flight load result is copied before it is needed.
  auto step = [&](Pos& P0, const Pos& P1, const Pos& P2, const Pos& P3, int (&Gcur)[NI], int (&Gnext)[NI],
                  uint32_t (&Ecur)[kWarpEntRegs], uint32_t (&Enext)[kWarpEntRegs], const int64_t (&EP0)[2],
                  const int64_t (&EP1)[2], int64_t (&EP2)[2]) -> bool {
    if (P0.rem <= 0) return true;
    const int s2 = s0 >= 1 ? s0 - 1 : s0 + 2;
    issue(P2, Gcur, s2);
    load_gidx(P3, Gnext);
    load_ent(EP1[0], EP1[1], Enext);
    load_ep(P2, EP2[0], EP2[1]);
    // slab of P0 (zero on entry: cleared after the previous chunk's MMAs): scatter the packed
    // entries (bf16 value << 16 | swizzled byte offset)
    const int ne = (int)(EP0[1] - EP0[0]);
    {
#pragma unroll
      for (int q = 0; q < kWarpEntRegs; ++q)
        if (lane + 32 * q < ne) sts16(slab + (Ecur[q] & 0x7FFu), Ecur[q] >> 16);
      // dense chunks (> 128 entries; e.g. windows after LOA): the remaining entries in
      // batches of 8 loads per lane, so one memory latency covers 256 entries
      for (int i0 = 32 * kWarpEntRegs; i0 < ne; i0 += 32 * 8) {
        uint32_t w[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const int i = i0 + 32 * u + lane;
          w[u] = i < ne ? ld_plan_u32(ent + EP0[0] + i, once) : 0u;
        }
#pragma unroll
        for (int u = 0; u < 8; ++u)
          if (i0 + 32 * u + lane < ne) sts16(slab + (w[u] & 0x7FFu), w[u] >> 16);
      }
    }
    cp_async_wait<2>();  // P0's gathers landed (P1, P2 may still be in flight)
    __syncwarp();
    {
      const uint32_t st = stage0 + s0 * kWarpStageBytes;
#pragma unroll
      for (int ks = 0; ks < 4; ++ks) {
        uint32_t af[4];
        const int kc = 2 * ks + akc;
        ldsm_x4(af, slab + ar * 128 + (((kc ^ ar) & 7) << 4));
        const int k = ks * 16 + bk;
#pragma unroll
        for (int pr = 0; pr < NPR; ++pr) {
          uint32_t bb[4];
          ldsm_x4_trans(bb, st + C::off(k, 2 * pr + bfc));
          hmma_16816(acc[2 * pr], af, bb[0], bb[1]);
          hmma_16816(acc[2 * pr + 1], af, bb[2], bb[3]);
        }
      }
    }
    __syncwarp();
    // clear the slab for the next chunk: undo this chunk's scatter (all entries in registers),
    // or zero it fully when the chunk overflowed the register-held entries
    if (ne <= 32 * kWarpEntRegs) {
#pragma unroll
      for (int q = 0; q < kWarpEntRegs; ++q)
        if (lane + 32 * q < ne) sts16(slab + (Ecur[q] & 0x7FFu), 0u);
    } else {
#pragma unroll
      for (int q = 0; q < 4; ++q) sts128_zero(slab + (lane + 32 * q) * 16);
    }
#ifndef HCS_EXP_NO_UNDO_SYNC
    __syncwarp();  // the next chunk's scatter may hit a slot another lane clears here (racecheck)
#endif
    // end of our part of the unit: Z (whole unit) or a scratch slot (split unit; the last of
    // its warps to arrive sums the slots in range order, below)
    const bool unit_done = P0.j + 1 == P0.nj;
    if (unit_done || P0.rem == 1) {
      const int64_t rs = (int64_t)__ldg(tile_list + P0.t) * wh;
      const int rows = (int)(n_rows - rs < wh ? n_rows - rs : wh);
      bool zsplit = false;
      if (z != nullptr) {
        if (!in_head && unit_done) {
          store_slice<SWV>(z, ldz, rs, rows, dim, P0.f + fw, acc, lane);
        } else {
          write_slot<SWV>(scratch + (gw * 2 + (in_head ? 0 : 1)) * C::kSlot, acc, lane);
          zsplit = true;  // finished after the fused epilogue has used acc
        }
      }
      in_head = false;
      if (FUSED) {
        // oacc += Z_slice (16 x 8*SWV, bf16 RNE) . M[slice rows, :]; the B fragments of two n8 tiles
        // (W^T rows n, k-halves lo / hi) per ldmatrix.x4 -- lane l addresses row l & 7 of matrix l >> 3
        // = (n8 pair half (l >> 4), k half ((l >> 3) & 1)); the 272-B row pitch is conflict-free
        const uint32_t wt_s = smem_u32(wsmem + C::kOffW);
        const int wrow_n = (lane & 7) + ((lane >> 4) << 3), wrow_k = ((lane >> 3) & 1) * 8;
#pragma unroll
        for (int j = 0; j < NPR; ++j) {
          uint32_t af[4];
          af[0] = pack_bf16(acc[2 * j][0], acc[2 * j][1]);
          af[1] = pack_bf16(acc[2 * j][2], acc[2 * j][3]);
          af[2] = pack_bf16(acc[2 * j + 1][0], acc[2 * j + 1][1]);
          af[3] = pack_bf16(acc[2 * j + 1][2], acc[2 * j + 1][3]);
          const int kb = (P0.f + fw) * C::kFeat + 16 * j;
#pragma unroll
          for (int n16 = 0; n16 < kFusedOutMax / 16; ++n16) {
            if (n16 * 16 < d_out) {
              uint32_t wb[4];
              ldsm_x4(wb, wt_s + (uint32_t)(((n16 * 16 + wrow_n) * kFusedLdw + kb + wrow_k) * 2));
              hmma_16816(oacc[2 * n16], af, wb[0], wb[1]);
              if (n16 * 16 + 8 < d_out) hmma_16816(oacc[2 * n16 + 1], af, wb[2], wb[3]);
            }
          }
        }
        const bool win_head = (int64_t)FSr * (P0.base - c0) < a;  // window began in an earlier range
        const bool win_done = unit_done && P0.f == FSr - 1;
        if (win_done || P0.rem == 1) {
          if (paired) {
            // the pair's slice partials: warp f = 1 hands its 16 x 64 out partial to warp f = 0
            // through its own ring slot of the chunk just computed (free until the next step's
            // issue), then out = partial(slice 0) + partial(slice 1)
            const uint32_t xs = smem_u32(wsmem + (warp | 1) * kWarpSmemPerWarp) + s0 * kWarpStageBytes;
            const int bar = 1 + (warp >> 1);
            if (fw == 1) {
#pragma unroll
              for (int n8 = 0; n8 < kFusedOutMax / 8; ++n8)
                sts128f(xs + (n8 * 32 + lane) * 16, oacc[n8][0], oacc[n8][1], oacc[n8][2], oacc[n8][3]);
            }
            named_bar_sync(bar, 64);
            if (fw == 0) {
#pragma unroll
              for (int n8 = 0; n8 < kFusedOutMax / 8; ++n8) {
                const float4 v = lds128f(xs + (n8 * 32 + lane) * 16);
                oacc[n8][0] += v.x;
                oacc[n8][1] += v.y;
                oacc[n8][2] += v.z;
                oacc[n8][3] += v.w;
              }
            }
            named_bar_sync(bar, 64);
          }
          if (fw == 0) {
            if (win_done && !win_head) {
              store_out(out, ldo, rs, rows, d_out, oacc, lane);
            } else {
              const int64_t gi = paired ? gw / FS : gw;
              write_slot(oscratch + (gi * 2 + (win_head ? 0 : 1)) * kOutSlot, oacc, lane);
              finish_split_out(chunk_ptr, T, FS, paired, kWarpTileWarps, cnt, oscratch, out, ldo, P0.base, P0.nj,
                               rs, rows, d_out, wb);
            }
          }
#pragma unroll
          for (int i = 0; i < kFusedOutMax / 8; ++i) oacc[i][0] = oacc[i][1] = oacc[i][2] = oacc[i][3] = 0.f;
        }
      }
      if (zsplit)
        finish_split_z<SWV, C::kSlot>(chunk_ptr, T, FS, paired, kWarpTileWarps, cnt, scratch, z, ldz, P0.base, P0.f,
                                      P0.nj, rs, rows, dim, wb);
#pragma unroll
      for (int i = 0; i < SWV; ++i) acc[i][0] = acc[i][1] = acc[i][2] = acc[i][3] = 0.f;
    }
    s0 = s0 == kWarpTileStages - 1 ? 0 : s0 + 1;
    P0 = P3;  // P0's variable becomes position +4
    adv(P0);
    return false;
  };

  // prologue: the slab starts zeroed and is kept zero between chunks
#pragma unroll
  for (int q = 0; q < 4; ++q) sts128_zero(slab + (lane + 32 * q) * 16);
  __syncwarp();
  const ChunkPos first = locate(chunk_ptr, T, FSr, a);
  in_head = first.j != 0;
  Pos Q0 = mk(first), Q1 = Q0;
  adv(Q1);
  Pos Q2 = Q1;
  adv(Q2);
  Pos Q3 = Q2;
  adv(Q3);
  int G0[NI], G1[NI];
  load_gidx(Q0, G0);
  load_gidx(Q1, G1);
  issue(Q0, G0, 0);
  issue(Q1, G1, 1);
  load_gidx(Q2, G0);
  int64_t EPa[2], EPb[2], EPc[2], EPd[2];
  load_ep(Q0, EPa[0], EPa[1]);
  load_ep(Q1, EPb[0], EPb[1]);
  uint32_t E0[kWarpEntRegs], E1[kWarpEntRegs];
  load_ent(EPa[0], EPa[1], E0);
  for (;;) {
    if (step(Q0, Q1, Q2, Q3, G0, G1, E0, E1, EPa, EPb, EPc)) break;
    if (step(Q1, Q2, Q3, Q0, G1, G0, E1, E0, EPb, EPc, EPd)) break;
    if (step(Q2, Q3, Q0, Q1, G0, G1, E0, E1, EPc, EPd, EPa)) break;
    if (step(Q3, Q0, Q1, Q2, G1, G0, E1, E0, EPd, EPa, EPb)) break;
  }
  cp_async_wait<0>();
}

// ---------------------------------------------------------------- tf32 variant
// Same schedule and fix-up; fp32 X rows (32-feature slices of 128 B), 16 x 64 fp32 slab,
// mma.sync m16n8k8 tf32 (X and values RNA-rounded to tf32 by the caller / plan).
// B fragments: n8 tile nt's column g is feature 4g + nt, so a lane's words for all four tiles
// are one conflict-free 128-bit load per k row (16-B chunk XOR 2*(row&3)); Z is stored unpermuted.
constexpr int kTfWarps = 8;
constexpr int kTfRow = 128;
constexpr int kTfStage = 64 * kTfRow;
constexpr int kTfSlab = 16 * 64 * 4;
constexpr int kTfPerWarp = kWarpTileStages * kTfStage + kTfSlab;
constexpr int kTfSmem = kTfWarps * kTfPerWarp + 128;
static_assert(kTfSmem <= 227 * 1024, "smem");
__device__ __forceinline__ int swz_tf(int k, int v) { return v ^ ((2 * k) & 6); }

// FUSED (K6/K7 in tf32): after each (window, 32-feature slice) unit the warp multiplies its 16 x 32
// aggregated slice (tf32 A fragments taken from the accumulators, features permuted within each
// 8-block so no shuffle is needed) by the slice's 32 x d_out block of M (tf32-rounded, read from
// global / L1: the kernel's shared memory is full) into an out accumulator; window partials cut by
// a warp boundary go to oscratch and are summed in warp order by the last of its warps.
template <bool FUSED>
__global__ void __launch_bounds__(kTfWarps * 32, 1)
    k_tile_warp_tf32(const int32_t* __restrict__ tile_list, int64_t T, const int64_t* __restrict__ chunk_ptr,
                     const int32_t* __restrict__ gidx, const int64_t* __restrict__ ent_ptr,
                     const uint2* __restrict__ ent, int64_t n_rows, int wh, const float* __restrict__ x, int64_t ldx,
                     int dim, int FS, float* __restrict__ z, int64_t ldz, float* __restrict__ scratch,
                     const float* __restrict__ mw, int d_out, float* __restrict__ out, int64_t ldo,
                     float* __restrict__ oscratch, unsigned* __restrict__ cnt, int paired) {
  constexpr int NI = 16;
  extern __shared__ uint8_t tsmem_raw[];
  uint8_t* tsmem = (uint8_t*)(((uintptr_t)tsmem_raw + 127) & ~(uintptr_t)127);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t nwarps = (int64_t)gridDim.x * kTfWarps;
  const int64_t gw = (int64_t)blockIdx.x * kTfWarps + warp;
  const int64_t c0 = chunk_ptr[0];
  // paired slices (plain SpMM, FS dividing the CTA's warps): the FS warps of a group walk one
  // balanced range of chunks, one 32-feature slice each, so each chunk's plan is read once
  const int FSr = paired ? 1 : FS;
  const int fw = paired ? (int)(gw % FS) : 0;
  const int64_t ngroups = paired ? nwarps / FS : nwarps;
  const int64_t total = (int64_t)FSr * (chunk_ptr[T] - c0);
  int64_t a = 0, b = 0;
  if (!paired || gw < ngroups * FS) warp_range(total, ngroups, paired ? gw / FS : gw, a, b);
  if (a >= b) return;
  const uint32_t stage0 = smem_u32(tsmem + warp * kTfPerWarp);
  const uint32_t slab = stage0 + kWarpTileStages * kTfStage;
  uint8_t* slab_p = tsmem + warp * kTfPerWarp + kWarpTileStages * kTfStage;
  const uint64_t keep = policy_evict_last();
  const uint64_t once = policy_evict_first();
  const char* xb = reinterpret_cast<const char*>(x);
  const int64_t ldxb = ldx * 4;
  // gather lane mapping: lane (grow, gv) copies 16-B vector gv of rows grow*16 + it, so its 16
  // gather indices are contiguous (4 x 128-bit loads); 8 lanes fill one 128-B row per copy
  const int grow = lane >> 3, gv = lane & 7;
  const int g8 = lane >> 2, t4 = lane & 3;
  const int arow = (lane & 7) + ((lane >> 3) & 1) * 8, ach = lane >> 4;

  ChunkPos p0 = locate(chunk_ptr, T, FSr, a);
  ChunkPos p1 = p0, p2, p3;
  advance(p1, chunk_ptr, T, FSr);
  p2 = p1;
  advance(p2, chunk_ptr, T, FSr);
  p3 = p2;
  advance(p3, chunk_ptr, T, FSr);
  bool in_head = p0.j != 0;

  auto load_gidx = [&](const ChunkPos& p, int (&g)[NI]) {
    if (p.fi < b) {
      const int4* gp = reinterpret_cast<const int4*>(gidx + (p.base + p.j) * 64 + grow * NI);
#pragma unroll
      for (int q = 0; q < NI / 4; ++q) {
        int4 v;
        asm volatile("ld.global.nc.L2::cache_hint.v4.s32 {%0,%1,%2,%3}, [%4], %5;"
                     : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                     : "l"(gp + q), "l"(once));
        g[4 * q] = v.x;
        g[4 * q + 1] = v.y;
        g[4 * q + 2] = v.z;
        g[4 * q + 3] = v.w;
      }
    }
  };
  auto issue = [&](const ChunkPos& p, const int (&g)[NI], int slot) {
    if (p.fi < b) {
      const int feat = (p.f + fw) * 32 + gv * 4;
      const uint32_t vb = feat < ldx ? 16u : 0u;  // zero padding read as data (see k_tile_warp)
      const char* src = xb + (int64_t)feat * 4;
      const uint32_t dst = stage0 + slot * kTfStage;
#pragma unroll
      for (int it = 0; it < NI; ++it) {
        const int row = grow * NI + it;
        const int gi = g[it];
        cp_async16(dst + row * kTfRow + (swz_tf(row, gv) << 4), src + (int64_t)max(gi, 0) * ldxb, gi >= 0 ? vb : 0u,
                   keep);
      }
    }
    cp_async_commit();
  };
  auto load_ep = [&](const ChunkPos& p, int64_t& e0, int64_t& e1) {
    if (p.fi < b) {
      const int64_t c = p.base + p.j;
      e0 = ld_plan_s64(ent_ptr + c, once);
      e1 = ld_plan_s64(ent_ptr + c + 1, once);
    } else {
      e0 = e1 = 0;
    }
  };
  auto load_ent = [&](int64_t e0, int64_t e1, uint2 (&e)[kWarpEntRegs]) {
#pragma unroll
    for (int q = 0; q < kWarpEntRegs; ++q) {
      const int64_t i = e0 + lane + 32 * q;
      e[q] = i < e1 ? __ldg(ent + i) : make_uint2(0u, 0u);
    }
  };

  int g_a[NI], g_b[NI], g2[NI];
  load_gidx(p0, g_a);
  load_gidx(p1, g_b);
  issue(p0, g_a, 0);
  issue(p1, g_b, 1);
  load_gidx(p2, g2);
  int64_t ep0a, ep0b, ep1a, ep1b;
  load_ep(p0, ep0a, ep0b);
  load_ep(p1, ep1a, ep1b);
  uint2 e0r[kWarpEntRegs], e1r[kWarpEntRegs];
  load_ent(ep0a, ep0b, e0r);
  float acc[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i) acc[i][0] = acc[i][1] = acc[i][2] = acc[i][3] = 0.f;
  constexpr int NO = FUSED ? kFusedOutMax / 8 : 1;
  float oacc[NO][4];
#pragma unroll
  for (int i = 0; i < NO; ++i) oacc[i][0] = oacc[i][1] = oacc[i][2] = oacc[i][3] = 0.f;
  int s0 = 0;
  {  // the slab starts zeroed and is kept zero between chunks (entries are undone after use)
    const int4 zero4 = make_int4(0, 0, 0, 0);
#pragma unroll
    for (int q = 0; q < 8; ++q) reinterpret_cast<int4*>(slab_p)[lane + 32 * q] = zero4;
    __syncwarp();
  }
  for (; p0.fi < b;) {
    const int s2 = s0 >= 1 ? s0 - 1 : s0 + 2;
    issue(p2, g2, s2);
    load_gidx(p3, g2);
    load_ent(ep1a, ep1b, e1r);
    int64_t ep2a, ep2b;
    load_ep(p2, ep2a, ep2b);
    const int ne = (int)(ep0b - ep0a);
    {
#pragma unroll
      for (int q = 0; q < kWarpEntRegs; ++q)
        if (lane + 32 * q < ne) *reinterpret_cast<uint32_t*>(slab_p + e0r[q].x) = e0r[q].y;
      for (int i = 32 * kWarpEntRegs + lane; i < ne; i += 32) {
        const uint2 w = __ldg(ent + ep0a + i);
        *reinterpret_cast<uint32_t*>(slab_p + w.x) = w.y;
      }
    }
    cp_async_wait<2>();
    __syncwarp();
    {
      const uint32_t st = stage0 + s0 * kTfStage;
#pragma unroll
      for (int ks = 0; ks < 8; ++ks) {
        uint32_t af[4];
        const int ch = 2 * ks + ach;
        ldsm_x4(af, slab + arow * 256 + ((((ch & 8) | ((ch ^ arow) & 7))) << 4));
        // n8 tile nt, column g <-> feature 4g + nt: a lane's B words of all four tiles are one
        // 16-B vector per k row (2 x LDS.128 per k step instead of 8 x LDS.32)
        const int k0 = ks * 8 + t4, k1 = k0 + 4;
        const uint4 v0 = lds128(st + k0 * kTfRow + (swz_tf(k0, g8) << 4));
        const uint4 v1 = lds128(st + k1 * kTfRow + (swz_tf(k1, g8) << 4));
        mma_tf32_1688(acc[0], af, v0.x, v1.x);
        mma_tf32_1688(acc[1], af, v0.y, v1.y);
        mma_tf32_1688(acc[2], af, v0.z, v1.z);
        mma_tf32_1688(acc[3], af, v0.w, v1.w);
      }
    }
    __syncwarp();
    if (ne <= 32 * kWarpEntRegs) {  // undo this chunk's scatter
#pragma unroll
      for (int q = 0; q < kWarpEntRegs; ++q)
        if (lane + 32 * q < ne) *reinterpret_cast<uint32_t*>(slab_p + e0r[q].x) = 0u;
    } else {
      const int4 zero4 = make_int4(0, 0, 0, 0);
#pragma unroll
      for (int q = 0; q < 8; ++q) reinterpret_cast<int4*>(slab_p)[lane + 32 * q] = zero4;
    }
    __syncwarp();
    const bool unit_done = p0.j + 1 == p0.nj;
    if (unit_done || p0.fi + 1 == b) {
      const int64_t rs = (int64_t)__ldg(tile_list + p0.t) * wh;
      const int rows = (int)(n_rows - rs < wh ? n_rows - rs : wh);
      bool zsplit = false;
      if (z != nullptr) {
        if (!in_head && unit_done) {
          store_slice_tf32p(z, ldz, rs, rows, dim, p0.f + fw, acc, lane);
        } else {
          write_slot<4>(scratch + (gw * 2 + (in_head ? 0 : 1)) * WarpCfg<4>::kSlot, acc, lane);
          zsplit = true;
        }
      }
      in_head = false;
      if (FUSED) {
        // oacc += Z_slice (16 x 32) . M[32 f .. 32 f + 31, :]; MMA step nt takes the accumulators of
        // n8 tile nt as its A fragment: k index t <-> feature 8t + nt, t + 4 <-> 8t + 4 + nt (the
        // permuted accumulator layout), on both operands
#pragma unroll
        for (int nt = 0; nt < 4; ++nt) {
          uint32_t af[4];
          asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(af[0]) : "f"(acc[nt][0]));
          asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(af[1]) : "f"(acc[nt][2]));
          asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(af[2]) : "f"(acc[nt][1]));
          asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(af[3]) : "f"(acc[nt][3]));
          const int k0 = p0.f * 32 + 8 * t4 + nt, k1 = k0 + 4;
#pragma unroll
          for (int n8 = 0; n8 < NO; ++n8) {
            if (n8 * 8 < d_out) {
              const int col = n8 * 8 + g8;
              const uint32_t b0 = (k0 < dim && col < d_out) ? __float_as_uint(__ldg(mw + (int64_t)k0 * d_out + col)) : 0u;
              const uint32_t b1 =
                  (k1 < dim && col < d_out) ? __float_as_uint(__ldg(mw + (int64_t)k1 * d_out + col)) : 0u;
              mma_tf32_1688(oacc[n8], af, b0, b1);
            }
          }
        }
        const bool win_head = (int64_t)FS * (p0.base - c0) < a;  // window began in an earlier warp's range
        const bool win_done = unit_done && p0.f == FS - 1;
        if (win_done || p0.fi + 1 == b) {
          if (win_done && !win_head) {
            store_out(out, ldo, rs, rows, d_out, oacc, lane);
          } else {
            write_slot<NO>(oscratch + (gw * 2 + (win_head ? 0 : 1)) * kOutSlot, oacc, lane);
            finish_split_out(chunk_ptr, T, FS, 0, kTfWarps, cnt, oscratch, out, ldo, p0.base, p0.nj, rs, rows, d_out);
          }
#pragma unroll
          for (int i = 0; i < NO; ++i) oacc[i][0] = oacc[i][1] = oacc[i][2] = oacc[i][3] = 0.f;
        }
      }
      if (zsplit)
        finish_split_z<4, WarpCfg<4>::kSlot, true>(chunk_ptr, T, FS, paired, kTfWarps, cnt, scratch, z, ldz, p0.base,
                                             p0.f, p0.nj, rs, rows, dim);
#pragma unroll
      for (int i = 0; i < 4; ++i) acc[i][0] = acc[i][1] = acc[i][2] = acc[i][3] = 0.f;
    }
    p0 = p1;
    p1 = p2;
    p2 = p3;
    advance(p3, chunk_ptr, T, FSr);
#pragma unroll
    for (int q = 0; q < kWarpEntRegs; ++q) e0r[q] = e1r[q];
    ep0a = ep1a;
    ep0b = ep1b;
    ep1a = ep2a;
    ep1b = ep2b;
    s0 = s0 == kWarpTileStages - 1 ? 0 : s0 + 1;
  }
  cp_async_wait<0>();
}

// paired 32-feature slices for the tf32 SpMM (1 default; hcs_set_tile_pairing(0) turns it off too)
static int g_warp_paired_tf32 = 1;

// CTAs of a tile launch: one per SM (default), or fewer when SMs are left to concurrent NCCL
// kernels (the multi-GPU exchange of the previous part runs beside the next part's tiles only if
// some SMs are free: a tile CTA holds 213 KB of shared memory and 57 K registers of its SM)
static int g_tile_grid = 0;
// CTAs of a tile launch: one per SM (or the hcs_set_tile_grid cap), fewer when the caller passes
// the launch's chunk count (positions > 0): ceil(positions / warp groups per CTA), so every group
// keeps >= 1 position while a small plan no longer fills every SM's shared memory with CTAs that
// exit at once -- the piece kernel forked beside it then starts on free SMs (C1 product
// 10.25 -> 8.22 us, tools/exp_c1.py; a 1-window plan launches 1 CTA)
static int tile_grid(int64_t positions = 0, int groups_per_cta = 1) {
  int g = g_tile_grid > 0 ? std::min(g_tile_grid, num_sms()) : num_sms();
  if (positions > 0)
    g = (int)std::max<int64_t>(1, std::min<int64_t>(g, (positions + groups_per_cta - 1) / groups_per_cta));
  return g;
}

// tf32 SpMM (m == nullptr) or fused GCN layer (m = tf32-rounded M [dim x d_out], d_out <= 64; z may
// be nullptr when no z_cache is wanted).
int spmm_tile_warp_tf32(const int32_t* tile_list, int64_t n_tile, const int64_t* chunk_ptr, const int32_t* gidx,
                        const int64_t* ent_ptr, const uint2* ent, int64_t n_rows, int wh, const float* x, int64_t ldx,
                        int dim, float* z, int64_t ldz, float* scratch, int64_t scratch_floats, cudaStream_t st,
                        const float* m = nullptr, int d_out = 0, float* out = nullptr, int64_t ldo = 0,
                        int64_t n_chunks = 0) {
  const int FS = (dim + 31) / 32;
  const bool fused = m != nullptr;
  const int paired = (!fused && FS > 1 && kTfWarps % FS == 0 && g_warp_paired_tf32) ? 1 : 0;
  const int grid = tile_grid((paired ? 1 : FS) * n_chunks, paired ? kTfWarps / FS : kTfWarps);
  const int64_t nwarps = (int64_t)grid * kTfWarps;
  const int64_t cw = 2 * tile_cnt_words();
  const int64_t need = cw + nwarps * 2 * (WarpCfg<4>::kSlot + (fused ? kOutSlot : 0));
  HCS_REQUIRE(scratch != nullptr && scratch_floats >= need, HCS_EINVAL, "tile scratch too small");
  unsigned* cnt = reinterpret_cast<unsigned*>(scratch);
  float* slots = scratch + cw;
  float* oscratch = slots + nwarps * 2 * WarpCfg<4>::kSlot;
  auto kern = fused ? k_tile_warp_tf32<true> : k_tile_warp_tf32<false>;
  HCS_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, kTfSmem));
  kern<<<grid, kTfWarps * 32, kTfSmem, st>>>(tile_list, n_tile, chunk_ptr, gidx, ent_ptr, ent, n_rows, wh, x, ldx, dim,
                                             FS, z, ldz, slots, m, d_out, out, ldo, oscratch, cnt, paired);
  HCS_LAUNCH_CHECK("k_tile_warp_tf32");
  return HCS_OK;
}

// Cost-weighted warp ranges.  The uniform split gives every warp (group) the same number of
// 64-column chunks, but a chunk costs a 64-row gather plus its entries' scatter, and the hub
// windows of a skewed graph (R-MAT C5: the first windows) hold chunks of up to ~900 entries, so
// the first ranges carry 1.8x the mean entries (tools/exp_tile_balance.py) and the launch waits
// for them.  k_tile_bounds splits the positions on the prefix cost alpha * chunks + entries
// (ent_ptr is already the entries' prefix sum) with one 32-way warp search per boundary; the tile
// kernel reads its range from the bounds and locates split-unit owners by binary search.
// alpha comes with the launch (hcs_spmm_tile_balanced; 0 = uniform).  Used when one position is one chunk (paired slices or a
// single slice) and the launch has >= kBalanceMinTilesPerGroup windows per group (host-known, so
// small plans keep one launch and no sync is needed).
constexpr int64_t kBalanceMinTilesPerGroup = 8;

__global__ void k_tile_bounds(const int64_t* __restrict__ chunk_ptr, int64_t T, const int64_t* __restrict__ ent_ptr,
                              int64_t ng, int64_t alpha, int64_t* __restrict__ wb) {
  // one warp per boundary g: wb[g] = smallest p with (alpha p + entries before p) * ng >= g * F,
  // found by a 32-way search (one round of 32 parallel ent_ptr loads per step, ~5 steps)
  const int lane = threadIdx.x & 31;
  const int64_t g = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (g > ng) return;
  const int64_t c0 = __ldg(chunk_ptr), total = __ldg(chunk_ptr + T) - c0;
  if (g == 0 || g == ng) {
    if (lane == 0) wb[g] = g == 0 ? 0 : total;
    return;
  }
  const int64_t e0 = __ldg(ent_ptr + c0);
  const int64_t F = alpha * total + (__ldg(ent_ptr + c0 + total) - e0);
  const int64_t target = g * F;
  auto pred = [&](int64_t p) { return (alpha * p + (__ldg(ent_ptr + c0 + p) - e0)) * ng >= target; };
  int64_t lo = 0, hi = total;  // answer in [lo, hi]; pred(total) holds
  while (hi - lo >= 32) {
    const int64_t step = (hi - lo + 31) / 32;
    const int64_t p = min(lo + lane * step, hi);
    const unsigned m = __ballot_sync(0xffffffffu, pred(p));
    if (m & 1u) {
      hi = lo;
      break;
    }
    const int j = m ? __ffs(m) - 1 : 32;  // answer in (p_{j-1}, p_j]
    const int64_t nlo = min(lo + (int64_t)(j - 1) * step, hi) + 1;
    hi = j < 32 ? min(lo + (int64_t)j * step, hi) : hi;
    lo = nlo;
  }
  const int64_t p = lo + lane;
  const unsigned m = __ballot_sync(0xffffffffu, p <= hi && pred(p));
  if (lane == 0) wb[g] = m ? lo + __ffs(m) - 1 : hi;
}

// int64 bounds of the weighted split, after the largest slot region of the workspace
inline int64_t tile_bounds_offset_floats() {
  static_assert(WarpCfg<4>::kWarps <= kMaxWarpsPerCta && WarpCfg<8>::kWarps <= kMaxWarpsPerCta &&
                    kTfWarps <= kMaxWarpsPerCta, "split counters");
  return 2 * tile_cnt_words() + std::max<int64_t>(
      std::max<int64_t>((int64_t)num_sms() * WarpCfg<4>::kWarps * 2 * WarpCfg<4>::kSlot,
                        (int64_t)num_sms() * WarpCfg<8>::kWarps * 2 * (WarpCfg<8>::kSlot + kOutSlot)),
      (int64_t)num_sms() * WarpCfg<16>::kWarps * 2 * WarpCfg<16>::kSlot);
}

static int g_warp_swv = 0;     // 0 auto, 4 or 8 (16-B vectors per row slice)
// Feature slices of a window walked side by side by sibling warps: 1 on (default), 0 off,
// 2 auto = on when X does not fit in L2.  Paired warps read each chunk's plan together (the
// second read hits L1), so the plan streams with evict_first and X stays L2-resident:
// C2/N=128 DRAM reads 3.25 -> 1.16 GB per launch, L2 hit 82.7 -> 93.5 %, same time (2.46 ms);
// C5 tile windows 29.9 -> 27.7 ms (tools/exp_pairing.py, exp_pair_ncu.py, exp_c5.py).
static int g_warp_paired = 1;
// 33..48-feature single slice: 1 = skip the empty 16-feature group at compile time (NPR = 3)
static int g_warp_npr3 = 1;
constexpr int64_t kPairMinXBytes = 96ll << 20;

template <int SWV, bool FUSED = false>
static int launch_warp(const int32_t* tile_list, int64_t n_tile, const int64_t* chunk_ptr, const int32_t* gidx,
                       const int64_t* ent_ptr, const uint32_t* ent, int64_t n_rows, int wh, const __nv_bfloat16* x,
                       int64_t ldx, int dim, float* z, int64_t ldz, float* scratch, int64_t scratch_floats,
                       cudaStream_t st, const float* mw = nullptr, int d_out = 0, float* out = nullptr,
                       int64_t ldo = 0, int64_t x_rows = 0, int alpha = 0, int64_t n_chunks = 0) {
  using C = WarpCfg<SWV>;
  const int FS = (dim + C::kFeat - 1) / C::kFeat;
  const bool want = g_warp_paired == 1 || (g_warp_paired == 2 && x_rows * ldx * 2 > kPairMinXBytes);
  // the fused epilogue pairs 2 slices (out partials summed through shared memory, one named barrier
  // pair per window end); the plain SpMM any FS dividing the CTA's warps
  const int paired = (FS > 1 && want && C::kWarps % FS == 0 && (!FUSED || FS == 2)) ? 1 : 0;
  const int grid = tile_grid((paired ? 1 : FS) * n_chunks, paired ? C::kWarps / FS : C::kWarps);
  const int64_t nwarps = (int64_t)grid * C::kWarps;
  const int64_t cw = 2 * tile_cnt_words();
  const int64_t need = cw + nwarps * 2 * C::kSlot + (FUSED ? nwarps * 2 * kOutSlot : 0);
  HCS_REQUIRE(scratch != nullptr && scratch_floats >= need, HCS_EINVAL, "tile scratch too small (%lld floats, need %lld)",
              (long long)scratch_floats, (long long)need);
  unsigned* cnt = reinterpret_cast<unsigned*>(scratch);
  float* slots = scratch + cw;
  float* oscratch = slots + nwarps * 2 * C::kSlot;
  const int smem = C::kSmem + (FUSED ? kFusedOutMax * kFusedLdw * 2 : 0);
  // one slice of 33..48 features: the fused (GCN) kernel skips the empty 16-feature group
  // (C3 5.92 -> 5.71 ms); the plain SpMM is faster with the full unrolled schedule now that
  // every lane copies whole padded rows (N = 40/41/48: 1.29 -> 1.21 ms; tools/exp_c3_npr3.sh)
  const bool npr3 = FUSED && g_warp_npr3 && SWV == 8 && FS == 1 && dim <= 48 && dim > 32;
  // cost-weighted ranges (positions are chunks when paired or FS == 1)
  int64_t* wb = nullptr;
  const int64_t ng = paired ? nwarps / FS : nwarps;
  if (alpha > 0 && !npr3 && (paired || FS == 1) && n_tile >= kBalanceMinTilesPerGroup * ng &&
      scratch_floats >= tile_bounds_offset_floats() + 2 * (ng + 1)) {
    wb = reinterpret_cast<int64_t*>(scratch + tile_bounds_offset_floats());
    k_tile_bounds<<<(unsigned)((ng + 8) / 8), 256, 0, st>>>(chunk_ptr, n_tile, ent_ptr, ng, alpha, wb);
    HCS_LAUNCH_CHECK("k_tile_bounds");
  }
  auto kern = npr3 ? k_tile_warp<SWV, FUSED, (SWV == 8 ? 3 : SWV / 2)>
                   : (wb ? k_tile_warp<SWV, FUSED, SWV / 2, true> : k_tile_warp<SWV, FUSED>);
  HCS_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  kern<<<grid, C::kWarps * 32, smem, st>>>(tile_list, n_tile, chunk_ptr, gidx, ent_ptr, ent, n_rows, wh, x, ldx, dim,
                                            FS, z, ldz, slots, mw, d_out, out, ldo, oscratch, paired, cnt, wb);
  HCS_LAUNCH_CHECK("k_tile_warp");
  return HCS_OK;
}

// K6/K7 on the warp kernel: dim <= 128, d_out <= 64, 64-feature slices.
int gcn_tile_warp(const int32_t* tile_list, int64_t n_tile, const int64_t* chunk_ptr, const int32_t* gidx,
                  const int64_t* ent_ptr, const uint32_t* ent, int64_t n_rows, int wh, const __nv_bfloat16* x,
                  int64_t ldx, int dim, float* z, int64_t ldz, const float* m, int d_out, float* out, int64_t ldo,
                  float* scratch, int64_t scratch_floats, cudaStream_t st) {
  return launch_warp<8, true>(tile_list, n_tile, chunk_ptr, gidx, ent_ptr, ent, n_rows, wh, x, ldx, dim, z, ldz,
                              scratch, scratch_floats, st, m, d_out, out, ldo);
}

int spmm_tile_warp(const int32_t* tile_list, int64_t n_tile, const int64_t* chunk_ptr, const int32_t* gidx,
                   const int64_t* ent_ptr, const uint32_t* ent, int64_t n_rows, int wh, const __nv_bfloat16* x,
                   int64_t x_rows, int64_t ldx, int dim, float* z, int64_t ldz, float* scratch, int64_t scratch_floats,
                   cudaStream_t st, int alpha = 0, int64_t n_chunks = 0) {
  // 64-feature slices halve the per-feature slab work once a window has >= 2 slices of 32
  const int swv = g_warp_swv ? g_warp_swv : (dim > 32 ? 8 : 4);
  if (swv == 16)
    return launch_warp<16>(tile_list, n_tile, chunk_ptr, gidx, ent_ptr, ent, n_rows, wh, x, ldx, dim, z, ldz, scratch,
                          scratch_floats, st, nullptr, 0, nullptr, 0, x_rows, 0, n_chunks);
  if (swv == 8)
    return launch_warp<8>(tile_list, n_tile, chunk_ptr, gidx, ent_ptr, ent, n_rows, wh, x, ldx, dim, z, ldz, scratch,
                          scratch_floats, st, nullptr, 0, nullptr, 0, x_rows, alpha, n_chunks);
  return launch_warp<4>(tile_list, n_tile, chunk_ptr, gidx, ent_ptr, ent, n_rows, wh, x, ldx, dim, z, ldz, scratch,
                          scratch_floats, st, nullptr, 0, nullptr, 0, x_rows, alpha, n_chunks);
}

int64_t tile_warp_scratch_floats() {
  // slots, then (ng + 1) int64 range bounds for up to one group per warp
  return tile_bounds_offset_floats() + 2 * ((int64_t)num_sms() * kMaxWarpsPerCta + 2);
}

}  // namespace hcs

using namespace hcs;

// K4: tile windows on the tensor cores (executors.py:111-141 tile_window for every window of
// tile_list).  bf16 plan + bf16 X: k_tile_warp (mma.sync m16n8k16); fp32 plan + tf32-rounded fp32
// X: k_tile_warp_tf32 (m16n8k8).  workspace: >= hcs_tile_scratch_floats() floats.
extern "C" int hcs_spmm_tile_balanced(const int32_t* tile_list, int64_t n_tile, const int64_t* chunk_ptr,
                                      const int32_t* gidx, const int64_t* ent_ptr, const void* ent, int ent_dtype,
                                      int64_t n_rows, int32_t wh, const void* x, int x_dtype, int64_t x_rows,
                                      int32_t dim, int64_t ldx, float* z, int64_t ldz, void* workspace,
                                      size_t ws_bytes, int alpha, int64_t n_chunks, void* stream) {
  HCS_REQUIRE(alpha >= 0 && alpha <= 1 << 16, HCS_EINVAL, "tile balance alpha must be in [0, 65536] (got %d)", alpha);
  HCS_REQUIRE(wh > 0 && wh <= 16, HCS_EINVAL, "tile path supports window heights 1..16 (got %d)", wh);
  HCS_REQUIRE(dim > 0, HCS_EINVAL, "dim must be positive");
  HCS_REQUIRE(((uintptr_t)x & 15) == 0, HCS_EINVAL, "x must be 16-byte aligned");
  HCS_REQUIRE(x_dtype == ent_dtype, HCS_EINVAL, "x and plan dtypes differ (%d vs %d)", x_dtype, ent_dtype);
  HCS_REQUIRE(((uintptr_t)z & 7) == 0 && ldz % 2 == 0, HCS_EINVAL, "z must be 8-byte aligned with even ldz");
  if (x_dtype == HCS_DTYPE_F32) {
    HCS_REQUIRE(ldx % 4 == 0 && ldx >= ((dim + 3) / 4) * 4, HCS_EINVAL, "ldx must be a multiple of 4 covering dim");
    if (n_tile == 0) return HCS_OK;
    return spmm_tile_warp_tf32(tile_list, n_tile, chunk_ptr, gidx, ent_ptr, (const uint2*)ent, n_rows, wh,
                               (const float*)x, ldx, dim, z, ldz, (float*)workspace,
                               (int64_t)(ws_bytes / sizeof(float)), as_stream(stream), nullptr, 0, nullptr, 0,
                               n_chunks);
  }
  HCS_REQUIRE(x_dtype == HCS_DTYPE_BF16, HCS_EINVAL, "tile path: x dtype must be bf16 or f32 (tf32)");
  HCS_REQUIRE(ldx % 8 == 0 && ldx >= ((dim + 7) / 8) * 8, HCS_EINVAL, "ldx must be a multiple of 8 covering dim");
  if (n_tile == 0) return HCS_OK;
  return spmm_tile_warp(tile_list, n_tile, chunk_ptr, gidx, ent_ptr, (const uint32_t*)ent, n_rows, wh,
                        (const __nv_bfloat16*)x, x_rows, ldx, dim, z, ldz, (float*)workspace,
                        (int64_t)(ws_bytes / sizeof(float)), as_stream(stream), alpha, n_chunks);
}

extern "C" int hcs_spmm_tile(const int32_t* tile_list, int64_t n_tile, const int64_t* chunk_ptr, const int32_t* gidx,
                             const int64_t* ent_ptr, const void* ent, int ent_dtype, int64_t n_rows, int32_t wh,
                             const void* x, int x_dtype, int64_t x_rows, int32_t dim, int64_t ldx, float* z,
                             int64_t ldz, void* workspace, size_t ws_bytes, void* stream) {
  return hcs_spmm_tile_balanced(tile_list, n_tile, chunk_ptr, gidx, ent_ptr, ent, ent_dtype, n_rows, wh, x, x_dtype,
                                x_rows, dim, ldx, z, ldz, workspace, ws_bytes, 0, 0, stream);
}

// K6/K7: tile windows with the fused GCN epilogue: out = (A_w X) M per TILE window, plus
// z = A_w X when z != NULL (the forward z_cache).  M: fp32 [dim x d_out] row-major device matrix
// (W forward, W^T backward).  bf16: dim <= 128, d_out <= 64; tf32 (fp32 plan + X, M already
// RNA-rounded to tf32 by the caller): any dim, d_out <= 64.
extern "C" int hcs_gcn_tile(const int32_t* tile_list, int64_t n_tile, const int64_t* chunk_ptr, const int32_t* gidx,
                            const int64_t* ent_ptr, const void* ent, int ent_dtype, int64_t n_rows, int32_t wh,
                            const void* x, int x_dtype, int64_t x_rows, int32_t dim, int64_t ldx, float* z,
                            int64_t ldz, const float* m, int32_t d_out, float* out, int64_t ldo, void* workspace,
                            size_t ws_bytes, void* stream) {
  HCS_REQUIRE(wh > 0 && wh <= 16, HCS_EINVAL, "tile path supports window heights 1..16 (got %d)", wh);
  HCS_REQUIRE(d_out > 0 && d_out <= kFusedOutMax, HCS_EINVAL, "fused GCN tile path needs 1 <= d_out <= %d (got %d)",
              kFusedOutMax, d_out);
  HCS_REQUIRE(x_dtype == ent_dtype, HCS_EINVAL, "x and plan dtypes differ (%d vs %d)", x_dtype, ent_dtype);
  HCS_REQUIRE(((uintptr_t)x & 15) == 0, HCS_EINVAL, "x must be 16-byte aligned");
  HCS_REQUIRE(m != nullptr && out != nullptr && ldo >= d_out, HCS_EINVAL, "fused GCN: bad M / out arguments");
  HCS_REQUIRE(z == nullptr || (((uintptr_t)z & 7) == 0 && ldz % 2 == 0), HCS_EINVAL,
              "z must be 8-byte aligned with even ldz");
  cudaStream_t st = as_stream(stream);
  if (x_dtype == HCS_DTYPE_F32) {
    HCS_REQUIRE(dim > 0 && ldx % 4 == 0 && ldx >= ((dim + 3) / 4) * 4, HCS_EINVAL,
                "ldx must be a multiple of 4 covering dim");
    if (n_tile == 0) return HCS_OK;
    return spmm_tile_warp_tf32(tile_list, n_tile, chunk_ptr, gidx, ent_ptr, (const uint2*)ent, n_rows, wh,
                               (const float*)x, ldx, dim, z, ldz, (float*)workspace,
                               (int64_t)(ws_bytes / sizeof(float)), st, m, d_out, out, ldo);
  }
  HCS_REQUIRE(x_dtype == HCS_DTYPE_BF16, HCS_EINVAL, "tile path: x dtype must be bf16 or f32 (tf32)");
  HCS_REQUIRE(dim > 0 && dim <= 128, HCS_EINVAL, "fused bf16 GCN tile path needs 1 <= d_in <= 128 (got %d)", dim);
  HCS_REQUIRE(ldx % 8 == 0 && ldx >= ((dim + 7) / 8) * 8, HCS_EINVAL, "ldx must be a multiple of 8 covering dim");
  if (n_tile == 0) return HCS_OK;
  return gcn_tile_warp(tile_list, n_tile, chunk_ptr, gidx, ent_ptr, (const uint32_t*)ent, n_rows, wh,
                       (const __nv_bfloat16*)x, ldx, dim, z, ldz, m, d_out, out, ldo, (float*)workspace,
                       (int64_t)(ws_bytes / sizeof(float)), st);
}

// Experiment switch: the fused kernel's NPR = 3 variant for a single 33..48-feature slice (1, default) or the full one (0).
extern "C" int hcs_set_tile_npr3(int on) {
  HCS_REQUIRE(on == 0 || on == 1, HCS_EINVAL, "npr3 must be 0 or 1 (got %d)", on);
  hcs::g_warp_npr3 = on;
  return HCS_OK;
}

// Row-slice width of the warp-independent tile kernel: 0 auto, 4 (32 features) or 8 (64).
extern "C" int hcs_set_tile_slice(int vectors) {
  HCS_REQUIRE(vectors == 0 || vectors == 4 || vectors == 8 || vectors == 16, HCS_EINVAL,
              "slice must be 0, 4, 8 or 16 (got %d)", vectors);
  hcs::g_warp_swv = vectors;
  return HCS_OK;
}

// Paired feature slices (1, default), one warp per (window, slice) range (0), or auto (2:
// paired when X exceeds 96 MB, i.e. is not L2-resident).  Both are
// deterministic; windows are cut at different chunk boundaries, so the last bits can differ.
extern "C" int hcs_set_tile_pairing(int on) {
  HCS_REQUIRE(on >= 0 && on <= 2, HCS_EINVAL, "pairing must be 0, 1 or 2 (got %d)", on);
  hcs::g_warp_paired = on;
  hcs::g_warp_paired_tf32 = on ? 1 : 0;
  return HCS_OK;
}

extern "C" int hcs_tile_scratch_floats(int64_t* floats) {
  HCS_REQUIRE(floats != nullptr, HCS_EINVAL, "floats is NULL");
  *floats = hcs::tile_warp_scratch_floats();
  return HCS_OK;
}

// CTAs per tile launch: 0 = one per SM (default), n > 0 = min(n, SMs).  Results are deterministic
// for a given grid; different grids cut windows at different chunks (fp32 summation order).
extern "C" int hcs_set_tile_grid(int ctas) {
  HCS_REQUIRE(ctas >= 0, HCS_EINVAL, "tile grid must be >= 0 (got %d)", ctas);
  hcs::g_tile_grid = ctas;
  return HCS_OK;
}
