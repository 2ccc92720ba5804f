// K8: LOA layout reorganisation (paper Alg. 6; reference layout.py:186-263
// build_windows_optimized, with sort_by_min_neighbor 99-109 done by the caller).
//
// The greedy builder is strictly sequential (the next seed and the candidate set
// depend on every earlier pick), so it runs as ONE persistent CTA of 1024
// threads that executes the whole outer loop on the device; each step is
// parallel inside the CTA:
//   scan   : the first vw UNVISITED sorted positions (>= the seed position, which
//            is the smallest unvisited one: layout.py:112-115, 221-226) from a
//            visited bitmap, by warp ballots/popc;
//   score  : cns[v] = |N(v) ∩ all_cols| is PULLED for the <= vw candidates from an
//            all_cols bitmap (the reference PUSHES cns[w] += 1 for every w in N(c)
//            of every new column c; both give the same integers on an undirected
//            graph, pull costs Σ deg(candidates) per step and no reset
//            bookkeeping); the candidates' neighbour lists are flattened and split
//            evenly over the 32 warps so hub candidates do not serialise a warp;
//   argmax : exact key (num*b_den vs b_num*den, then strictly higher degree,
//            then earliest scan index; layout.py:118-130) reduced over the CTA;
//            (num, den) = (cur_eles+deg, cur_cols+deg-cns), den 0 -> (0, 1)
//            (layout.py:80-91);
//   admit  : atomicOr of the winner's neighbours into all_cols; the count of
//            newly set bits is cur_cols' increment (layout.py:211-219);
//   close  : the words touched by the group's neighbours are zeroed (the sparse
//            reset of layout.py:260-262).
// Bitmaps live in shared memory when 2*ceil(n/32) words fit, else in a global
// workspace (L2-resident).  All integer arithmetic: bit-exact with the reference.
#include "common.cuh"

namespace hcs {

constexpr int kLoaThreads = 1024;
constexpr int kLoaMaxVw = 1024;
constexpr int kLoaSmemBitmapBytes = 192 * 1024;  // both bitmaps in smem up to n = 786,432

struct LoaKey {
  int64_t num, den, deg;
  int k;
};
// strict total order of the reference's _pick_best (layout.py:118-130): larger wins
__device__ __forceinline__ bool loa_better(const LoaKey& a, const LoaKey& b) {
  if (a.k < 0) return false;
  if (b.k < 0) return true;
  const __int128 lhs = (__int128)a.num * b.den, rhs = (__int128)b.num * a.den;
  if (lhs != rhs) return lhs > rhs;
  if (a.deg != b.deg) return a.deg > b.deg;
  return a.k < b.k;
}
__device__ __forceinline__ LoaKey shfl_key(const LoaKey& a, int src) {
  LoaKey r;
  r.num = __shfl_sync(0xffffffffu, a.num, src);
  r.den = __shfl_sync(0xffffffffu, a.den, src);
  r.deg = __shfl_sync(0xffffffffu, a.deg, src);
  r.k = __shfl_sync(0xffffffffu, a.k, src);
  return r;
}

struct LoaShared {
  int cand_pos[kLoaMaxVw];
  int cand_v[kLoaMaxVw];
  int64_t cand_row[kLoaMaxVw];   // row_ptr[v]
  int64_t prefix[kLoaMaxVw + 1]; // exclusive prefix of candidate degrees
  int cnt[kLoaMaxVw];            // cns of each candidate
  LoaKey wbest[32];
  int64_t warp_sum[32];
  int64_t seed_pos, cur_eles, cur_cols, outpos, ngroups;
  int nc, glen, best_k;
  unsigned long long newcols;
};

__device__ __forceinline__ bool bit_test(const uint32_t* bm, int64_t i) { return (bm[i >> 5] >> (i & 31)) & 1u; }

// admit(v): OR N(v) into all_cols, return #new columns (block-wide; all threads get it)
__device__ void loa_admit(LoaShared& sh, const int64_t* __restrict__ rp, const int32_t* __restrict__ ci,
                          uint32_t* allcols, int v) {
  const int64_t e0 = rp[v], e1 = rp[v + 1];
  unsigned long long mine = 0;
  for (int64_t e = e0 + threadIdx.x; e < e1; e += blockDim.x) {
    const int c = ci[e];
    const uint32_t bit = 1u << (c & 31);
    const uint32_t old = atomicOr(&allcols[c >> 5], bit);
    mine += (old & bit) ? 0ull : 1ull;
  }
  for (int o = 16; o > 0; o >>= 1) mine += __shfl_xor_sync(0xffffffffu, mine, o);
  if ((threadIdx.x & 31) == 0 && mine) atomicAdd(&sh.newcols, mine);
  __syncthreads();
  if (threadIdx.x == 0) {
    sh.cur_cols += (int64_t)sh.newcols;
    sh.cur_eles += e1 - e0;
    sh.newcols = 0;
  }
  __syncthreads();
}

__global__ void __launch_bounds__(kLoaThreads, 1)
    k_loa(const int64_t* __restrict__ rp, const int32_t* __restrict__ ci, int64_t n, int vw, int gs,
          const int32_t* __restrict__ order, int32_t* __restrict__ out_order, int64_t* __restrict__ gptr,
          int64_t* __restrict__ ngroups_out, uint32_t* gbits, int use_smem_bits) {
  extern __shared__ __align__(16) uint8_t loa_smem[];
  __shared__ LoaShared sh;
  const int64_t nwords = (n + 31) >> 5;
  uint32_t* allcols = use_smem_bits ? reinterpret_cast<uint32_t*>(loa_smem) : gbits;
  uint32_t* visited = allcols + nwords;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (use_smem_bits) {
    for (int64_t i = tid; i < 2 * nwords; i += blockDim.x) allcols[i] = 0u;
  }
  if (tid == 0) {
    sh.seed_pos = 0;
    sh.outpos = 0;
    sh.ngroups = 0;
    sh.newcols = 0;
    gptr[0] = 0;
  }
  __syncthreads();
  for (;;) {
    // ---- next seed: smallest unvisited position (layout.py:221-226)
    if (tid == 0) {
      int64_t p = sh.seed_pos;
      while (p < n && bit_test(visited, p)) ++p;
      sh.seed_pos = p;
      if (p < n) {
        visited[p >> 5] |= 1u << (p & 31);
        const int v0 = order[p];
        out_order[sh.outpos] = v0;
        sh.glen = 1;
        sh.cur_eles = 0;
        sh.cur_cols = 0;
        sh.cand_v[0] = v0;  // scratch: seed vertex for the admit below
      }
    }
    __syncthreads();
    if (sh.seed_pos >= n) break;
    loa_admit(sh, rp, ci, allcols, sh.cand_v[0]);
    while (sh.glen < gs) {
      // ---- scan: first vw unvisited positions (warp 0)
      if (warp == 0) {
        int got = 0;
        for (int64_t wb = sh.seed_pos >> 5; got < vw && wb < nwords; wb += 32) {
          const int64_t w = wb + lane;
          uint32_t bits = 0;
          if (w < nwords) {
            bits = ~visited[w];
            const int64_t hi = n - w * 32;  // valid positions in this word
            if (hi < 32) bits &= (1u << hi) - 1u;
          }
          const int c = __popc(bits);
          int incl = c;
          for (int o = 1; o < 32; o <<= 1) {
            const int t = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += t;
          }
          int slot = got + incl - c;
          while (bits && slot < vw) {
            const int b = __ffs(bits) - 1;
            sh.cand_pos[slot++] = (int)(w * 32 + b);
            bits &= bits - 1u;
          }
          got += __shfl_sync(0xffffffffu, incl, 31);
        }
        if (lane == 0) sh.nc = got < vw ? got : vw;
      }
      __syncthreads();
      const int nc = sh.nc;
      if (nc == 0) break;
      // ---- candidate vertices, degrees and their exclusive prefix (warp-scan + warp sums)
      int64_t d = 0;
      if (tid < nc) {
        const int v = order[sh.cand_pos[tid]];
        sh.cand_v[tid] = v;
        const int64_t r0 = rp[v];
        sh.cand_row[tid] = r0;
        d = rp[v + 1] - r0;
        sh.cnt[tid] = 0;
      }
      int64_t incl = d;
      for (int o = 1; o < 32; o <<= 1) {
        const int64_t t = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += t;
      }
      if (lane == 31) sh.warp_sum[warp] = incl;
      __syncthreads();
      if (warp == 0) {
        int64_t s = sh.warp_sum[lane];
        int64_t si = s;
        for (int o = 1; o < 32; o <<= 1) {
          const int64_t t = __shfl_up_sync(0xffffffffu, si, o);
          if (lane >= o) si += t;
        }
        sh.warp_sum[lane] = si - s;  // exclusive warp offsets
      }
      __syncthreads();
      if (tid < nc) sh.prefix[tid] = sh.warp_sum[warp] + incl - d;
      if (tid == nc - 1) sh.prefix[nc] = sh.warp_sum[warp] + incl;
      __syncthreads();
      // ---- pull: cns[k] = |N(v_k) ∩ all_cols| over the flattened candidate adjacency
      {
        const int64_t total = sh.prefix[nc];
        const int64_t per = ((total + 31) / 32 + 31) & ~(int64_t)31;  // per-warp segment, multiple of 32
        const int64_t s0 = (int64_t)warp * per, s1 = min(total, s0 + per);
        int k = 0;
        {  // first candidate of this warp's segment
          int lo = 0, hi = nc;  // last k with prefix[k] <= s0
          while (hi - lo > 1) {
            const int mid = (lo + hi) >> 1;
            if (sh.prefix[mid] <= s0) lo = mid; else hi = mid;
          }
          k = lo;
        }
        // kLoaProbe neighbour loads in flight per lane; hits summed lane-locally and flushed
        // once per candidate (integer sums: the counts are exact in any order)
        constexpr int kLoaProbe = 8;
        int local = 0, kcur = k;
        for (int64_t ib = s0 + lane; ib < s1; ib += 32 * kLoaProbe) {
          int cc[kLoaProbe], kk[kLoaProbe];
#pragma unroll
          for (int u = 0; u < kLoaProbe; ++u) {
            const int64_t i = ib + 32 * u;
            kk[u] = -1;
            cc[u] = 0;
            if (i < s1) {
              while (sh.prefix[k + 1] <= i) ++k;
              kk[u] = k;
              cc[u] = __ldg(ci + sh.cand_row[k] + (i - sh.prefix[k]));
            }
          }
#pragma unroll
          for (int u = 0; u < kLoaProbe; ++u) {
            if (kk[u] < 0) continue;
            if (kk[u] != kcur) {
              if (local) atomicAdd(&sh.cnt[kcur], local);
              local = 0;
              kcur = kk[u];
            }
            local += bit_test(allcols, cc[u]) ? 1 : 0;
          }
        }
        if (local) atomicAdd(&sh.cnt[kcur], local);
      }
      __syncthreads();
      // ---- argmax over the candidates (exact key, CTA reduction)
      LoaKey key;
      key.k = -1;
      key.num = 0;
      key.den = 1;
      key.deg = 0;
      if (tid < nc) {
        const int64_t dg = sh.prefix[tid + 1] - sh.prefix[tid];
        int64_t num = sh.cur_eles + dg;
        int64_t den = sh.cur_cols + dg - sh.cnt[tid];
        if (den == 0) {
          num = 0;
          den = 1;
        }
        key.num = num;
        key.den = den;
        key.deg = dg;
        key.k = tid;
      }
      for (int o = 16; o > 0; o >>= 1) {
        const LoaKey other = shfl_key(key, lane ^ o);
        if (loa_better(other, key)) key = other;
      }
      if (lane == 0) sh.wbest[warp] = key;
      __syncthreads();
      if (warp == 0) {
        key = sh.wbest[lane];
        for (int o = 16; o > 0; o >>= 1) {
          const LoaKey other = shfl_key(key, lane ^ o);
          if (loa_better(other, key)) key = other;
        }
        if (lane == 0) {
          const int kb = key.k;
          const int p = sh.cand_pos[kb];
          visited[p >> 5] |= 1u << (p & 31);
          out_order[sh.outpos + sh.glen] = sh.cand_v[kb];
          sh.glen += 1;
          sh.best_k = kb;
        }
      }
      __syncthreads();
      loa_admit(sh, rp, ci, allcols, sh.cand_v[sh.best_k]);
    }
    // ---- close the group: record it, zero the all_cols words its neighbours touched
    const int glen = sh.glen;
    const int64_t o0 = sh.outpos;
    for (int j = 0; j < glen; ++j) {
      const int v = out_order[o0 + j];
      for (int64_t e = rp[v] + tid; e < rp[v + 1]; e += blockDim.x) allcols[ci[e] >> 5] = 0u;
    }
    __syncthreads();
    if (tid == 0) {
      sh.outpos = o0 + glen;
      sh.ngroups += 1;
      gptr[sh.ngroups] = sh.outpos;
    }
    __syncthreads();
  }
  if (tid == 0) *ngroups_out = sh.ngroups;
}

}  // namespace hcs

using namespace hcs;

extern "C" int hcs_loa_workspace_bytes(int64_t n, size_t* bytes) {
  HCS_REQUIRE(n >= 0 && bytes, HCS_EINVAL, "bad arguments");
  const int64_t nwords = (n + 31) / 32;
  *bytes = (2 * nwords * 4 <= kLoaSmemBitmapBytes) ? 16 : (size_t)(2 * nwords * 4);
  return HCS_OK;
}

extern "C" int hcs_loa(const int64_t* row_ptr, const int32_t* col_idx, int64_t n, int32_t vw, int32_t group_size,
                       const int32_t* order, int32_t* out_order, int64_t* gptr, int64_t* ngroups, void* workspace,
                       size_t ws_bytes, void* stream) {
  HCS_REQUIRE(vw >= 1, HCS_EINVAL, "vw must be >= 1");
  HCS_REQUIRE(vw <= kLoaMaxVw, HCS_EINVAL, "vw must be <= %d on the GPU builder (got %d)", kLoaMaxVw, vw);
  HCS_REQUIRE(group_size >= 1, HCS_EINVAL, "group_size must be >= 1");
  HCS_REQUIRE(n >= 0 && n < (1LL << 31) - 1, HCS_EINVAL, "vertex count must fit in int32");
  cudaStream_t st = as_stream(stream);
  if (n == 0) {
    HCS_CUDA(cudaMemsetAsync(gptr, 0, sizeof(int64_t), st));
    HCS_CUDA(cudaMemsetAsync(ngroups, 0, sizeof(int64_t), st));
    return HCS_OK;
  }
  const int64_t nwords = (n + 31) / 32;
  const bool smem_bits = 2 * nwords * 4 <= kLoaSmemBitmapBytes;
  size_t dyn = 0;
  uint32_t* gbits = nullptr;
  if (smem_bits) {
    dyn = (size_t)(2 * nwords * 4);
  } else {
    HCS_REQUIRE(workspace && ws_bytes >= (size_t)(2 * nwords * 4), HCS_EINVAL, "LOA workspace too small");
    gbits = reinterpret_cast<uint32_t*>(workspace);
    HCS_CUDA(cudaMemsetAsync(gbits, 0, (size_t)(2 * nwords * 4), st));
  }
  HCS_CUDA(cudaFuncSetAttribute(k_loa, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kLoaSmemBitmapBytes));
  k_loa<<<1, kLoaThreads, dyn, st>>>(row_ptr, col_idx, n, vw, group_size, order, out_order, gptr, ngroups, gbits,
                                     smem_bits ? 1 : 0);
  HCS_LAUNCH_CHECK("k_loa");
  return HCS_OK;
}
