// K4 variant for feature widths <= 32 (one 32-feature slice): the X rows of a chunk are
// gathered straight into registers (LDG.64, 4 features per lane) instead of through shared
// memory, so a gathered byte costs the L1 data path once instead of cp.async write +
// ldmatrix read ("past the LSU floor").
//
// mma.sync m16n8k16 B fragments want, per lane (g8 = lane/4, t4 = lane%4), the k-pairs
// {2t4, 2t4+1} and {2t4+8, 2t4+9} of one column n = g8.  Each lane loads features
// 4 g8 .. 4 g8 + 3 of its four chunk rows and pairs rows with prmt, which makes the n-tile
// index the feature's low 2 bits: n-tile j, column g8 holds feature 4 g8 + j.  The
// accumulators therefore hold, for row g8 (+8), features 8 t4 + j and 8 t4 + 4 + j: two
// contiguous float4 per row at the store.  The slab (A operand), the plan, the warp ranges
// and the fix-up are those of k_tile_warp (partial slots are written in its layout).
#include "common.cuh"
#include "mma_helpers.cuh"

namespace hcs {

constexpr int kRegWarps = 12;
constexpr int kRegSlabBytes = 16 * 64 * 2;
constexpr int kRegEntRegs = 4;  // 128 packed entries per chunk held in registers
constexpr int kRegSlot = 16 * 32;  // floats of one 16 x 32 partial (k_tile_warp_fixup<4> layout)

__device__ __forceinline__ int64_t rg_ld64(const int64_t* p) { return __ldg(p); }

__device__ __forceinline__ uint32_t rg_plan_u32(const uint32_t* p, uint64_t pol) {
  uint32_t r;
  asm volatile("ld.global.nc.L2::cache_hint.u32 %0, [%1], %2;" : "=r"(r) : "l"(p), "l"(pol));
  return r;
}
__device__ __forceinline__ int2 rg_plan_s32x2(const int32_t* p, uint64_t pol) {
  int2 r;
  asm volatile("ld.global.nc.L2::cache_hint.v2.s32 {%0,%1}, [%2], %3;" : "=r"(r.x), "=r"(r.y) : "l"(p), "l"(pol));
  return r;
}
__device__ __forceinline__ uint2 rg_x8(const void* p, uint64_t pol) {
  uint2 r;
  asm volatile("ld.global.nc.L2::cache_hint.v2.u32 {%0,%1}, [%2], %3;" : "=r"(r.x), "=r"(r.y) : "l"(p), "l"(pol));
  return r;
}

__global__ void __launch_bounds__(kRegWarps * 32, 1)
    k_tile_reg32(const int32_t* __restrict__ tile_list, int64_t T, const int64_t* __restrict__ chunk_ptr,
                 const int32_t* __restrict__ gidx, const int64_t* __restrict__ ent_ptr,
                 const uint32_t* __restrict__ ent, int64_t n_rows, int wh, const __nv_bfloat16* __restrict__ x,
                 int64_t ldx, int dim, float* __restrict__ z, int64_t ldz, float* __restrict__ scratch) {
  extern __shared__ uint8_t rsm_raw[];
  uint8_t* rsm = (uint8_t*)(((uintptr_t)rsm_raw + 127) & ~(uintptr_t)127);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t nwarps = (int64_t)gridDim.x * kRegWarps;
  const int64_t gw = (int64_t)blockIdx.x * kRegWarps + warp;
  const int64_t c0 = chunk_ptr[0];
  const int64_t total = chunk_ptr[T] - c0;
  const int64_t a = (total * gw) / nwarps, b = (total * (gw + 1)) / nwarps;
  if (a >= b) return;
  const uint32_t slab = smem_u32(rsm + warp * kRegSlabBytes);
  const uint64_t keep = policy_evict_last();
  const uint64_t once = policy_evict_first();
  const int g8 = lane >> 2, t4 = lane & 3;
  const int ar = lane & 15, akc = lane >> 4;
  const bool feat_live = 4 * g8 < dim;
  const char* xb = reinterpret_cast<const char*>(x) + 8 * g8;  // features 4 g8 .. 4 g8 + 3
  const int64_t ldxb = ldx * 2;

  // window t containing flattened chunk v (largest t with chunk_ptr[t] - c0 <= v)
  int64_t lo = 0, hi = T;
  while (hi - lo > 1) {
    const int64_t mid = (lo + hi) >> 1;
    if (rg_ld64(chunk_ptr + mid) - c0 <= a) lo = mid; else hi = mid;
  }
  struct Pos {
    int64_t base, c;  // chunk_ptr[t], absolute chunk
    int32_t t, rem;   // rem = chunks left in the warp's range (valid while > 0)
  };
  Pos P;
  P.t = (int32_t)lo;
  P.base = rg_ld64(chunk_ptr + lo);
  P.c = c0 + a;
  P.rem = (int32_t)(b - a);
  const bool in_head0 = P.c != P.base;  // our first window began in an earlier warp's range
  auto adv = [&](Pos& p) {
    --p.rem;
    ++p.c;
    if (p.rem > 0 && p.c == rg_ld64(chunk_ptr + p.t + 1)) {
      ++p.t;
      p.base = p.c;
    }
  };
  // gather indices of the lane's four rows in each k16 step: slots ks*16 + {2t4, 2t4+1, 2t4+8, 2t4+9}
  auto load_g = [&](const Pos& p, int2 (&g)[8]) {
#pragma unroll
    for (int ks = 0; ks < 4; ++ks) {
      if (p.rem > 0) {
        const int32_t* gp = gidx + p.c * 64 + ks * 16 + 2 * t4;
        g[2 * ks] = rg_plan_s32x2(gp, once);
        g[2 * ks + 1] = rg_plan_s32x2(gp + 8, once);
      } else {
        g[2 * ks] = g[2 * ks + 1] = make_int2(-1, -1);
      }
    }
  };
  auto load_x = [&](const int2 (&g)[8], uint2 (&xv)[16]) {
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const int i0 = g[q].x, i1 = g[q].y;
      xv[2 * q] = (feat_live && i0 >= 0) ? rg_x8(xb + (int64_t)i0 * ldxb, keep) : make_uint2(0u, 0u);
      xv[2 * q + 1] = (feat_live && i1 >= 0) ? rg_x8(xb + (int64_t)i1 * ldxb, keep) : make_uint2(0u, 0u);
    }
  };
  auto load_ep = [&](const Pos& p, int64_t& e0, int64_t& e1) {
    if (p.rem > 0) {
      e0 = rg_ld64(ent_ptr + p.c);
      e1 = rg_ld64(ent_ptr + p.c + 1);
    } else {
      e0 = e1 = 0;
    }
  };
  auto load_ent = [&](int64_t e0, int64_t e1, uint32_t (&e)[kRegEntRegs]) {
#pragma unroll
    for (int q = 0; q < kRegEntRegs; ++q) {
      const int64_t i = e0 + lane + 32 * q;
      e[q] = i < e1 ? rg_plan_u32(ent + i, once) : 0u;
    }
  };

  float acc[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i) acc[i][0] = acc[i][1] = acc[i][2] = acc[i][3] = 0.f;
  bool in_head = in_head0;
#pragma unroll
  for (int q = 0; q < 4; ++q) sts128_zero(slab + (lane + 32 * q) * 16);
  __syncwarp();

  // one chunk: compute P0 with Xc/Ec while P1's rows (indices G1) load into Xn and P2's
  // indices into G2 (register sets are renamed by the caller, so no in-flight load is copied)
  auto step = [&](const Pos& P0, const Pos& P1, const Pos& P2, uint2 (&Xc)[16], uint2 (&Xn)[16],
                  const int2 (&G1)[8], int2 (&G2)[8], uint32_t (&Ec)[kRegEntRegs], uint32_t (&En)[kRegEntRegs],
                  const int64_t (&EPc)[2], int64_t (&EPn)[2]) -> bool {
    if (P0.rem <= 0) return true;
    load_x(G1, Xn);  // P1's rows
    load_g(P2, G2);
    load_ep(P1, EPn[0], EPn[1]);
    load_ent(EPn[0], EPn[1], En);
    const int ne = (int)(EPc[1] - EPc[0]);
#pragma unroll
    for (int q = 0; q < kRegEntRegs; ++q)
      if (lane + 32 * q < ne) sts16(slab + (Ec[q] & 0x7FFu), Ec[q] >> 16);
    for (int i = 32 * kRegEntRegs + lane; i < ne; i += 32) {
      const uint32_t w = rg_plan_u32(ent + EPc[0] + i, once);
      sts16(slab + (w & 0x7FFu), w >> 16);
    }
    __syncwarp();
#pragma unroll
    for (int ks = 0; ks < 4; ++ks) {
      uint32_t af[4];
      const int kc = 2 * ks + akc;
      ldsm_x4(af, slab + ar * 128 + (((kc ^ ar) & 7) << 4));
      // rows r0 = 2t4, r1 = 2t4+1 (xv[4ks], xv[4ks+1]) and r2 = 2t4+8, r3 = 2t4+9 (xv[4ks+2], xv[4ks+3])
      const uint2 v0 = Xc[4 * ks], v1 = Xc[4 * ks + 1], v2 = Xc[4 * ks + 2], v3 = Xc[4 * ks + 3];
      hmma_16816(acc[0], af, __byte_perm(v0.x, v1.x, 0x5410), __byte_perm(v2.x, v3.x, 0x5410));
      hmma_16816(acc[1], af, __byte_perm(v0.x, v1.x, 0x7632), __byte_perm(v2.x, v3.x, 0x7632));
      hmma_16816(acc[2], af, __byte_perm(v0.y, v1.y, 0x5410), __byte_perm(v2.y, v3.y, 0x5410));
      hmma_16816(acc[3], af, __byte_perm(v0.y, v1.y, 0x7632), __byte_perm(v2.y, v3.y, 0x7632));
    }
    __syncwarp();
    if (ne <= 32 * kRegEntRegs) {
#pragma unroll
      for (int q = 0; q < kRegEntRegs; ++q)
        if (lane + 32 * q < ne) sts16(slab + (Ec[q] & 0x7FFu), 0u);
    } else {
#pragma unroll
      for (int q = 0; q < 4; ++q) sts128_zero(slab + (lane + 32 * q) * 16);
    }
    __syncwarp();
    const bool unit_done = P0.c + 1 == rg_ld64(chunk_ptr + P0.t + 1);
    if (unit_done || P0.rem == 1) {
      const int64_t rs = (int64_t)__ldg(tile_list + P0.t) * wh;
      const int rows = (int)(n_rows - rs < wh ? n_rows - rs : wh);
      if (!in_head && unit_done) {
        // row g8 (+8): features 8 t4 + j (acc[j][0..1] -> rows g8, acc[j][2..3] -> g8+8; cols 2t4, 2t4+1)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int r = g8 + 8 * h;
          if (r < rows) {
            float* zr = z + (rs + r) * ldz;
            const int f0 = 8 * t4;
            const float o[8] = {acc[0][2 * h], acc[1][2 * h], acc[2][2 * h], acc[3][2 * h],
                                acc[0][2 * h + 1], acc[1][2 * h + 1], acc[2][2 * h + 1], acc[3][2 * h + 1]};
            if (f0 + 8 <= dim) {
              reinterpret_cast<float4*>(zr + f0)[0] = make_float4(o[0], o[1], o[2], o[3]);
              reinterpret_cast<float4*>(zr + f0)[1] = make_float4(o[4], o[5], o[6], o[7]);
            } else {
#pragma unroll
              for (int i = 0; i < 8; ++i)
                if (f0 + i < dim) zr[f0 + i] = o[i];
            }
          }
        }
      } else {
        // partial slot in k_tile_warp_fixup<4>'s layout: element (row r, feature f) at
        // ((f/8)*4 + (r/8)*2 + (f%2)) * 32 + (r%8)*4 + (f%8)/2
        float* slot = scratch + (gw * 2 + (in_head ? 0 : 1)) * kRegSlot;
#pragma unroll
        for (int h = 0; h < 2; ++h)
#pragma unroll
          for (int cc = 0; cc < 2; ++cc)
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              const int f = 4 * (2 * t4 + cc) + j, r = g8 + 8 * h;
              slot[((f >> 3) * 4 + h * 2 + (f & 1)) * 32 + (r & 7) * 4 + ((f & 7) >> 1)] = acc[j][2 * h + cc];
            }
      }
      in_head = false;
#pragma unroll
      for (int i = 0; i < 4; ++i) acc[i][0] = acc[i][1] = acc[i][2] = acc[i][3] = 0.f;
    }
    return false;
  };

  Pos Q0 = P, Q1 = P;
  adv(Q1);
  Pos Q2 = Q1;
  adv(Q2);
  int2 GA[8], GB[8];
  uint2 XA[16], XB[16];
  uint32_t EA[kRegEntRegs], EB[kRegEntRegs];
  int64_t EPA[2], EPB[2];
  load_g(Q0, GA);
  load_x(GA, XA);
  load_g(Q1, GB);
  load_ep(Q0, EPA[0], EPA[1]);
  load_ent(EPA[0], EPA[1], EA);
  for (;;) {
    if (step(Q0, Q1, Q2, XA, XB, GB, GA, EA, EB, EPA, EPB)) break;
    Q0 = Q1;
    Q1 = Q2;
    adv(Q2);
    if (step(Q0, Q1, Q2, XB, XA, GA, GB, EB, EA, EPB, EPA)) break;
    Q0 = Q1;
    Q1 = Q2;
    adv(Q2);
  }
}

int spmm_tile_reg32(const int32_t* tile_list, int64_t n_tile, const int64_t* chunk_ptr, const int32_t* gidx,
                    const int64_t* ent_ptr, const uint32_t* ent, int64_t n_rows, int wh, const __nv_bfloat16* x,
                    int64_t ldx, int dim, float* z, int64_t ldz, float* scratch, int64_t scratch_floats,
                    cudaStream_t st, int64_t* nwarps_out) {
  const int grid = num_sms();
  const int64_t nwarps = (int64_t)grid * kRegWarps;
  HCS_REQUIRE(scratch != nullptr && scratch_floats >= nwarps * 2 * kRegSlot, HCS_EINVAL, "tile scratch too small");
  const int smem = kRegWarps * kRegSlabBytes + 128;
  k_tile_reg32<<<grid, kRegWarps * 32, smem, st>>>(tile_list, n_tile, chunk_ptr, gidx, ent_ptr, ent, n_rows, wh, x,
                                                    ldx, dim, z, ldz, scratch);
  HCS_LAUNCH_CHECK("k_tile_reg32");
  *nwarps_out = nwarps;
  return HCS_OK;
}

}  // namespace hcs
