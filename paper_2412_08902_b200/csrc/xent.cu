// Softmax cross-entropy of the C3 training epoch (model.Gcn2; the reference has no loss):
//   loss   = -mean_i log_softmax(logits_i)[label_i]
//   grad_i = grad_scale * (softmax(logits_i) - onehot(label_i))
// in one pass over the logits, the gradient written straight as the backward aggregation's operand
// (bf16, rows padded with zeros to n_store columns = whole gather slices) or as fp32.  Replaces
// torch's log_softmax / gather / mean, their backward kernels and the operand staging copies
// (~170 us of small kernels per C3 epoch).
//
// One warp per row, kXentRows rows per pass with their loads in flight together (rows are a few
// hundred bytes: the kernel is load-latency bound); the loss is reduced deterministically: warp
// sums -> per-CTA partial in warp order -> the last CTA to finish (counter in the workspace) adds
// the partials in a fixed order.  A label outside [0, classes) makes its row's loss NaN (and its
// gradient row the plain softmax), so a bad label poisons the loss visibly instead of reading
// out of bounds.
#include <cmath>

#include "common.cuh"

namespace hcs {

constexpr int kXentThreads = 256;
constexpr int kXentRows = 4;  // rows per warp and pass
constexpr float kLog2e = 1.4426950408889634f;

// resident CTAs only (8 per SM): the loss partials the last CTA sums stay few (C3: 7,280 partials
// read ~28 deep per thread by the last CTA were most of the kernel's 40 us)
static int xent_grid(int64_t rows) {
  const int64_t per = (kXentThreads / 32) * kXentRows;
  return (int)std::max<int64_t>(1, std::min<int64_t>((rows + per - 1) / per, (int64_t)num_sms() * 8));
}

__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// one gradient value: grad_scale * (softmax - onehot); zero past C
__device__ __forceinline__ float xent_grad(float x, float m, float inv, int c, int C, int64_t lab, float scale) {
  return c < C ? (expf(x - m) * inv - (c == lab ? 1.f : 0.f)) * scale : 0.f;
}

template <bool BF16>
__device__ __forceinline__ void xent_store(void* grad, int64_t ldg, int64_t r, int c, int n_store, float v0,
                                           float v1) {
  if (BF16) {
    *reinterpret_cast<__nv_bfloat162*>(static_cast<__nv_bfloat16*>(grad) + r * ldg + c) =
        __floats2bfloat162_rn(v0, v1);
  } else {
    float* gp = static_cast<float*>(grad) + r * ldg + c;
    gp[0] = v0;
    if (c + 1 < n_store) gp[1] = v1;
  }
}

// GROUP: C <= 64 and n_store <= 64 -- 8 lanes per row, lane j of a group holding columns 8j..8j+7
// in registers, 4 rows per warp (the kernel is instruction-issue bound: 3-step group reductions
// shared by 4 rows, ex2/lg2 intrinsics, 16-byte loads and stores; C3: 101 -> 40 us); otherwise one
// warp per row with strided loops.  VEC: logits rows 16-byte aligned (ld % 4 == 0) and the bf16
// gradient rows too (ld_grad % 8 == 0).
template <bool BF16, bool GROUP, bool VEC>
__global__ void __launch_bounds__(kXentThreads) k_softmax_xent(const float* __restrict__ logits, int64_t ld,
                                                               int64_t rows, int C, const int64_t* __restrict__ labels,
                                                               float grad_scale, void* __restrict__ grad, int64_t ldg,
                                                               int n_store, float* __restrict__ partial,
                                                               unsigned* __restrict__ cnt, float* __restrict__ loss) {
  __shared__ float red[kXentThreads];
  __shared__ int last;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t step = (int64_t)gridDim.x * (kXentThreads / 32) * kXentRows;
  float lsum = 0.f;
  auto group_load = [&](int64_t r, int c0, float (&v)[8], int64_t& lab) {
    const bool live = r < rows;
    const float* x = logits + (live ? r : 0) * ld + c0;
    if (VEC) {
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        float4 q = make_float4(0.f, 0.f, 0.f, 0.f);
        if (live && c0 + 4 * h < C) q = __ldg(reinterpret_cast<const float4*>(x) + h);
        v[4 * h] = q.x, v[4 * h + 1] = q.y, v[4 * h + 2] = q.z, v[4 * h + 3] = q.w;
      }
    } else {
#pragma unroll
      for (int j = 0; j < 8; ++j) v[j] = (live && c0 + j < C) ? __ldg(x + j) : 0.f;
    }
    lab = live ? __ldg(labels + r) : 0;
  };
  float nv[8];
  int64_t nlab = 0;
  bool have_next = false;
  for (int64_t r0 = ((int64_t)blockIdx.x * (kXentThreads / 32) + warp) * kXentRows; r0 < rows; r0 += step) {
    if (GROUP) {
      const int64_t r = r0 + (lane >> 3);
      const int c0 = (lane & 7) * 8;
      const bool live = r < rows;
      float v[8];
      int64_t lab;
      if (have_next) {  // loaded during the previous row group
#pragma unroll
        for (int j = 0; j < 8; ++j) v[j] = nv[j];
        lab = nlab;
      } else {
        group_load(r, c0, v, lab);
      }
      // the next row group's loads go out before this group's math
      have_next = r0 + step < rows;
      if (have_next) group_load(r + step, c0, nv, nlab);
      float m = -INFINITY;
#pragma unroll
      for (int j = 0; j < 8; ++j) m = c0 + j < C ? fmaxf(m, v[j]) : m;
#pragma unroll
      for (int o = 4; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
      const float ml = m * kLog2e;
      float e[8], sum = 0.f;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        e[j] = c0 + j < C ? exp2f(fmaf(v[j], kLog2e, -ml)) : 0.f;
        sum += e[j];
      }
#pragma unroll
      for (int o = 4; o > 0; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
      const bool ok = lab >= 0 && lab < C;
      if (live) {
        if (ok && (int)(lab >> 3) == (lane & 7)) {  // the lane holding the label's logit
          float xl = 0.f;
#pragma unroll
          for (int j = 0; j < 8; ++j) xl = (c0 + j == (int)lab) ? v[j] : xl;
          lsum += (m + __logf(sum)) - xl;
        } else if (!ok && (lane & 7) == 0) {
          lsum += NAN;
        }
        const float inv = __frcp_rn(sum) * grad_scale;
        float g[8];
#pragma unroll
        for (int j = 0; j < 8; ++j)
          g[j] = c0 + j < C ? fmaf(e[j], inv, (c0 + j == (int)lab) ? -grad_scale : 0.f) : 0.f;
        if (c0 < n_store) {
          if (BF16) {
            __nv_bfloat16* gp = static_cast<__nv_bfloat16*>(grad) + r * ldg + c0;
            if (VEC && c0 + 8 <= n_store) {
              uint4 u;
              __nv_bfloat162 p0 = __floats2bfloat162_rn(g[0], g[1]), p1 = __floats2bfloat162_rn(g[2], g[3]);
              __nv_bfloat162 p2 = __floats2bfloat162_rn(g[4], g[5]), p3 = __floats2bfloat162_rn(g[6], g[7]);
              u.x = *reinterpret_cast<uint32_t*>(&p0), u.y = *reinterpret_cast<uint32_t*>(&p1);
              u.z = *reinterpret_cast<uint32_t*>(&p2), u.w = *reinterpret_cast<uint32_t*>(&p3);
              *reinterpret_cast<uint4*>(gp) = u;
            } else {
#pragma unroll
              for (int j = 0; j < 8; j += 2)
                if (c0 + j < n_store)
                  *reinterpret_cast<__nv_bfloat162*>(gp + j) = __floats2bfloat162_rn(g[j], g[j + 1]);
            }
          } else {
            float* gp = static_cast<float*>(grad) + r * ldg + c0;
#pragma unroll
            for (int j = 0; j < 8; ++j)
              if (c0 + j < n_store) gp[j] = g[j];
          }
        }
      }
    } else {
      for (int i = 0; i < kXentRows; ++i) {
        const int64_t r = r0 + i;
        if (r >= rows) break;
        const float* x = logits + r * ld;
        float m = -INFINITY;
        for (int c = lane; c < C; c += 32) m = fmaxf(m, __ldg(x + c));
        m = warp_max(m);
        float s = 0.f;
        for (int c = lane; c < C; c += 32) s += expf(__ldg(x + c) - m);
        s = warp_sum(s);
        const int64_t lab = __ldg(labels + r);
        const bool ok = lab >= 0 && lab < C;
        if (lane == 0) lsum += ok ? (m + logf(s)) - __ldg(x + lab) : NAN;
        const float inv = 1.f / s;
        for (int c = 2 * lane; c < n_store; c += 64) {
          const float v0 = c < C ? __ldg(x + c) : 0.f, v1 = c + 1 < C ? __ldg(x + c + 1) : 0.f;
          xent_store<BF16>(grad, ldg, r, c, n_store, xent_grad(v0, m, inv, c, C, lab, grad_scale),
                           xent_grad(v1, m, inv, c + 1, C, lab, grad_scale));
        }
      }
    }
  }
  lsum = warp_sum(lsum);  // fixed lane order
  // deterministic loss: warp sums -> CTA partial (warp order) -> last CTA: thread t sums partials
  // t, t + 256, ... in order, thread 0 the 256 sums in order
  if (lane == 0) red[warp] = lsum;
  __syncthreads();
  if (threadIdx.x == 0) {
    float b = 0.f;
#pragma unroll
    for (int w = 0; w < kXentThreads / 32; ++w) b += red[w];
    partial[blockIdx.x] = b;
    __threadfence();
    const unsigned old = atomicAdd(cnt, 1u);
    last = old + 1 == gridDim.x;
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  // thread t: partials t, t + 256, ... (loads batched 8 deep, summed in order); then a fixed tree
  float t = 0.f;
  for (unsigned i0 = threadIdx.x; i0 < gridDim.x; i0 += 8 * kXentThreads) {
    float pv[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const unsigned i = i0 + u * kXentThreads;
      pv[u] = i < gridDim.x ? __ldcg(partial + i) : 0.f;
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) t += pv[u];
  }
  red[threadIdx.x] = t;
  __syncthreads();
  if (warp == 0) {
    float w8 = 0.f;
#pragma unroll
    for (int i = 0; i < kXentThreads / 32; ++i) w8 += red[lane * (kXentThreads / 32) + i];
    const float tot = warp_sum(w8);
    if (lane == 0) {
      *loss = tot / (float)rows;
      *cnt = 0u;  // the workspace is left as it was found (zeroed counter)
    }
  }
}

}  // namespace hcs

using namespace hcs;

extern "C" int hcs_softmax_xent_workspace_bytes(int64_t rows, size_t* bytes) {
  HCS_REQUIRE(bytes != nullptr && rows >= 0, HCS_EINVAL, "bad softmax cross-entropy shape");
  *bytes = (size_t)(32 + xent_grid(rows)) * sizeof(float);
  return HCS_OK;
}

extern "C" int hcs_softmax_xent(const float* logits, int64_t ld, int64_t rows, int32_t classes,
                                const int64_t* labels, float grad_scale, float* loss, void* grad, int grad_dtype,
                                int64_t ld_grad, int32_t n_store, void* workspace, size_t ws_bytes, void* stream) {
  HCS_REQUIRE(rows > 0 && classes > 0 && ld >= classes, HCS_EINVAL,
              "bad softmax cross-entropy shape (rows %lld, classes %d, ld %lld)", (long long)rows, classes,
              (long long)ld);
  HCS_REQUIRE(n_store >= classes && ld_grad >= n_store, HCS_EINVAL, "gradient needs ld_grad >= n_store >= classes");
  HCS_REQUIRE(grad_dtype == HCS_DTYPE_BF16 || grad_dtype == HCS_DTYPE_F32, HCS_EINVAL,
              "gradient dtype must be bf16 or f32 (got %d)", grad_dtype);
  HCS_REQUIRE(grad_dtype != HCS_DTYPE_BF16 || (n_store % 2 == 0 && ld_grad % 2 == 0 && ((uintptr_t)grad & 3) == 0),
              HCS_EINVAL, "bf16 gradient needs an even n_store and ld_grad and a 4-byte aligned base");
  HCS_REQUIRE(logits != nullptr && labels != nullptr && loss != nullptr && grad != nullptr, HCS_EINVAL, "null buffer");
  const int grid = xent_grid(rows);
  HCS_REQUIRE(workspace != nullptr && ws_bytes >= (size_t)(32 + grid) * sizeof(float), HCS_EINVAL,
              "softmax cross-entropy workspace too small (hcs_softmax_xent_workspace_bytes)");
  unsigned* cnt = static_cast<unsigned*>(workspace);
  float* partial = static_cast<float*>(workspace) + 32;
  cudaStream_t st = as_stream(stream);
  const bool group = classes <= 64 && n_store <= 64;
  const bool vec = ld % 4 == 0 && ((uintptr_t)logits & 15) == 0 &&
                   (grad_dtype != HCS_DTYPE_BF16 || (ld_grad % 8 == 0 && ((uintptr_t)grad & 15) == 0));
  auto kern = grad_dtype == HCS_DTYPE_BF16
                  ? (group ? (vec ? k_softmax_xent<true, true, true> : k_softmax_xent<true, true, false>)
                           : k_softmax_xent<true, false, false>)
                  : (group ? (vec ? k_softmax_xent<false, true, true> : k_softmax_xent<false, true, false>)
                           : k_softmax_xent<false, false, false>);
  kern<<<grid, kXentThreads, 0, st>>>(logits, ld, rows, classes, labels, grad_scale, grad, ld_grad, n_store, partial,
                                      cnt, loss);
  HCS_LAUNCH_CHECK("k_softmax_xent");
  return HCS_OK;
}
