// Host staging of reference-typed operands (the drop-in call): a rowwin caller passes X as a
// float64 row-major DenseMatrix (reference matrices.py:126-149), 238 MB at C2 / N = 128.  Copying
// that pageable array to the device and converting there took 25 ms end to end (the driver
// stages pageable memory at ~10 GB/s); here host threads convert row blocks straight into a
// pinned staging buffer in the compute dtype (4x fewer bytes for bf16), so the H2D copy of one
// block overlaps the conversion of the next (executors.stage_operand drives the pipeline).
//
// Rounding matches torch's double -> bfloat16 cast bit for bit (c10: double -> float, RNE, then
// float -> bfloat16, RNE; NaN -> 0x7fc0), so the staged operand equals what the device-side
// conversion of the same array produces (tests/test_abi_host.py; NaN payloads aside).
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <thread>
#include <vector>

#include "common.cuh"

namespace {

inline uint16_t f32_to_bf16_rne(float f) {
  uint32_t u;
  std::memcpy(&u, &f, 4);
  if ((u & 0x7fffffffu) > 0x7f800000u) return 0x7fc0u;  // NaN: c10's canonical quiet NaN
  const uint32_t lsb = (u >> 16) & 1u;
  u += 0x7fffu + lsb;
  return (uint16_t)(u >> 16);
}

// rows [r0, r1): dst row r = dim converted values, then zeros up to ld_dst
void convert_rows(const double* src, int64_t ld_src, int64_t r0, int64_t r1, int64_t dim, void* dst, int64_t ld_dst,
                  int out_dtype) {
  if (out_dtype == HCS_DTYPE_BF16) {
    uint16_t* d = static_cast<uint16_t*>(dst);
    for (int64_t r = r0; r < r1; ++r) {
      const double* s = src + r * ld_src;
      uint16_t* o = d + r * ld_dst;
      for (int64_t c = 0; c < dim; ++c) o[c] = f32_to_bf16_rne((float)s[c]);
      for (int64_t c = dim; c < ld_dst; ++c) o[c] = 0;
    }
  } else {
    float* d = static_cast<float*>(dst);
    for (int64_t r = r0; r < r1; ++r) {
      const double* s = src + r * ld_src;
      float* o = d + r * ld_dst;
      for (int64_t c = 0; c < dim; ++c) o[c] = (float)s[c];
      for (int64_t c = dim; c < ld_dst; ++c) o[c] = 0.f;
    }
  }
}

}  // namespace

// Converts rows [0, rows) of a row-major float64 host matrix (leading dimension ld_src) into dst
// (host memory, typically pinned; leading dimension ld_dst >= dim, padding columns zeroed) as
// bf16 (HCS_DTYPE_BF16) or fp32 (HCS_DTYPE_F32), with `threads` host threads (<= 0: all cores).
extern "C" int hcs_host_convert_f64(const double* src, int64_t rows, int64_t dim, int64_t ld_src, void* dst,
                                    int64_t ld_dst, int out_dtype, int threads) {
  HCS_REQUIRE(rows >= 0 && dim >= 0, HCS_EINVAL, "rows and dim must be non-negative");
  HCS_REQUIRE(ld_src >= dim && ld_dst >= dim, HCS_EINVAL, "leading dimensions must cover dim");
  HCS_REQUIRE(out_dtype == HCS_DTYPE_BF16 || out_dtype == HCS_DTYPE_F32, HCS_EINVAL,
              "out_dtype must be bf16 or f32 (got %d)", out_dtype);
  HCS_REQUIRE(rows == 0 || (src != nullptr && dst != nullptr), HCS_EINVAL, "null buffer");
  if (rows == 0) return HCS_OK;
  int nt = threads > 0 ? threads : (int)std::max(1u, std::thread::hardware_concurrency());
  // at least ~256 KB of input per thread (thread start-up is ~10-20 us)
  const int64_t per = std::max<int64_t>(1, (int64_t)(262144 / 8) / std::max<int64_t>(dim, 1));
  nt = (int)std::max<int64_t>(1, std::min<int64_t>(nt, (rows + per - 1) / per));
  if (nt == 1) {
    convert_rows(src, ld_src, 0, rows, dim, dst, ld_dst, out_dtype);
    return HCS_OK;
  }
  std::vector<std::thread> pool;
  pool.reserve(nt - 1);
  for (int t = 1; t < nt; ++t) {
    const int64_t r0 = rows * t / nt, r1 = rows * (t + 1) / nt;
    pool.emplace_back(convert_rows, src, ld_src, r0, r1, dim, dst, ld_dst, out_dtype);
  }
  convert_rows(src, ld_src, 0, rows / nt, dim, dst, ld_dst, out_dtype);
  for (auto& th : pool) th.join();
  return HCS_OK;
}
