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
#include <condition_variable>
#include <cstdint>
#include <cstring>
#include <functional>
#include <mutex>
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

// Persistent worker threads: a staged operand is converted in several blocks per call, and
// starting threads per block cost more than the conversion of a small block (16 threads x 8 blocks
// of a C2 operand: ~2 ms of thread start-up, tools/exp_dropin.py).  run(n, fn) calls fn(0..n-1),
// fn(0) on the caller; calls are serialised.
class Pool {
 public:
  void run(int n, const std::function<void(int)>& fn) {
    std::lock_guard<std::mutex> serial(call_mu_);
    {
      std::unique_lock<std::mutex> lk(mu_);
      while ((int)workers_.size() < n - 1) {
        const int id = (int)workers_.size() + 1;
        workers_.emplace_back([this, id] { loop(id); });
      }
      job_ = &fn;
      active_ = n;
      pending_ = n - 1;
      ++gen_;
    }
    cv_.notify_all();
    fn(0);
    std::unique_lock<std::mutex> lk(mu_);
    done_.wait(lk, [this] { return pending_ == 0; });
    job_ = nullptr;
  }
  ~Pool() {
    {
      std::lock_guard<std::mutex> lk(mu_);
      stop_ = true;
      ++gen_;
    }
    cv_.notify_all();
    for (auto& t : workers_) t.join();
  }

 private:
  void loop(int id) {
    uint64_t seen = 0;
    for (;;) {
      const std::function<void(int)>* job;
      {
        std::unique_lock<std::mutex> lk(mu_);
        cv_.wait(lk, [&] { return gen_ != seen; });
        seen = gen_;
        if (stop_) return;
        if (id >= active_) continue;
        job = job_;
      }
      (*job)(id);
      {
        std::lock_guard<std::mutex> lk(mu_);
        if (--pending_ == 0) done_.notify_one();
      }
    }
  }
  std::mutex call_mu_, mu_;
  std::condition_variable cv_, done_;
  std::vector<std::thread> workers_;
  const std::function<void(int)>* job_ = nullptr;
  uint64_t gen_ = 0;
  int active_ = 0, pending_ = 0;
  bool stop_ = false;
};

Pool& pool() {
  static Pool* p = new Pool();  // never destroyed: workers may outlive static destruction order
  return *p;
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
  pool().run(nt, [&](int t) {
    convert_rows(src, ld_src, rows * t / nt, rows * (t + 1) / nt, dim, dst, ld_dst, out_dtype);
  });
  return HCS_OK;
}
