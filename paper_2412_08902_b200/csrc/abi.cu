// C-ABI plumbing: thread-local error state, device queries, tensor-map encoding,
// and small elementwise helpers.
#include <cudaTypedefs.h>
#include <cstdarg>
#include <cstring>
#include <mutex>

#include "common.cuh"

namespace hcs {

static thread_local char g_err[1024] = "";

int set_error(int code, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
  return code;
}

int cuda_status(cudaError_t e, const char* what) {
  return set_error(HCS_ECUDA, "CUDA error in %s: %s", what, cudaGetErrorString(e));
}

int num_sms() {
  static int sms = 0;
  if (sms == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (sms <= 0) sms = 148;
  }
  return sms;
}

static PFN_cuTensorMapEncodeTiled_v12000 g_encode = nullptr;
static std::once_flag g_encode_once;

int encode_tiled_2d(CUtensorMap* tm, CUtensorMapDataType dt, void* base, uint64_t inner, uint64_t outer,
                    uint64_t row_stride_bytes, uint32_t box_inner, uint32_t box_outer, CUtensorMapSwizzle sw) {
  std::call_once(g_encode_once, [] {
    cudaDriverEntryPointQueryResult q;
    void* fn = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      g_encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  });
  HCS_REQUIRE(g_encode != nullptr, HCS_ECUDA, "cuTensorMapEncodeTiled unavailable");
  cuuint64_t gdim[2] = {inner, outer};
  cuuint64_t gstride[1] = {row_stride_bytes};
  cuuint32_t box[2] = {box_inner, box_outer};
  cuuint32_t es[2] = {1, 1};
  CUresult r = g_encode(tm, dt, 2, base, gdim, gstride, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, sw,
                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  HCS_REQUIRE(r == CUDA_SUCCESS, HCS_ECUDA, "cuTensorMapEncodeTiled failed (%d)", (int)r);
  return HCS_OK;
}

__global__ void k_convert(const float* __restrict__ src, void* __restrict__ dst, int64_t n, int kind) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (; i < n; i += stride) {
    float v = src[i];
    if (kind == HCS_DTYPE_BF16) {
      reinterpret_cast<__nv_bfloat16*>(dst)[i] = __float2bfloat16_rn(v);
    } else {
      uint32_t t;
      asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(t) : "f"(v));
      reinterpret_cast<float*>(dst)[i] = __uint_as_float(t);
    }
  }
}

}  // namespace hcs

extern "C" {

int hcs_version(void) { return 100; }
const char* hcs_last_error(void) { return hcs::g_err; }
int hcs_device_sm_count(void) { return hcs::num_sms(); }

int hcs_convert(const float* src, void* dst, int64_t n, int dst_kind, void* stream) {
  HCS_REQUIRE(n >= 0, HCS_EINVAL, "negative length");
  if (n == 0) return HCS_OK;
  int grid = (int)std::min<int64_t>((n + 255) / 256, (int64_t)hcs::num_sms() * 16);
  hcs::k_convert<<<grid, 256, 0, hcs::as_stream(stream)>>>(src, dst, n, dst_kind);
  HCS_LAUNCH_CHECK("hcs_convert");
  return HCS_OK;
}

}  // extern "C"
