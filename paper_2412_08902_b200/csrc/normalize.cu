// Aggregation-operator normalisation values (reference gnn.py:68-95 normalize_adj).
// The sparsity structure (A + I with duplicates merged) is assembled by the
// caller; these kernels compute the float64 values with the reference's exact
// operation order so the normalised operator is bit-identical:
//   gcn: deg[r] = sum of row r in entry order (np.add.at, gnn.py:93);
//        inv = 1.0 / sqrt(deg) (two correctly rounded ops, gnn.py:94);
//        v' = (v * inv[r]) * inv[c]                       (gnn.py:95)
//   row: scale = deg > 0 ? 1.0 / deg : 0 with deg = entry count (gnn.py:80-83)
#include "common.cuh"

namespace hcs {

__global__ void k_row_sum_f64(const int64_t* __restrict__ row_ptr, const double* __restrict__ v, int64_t n,
                              double* __restrict__ out) {
  int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (r >= n) return;
  double s = 0.0;
  for (int64_t e = row_ptr[r]; e < row_ptr[r + 1]; ++e) s = __dadd_rn(s, v[e]);
  out[r] = s;
}

__global__ void k_gcn_scale(const int64_t* __restrict__ row_ptr, const int32_t* __restrict__ col,
                            const double* __restrict__ v, const double* __restrict__ deg, int64_t n,
                            double* __restrict__ out, float* __restrict__ out32) {
  int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  int lane = threadIdx.x & 31;
  for (int64_t r = warp; r < n; r += nw) {
    double ir = __ddiv_rn(1.0, __dsqrt_rn(deg[r]));
    for (int64_t e = row_ptr[r] + lane; e < row_ptr[r + 1]; e += 32) {
      double ic = __ddiv_rn(1.0, __dsqrt_rn(deg[col[e]]));
      double x = __dmul_rn(__dmul_rn(v[e], ir), ic);
      out[e] = x;
      if (out32) out32[e] = (float)x;
    }
  }
}

__global__ void k_row_scale(const int64_t* __restrict__ row_ptr, const double* __restrict__ v, int64_t n,
                            double* __restrict__ out, float* __restrict__ out32) {
  int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  int lane = threadIdx.x & 31;
  for (int64_t r = warp; r < n; r += nw) {
    int64_t d = row_ptr[r + 1] - row_ptr[r];
    double s = d > 0 ? __ddiv_rn(1.0, (double)d) : 0.0;
    for (int64_t e = row_ptr[r] + lane; e < row_ptr[r + 1]; e += 32) {
      double x = __dmul_rn(v[e], s);
      out[e] = x;
      if (out32) out32[e] = (float)x;
    }
  }
}

}  // namespace hcs

using namespace hcs;

extern "C" int hcs_normalize_values(int kind, const int64_t* row_ptr, const int32_t* col, const double* v_in,
                                    int64_t n, double* workspace_deg, double* v_out, float* v_out32, void* stream) {
  HCS_REQUIRE(kind == 0 || kind == 1, HCS_EINVAL, "kind must be 0 (gcn) or 1 (row)");
  if (n == 0) return HCS_OK;
  cudaStream_t st = as_stream(stream);
  int grid = (int)std::min<int64_t>((n * 32 + 255) / 256, (int64_t)num_sms() * 16);
  if (kind == 0) {
    HCS_REQUIRE(workspace_deg != nullptr, HCS_EINVAL, "degree workspace is NULL");
    k_row_sum_f64<<<(int)((n + 255) / 256), 256, 0, st>>>(row_ptr, v_in, n, workspace_deg);
    HCS_LAUNCH_CHECK("k_row_sum_f64");
    k_gcn_scale<<<grid, 256, 0, st>>>(row_ptr, col, v_in, workspace_deg, n, v_out, v_out32);
    HCS_LAUNCH_CHECK("k_gcn_scale");
  } else {
    k_row_scale<<<grid, 256, 0, st>>>(row_ptr, v_in, n, v_out, v_out32);
    HCS_LAUNCH_CHECK("k_row_scale");
  }
  return HCS_OK;
}
