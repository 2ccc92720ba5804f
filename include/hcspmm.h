/*
 * hcspmm.h -- C ABI of libhcspmm.so, the B200 (sm_100a) HC-SpMM hot path.
 *
 * Every entry point takes plain device pointers, sizes and a cudaStream_t
 * (passed as void*), is stream-ordered, never allocates user-visible memory,
 * and returns an HCS_* status; hcs_last_error() gives the thread-local message.
 * The Python package paper_2412_08902_b200 binds these with ctypes and maps
 * the status codes onto the reference's exception classes (ValueError /
 * InvariantError), see paper_2412_08902_b200/_lib.py.
 *
 * The reference (rowwin, /root/reference/pkg/src/rowwin) has no FFI layer;
 * each function below names the reference Python function(s) it replaces.
 */
#ifndef HCSPMM_H_
#define HCSPMM_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define HCS_OK 0
#define HCS_EINVAL 1     /* bad argument                 -> ValueError     */
#define HCS_EDIM 2       /* dimension mismatch           -> ValueError     */
#define HCS_EINVARIANT 3 /* internal consistency failure -> InvariantError */
#define HCS_ECUDA 4      /* CUDA runtime / launch error  -> RuntimeError   */
#define HCS_ENCCL 5      /* collective failure           -> RuntimeError   */

#define HCS_DTYPE_F32 0
#define HCS_DTYPE_BF16 1

int hcs_version(void);
const char* hcs_last_error(void);
int hcs_device_sm_count(void);

/* ---------------------------------------------------------------- K1
 * windows.py:81-106 partition + windows.py:109-123 features +
 * selector.py:48-64 SelectorModel.score/decide + classify_windows.
 * Window w covers rows [w*wh, min((w+1)*wh, n_rows)); W = ceil(n_rows/wh).
 * selector: HOST pointer to the 7 doubles {w_ncols, w_density, bias, mean0, mean1,
 * scale0, scale1} (data/selector_default.json) or NULL to skip classification.
 * Two phases sharing one caller-owned workspace:
 *   count: win_col_ptr[W+1] (exclusive prefix of ncols), density[W], ci[W], codes[W]
 *   fill : nonzero_cols[win_col_ptr[W]] (ascending per window), cond_cols[nnz]
 * Bit-exact with the reference (integer outputs; features/decisions in IEEE fp64). */
int hcs_partition_workspace_bytes(int64_t n_rows, int64_t n_cols, int64_t nnz, int32_t wh, size_t* bytes);
int hcs_partition_count(const int64_t* row_ptr, const int32_t* col_idx, int64_t n_rows, int64_t n_cols, int64_t nnz,
                        int32_t wh, const double* selector, int64_t* win_col_ptr, double* density, double* ci,
                        uint8_t* codes, void* workspace, size_t ws_bytes, void* stream);
int hcs_partition_fill(const int64_t* row_ptr, const int32_t* col_idx, int64_t n_rows, int64_t n_cols, int64_t nnz,
                       int32_t wh, const int64_t* win_col_ptr, int32_t* nonzero_cols, int32_t* cond_cols,
                       void* workspace, size_t ws_bytes, void* stream);
/* selector.py:48-56 on caller-given features (classify_windows with a non-default model);
 * selector is a HOST pointer to the 7 doubles, the other pointers are device memory. */
int hcs_classify(const int64_t* win_col_ptr, const double* density, int64_t n_windows, const double* selector,
                 uint8_t* codes, void* stream);

/* ---------------------------------------------------------------- K2
 * Execution plan for the TILE windows of executors.py:160-188 _run_windows:
 * packs each TILE window's entries into 64-column chunks for the tensor-core
 * kernel.  tile_list: T window ids (schedule order); chunk_ptr[T+1] (chunks of
 * 64 condensed columns per window, exclusive prefix); gidx[nchunks*64] gather
 * row per chunk slot (-1 = padding, zero-filled in shared memory);
 * ent_ptr[nchunks+1]; ent[nnz_tile] packed (bf16 value << 16 | slab position
 * r*64+c) for HCS_DTYPE_BF16, or {pos, fp32 bits} pairs (uint64) for F32. */
int hcs_tile_plan_workspace_bytes(int64_t nnz_tile, int64_t nchunks, size_t* bytes);
/* ---------------------------------------------------------------- host ingestion
 * matrices.py:175-307 (load_matrix_market / parse_edge_list): multi-threaded parse of the
 * entry lines from byte `offset` (kind 0: Matrix Market entries, `expected` = 2 pattern or 3
 * fields; kind 1: 'u v' edge list).  A strict subset of the reference grammar; *irregular = 1
 * means "re-parse with the reference rules" (exact FormatError messages and line numbers).
 * nthreads <= 0: all hardware threads.  a/b: row,col (1-based as written) or u,v; v: values. */
int hcs_io_count(const char* path, int64_t offset, int kind, int nthreads, int64_t* count, int* irregular);
int hcs_io_parse(const char* path, int64_t offset, int kind, int expected, int64_t count, int nthreads, int64_t* a,
                 int64_t* b, double* v, int* irregular);
/* matrices.py:126-149 DenseMatrix (float64, row-major) staged for the device: rows [0, rows) of a
 * host float64 matrix converted by `threads` host threads (<= 0: all) into host memory `dst`
 * (typically pinned) as bf16 (out_dtype HCS_DTYPE_BF16; torch's double -> float -> bfloat16
 * rounding, bit for bit) or fp32 (HCS_DTYPE_F32), leading dimension ld_dst >= dim, padding
 * columns zeroed.  The drop-in spmm_hybrid(DenseMatrix) call pipelines it with the H2D copy. */
int hcs_host_convert_f64(const double* src, int64_t rows, int64_t dim, int64_t ld_src, void* dst, int64_t ld_dst,
                         int out_dtype, int threads);

/* plan builder: 0 (default) = per-window stable bucketing by chunk, 1 = global radix sort on
 * (chunk, row, column); both produce identical plans */
int hcs_set_tile_plan_builder(int builder);
int hcs_tile_plan(const int64_t* row_ptr, const int32_t* cond_cols, const void* values, int values_dtype,
                  const int64_t* win_col_ptr, const int32_t* nonzero_cols, int64_t n_rows, int64_t n_cols, int32_t wh,
                  const int32_t* tile_list, int64_t n_tile, const int64_t* chunk_ptr, int64_t nchunks,
                  int32_t* gidx, int64_t* ent_ptr, void* ent, int ent_dtype, int64_t nnz_tile,
                  void* workspace, size_t ws_bytes, void* stream);

/* ---------------------------------------------------------------- K3
 * executors.py:100-108 scalar_window (per window list) and 191-213
 * spmm_scalar (pass all windows).  One warp per row, 128-bit X loads, fp32
 * accumulation, fixed-order warp-shuffle reduction (deterministic).
 * x: [*, ldx] (dtype x_dtype); z: fp32 [n_rows, ldz]; window rows beyond the
 * listed windows are untouched; listed empty windows are zero-filled. */
int hcs_spmm_scalar(const int64_t* row_ptr, const int32_t* col_idx, const void* values, int values_dtype,
                    int64_t n_rows, int32_t wh, const int32_t* win_list, int64_t n_list, const void* x, int x_dtype,
                    int64_t x_rows, int32_t dim, int64_t ldx, float* z, int64_t ldz, void* stream);
/* K3 kernel choice: 0 auto (warp per window, col/val staged in shared memory, 32-byte X
 * vectors when rows are 32-byte aligned and padded), 1 block per window (8 warps, one row
 * each, lane groups reduced by a fixed shuffle tree), 2 warp per window with 16-byte vectors.
 * Window heights > 31 always use variant 1.  Every variant is deterministic. */
int hcs_set_scalar_variant(int variant);

/* K3 for small plans (executors.HybridPlan, <= 1,024 scalar windows): one warp per piece of <= 32
 * entries of a row of the listed windows, so a hub row is spread over many warps.  Pieces of a row
 * are consecutive: p_first = the row's first piece, p_count = its pieces, p_k = [k0, k1) entry
 * range per piece (2 int64), p_row = output row.  A row of one piece is stored directly; the last
 * piece of a longer row to finish sums the partials (slots: npieces x ld_slot floats) in piece
 * order.  cnt: npieces uint32, zero before first use and left zero; one (slots, cnt) workspace
 * must not be shared by concurrent launches. */
int hcs_spmm_scalar_pieces(const int32_t* col_idx, const void* values, int values_dtype, const int32_t* p_row,
                           const int64_t* p_k, const int32_t* p_first, const int32_t* p_count, int64_t npieces,
                           const void* x, int x_dtype, int32_t dim, int64_t ldx, float* z, int64_t ldz, float* slots,
                           int64_t ld_slot, unsigned* cnt, void* stream);

/* ---------------------------------------------------------------- K4
 * executors.py:111-141 tile_window for every window of a tile plan, on warp-independent
 * workers: each warp owns a balanced range of (window, feature slice, 64-column chunk) work
 * with its own cp.async ring and mma.sync (bf16 m16n8k16, or tf32 m16n8k8 for an fp32 plan),
 * fp32 register accumulators; windows cut by a warp boundary are summed in warp order by the
 * last of their warps to finish (completion counters in the workspace), so results are
 * deterministic and one product is one launch.  (Round 1's warp-specialised tcgen05 / mma.sync
 * pipeline engines and its fix-up launch were removed in round 2: DESIGN.md section 4.)
 * workspace: >= hcs_tile_scratch_floats() floats: split-window completion counters followed by
 * partial sums.  It must be ZEROED before its first use (the kernels leave the counters zero
 * again), and one workspace must not be shared by launches that can run concurrently. */
int hcs_tile_scratch_floats(int64_t* floats);
/* tile kernel row-slice width in 16-B vectors: 0 auto (8 for dim > 32, else 4), 4 or 8 */
int hcs_set_tile_slice(int vectors);
/* tile kernel fused GCN epilogue, one 33..48-feature slice: 1 (default) = kernel that skips the
 * empty 16-feature group, 0 = the full 64-feature kernel (experiment switch) */
int hcs_set_tile_npr3(int on);
/* tile kernel with > 1 feature slice: 1 (default) = the FS warps of a group walk the same
 * (window, chunk) range, one slice each (plan read once, an X row's slices fetched together);
 * 0 = one warp per contiguous range of (window, slice, chunk); 2 = 1 only when X exceeds 96 MB.
 * All deterministic. */
int hcs_set_tile_pairing(int on);
/* CTAs per tile launch: 0 = one per SM (default), n > 0 = min(n, SMs) -- the multi-GPU runs leave
 * SMs to the NCCL kernels of the overlapped exchange (a tile CTA fills its SM's shared memory) */
int hcs_set_tile_grid(int ctas);
int hcs_spmm_tile(const int32_t* tile_list, int64_t n_tile, const int64_t* chunk_ptr, const int32_t* gidx,
                  const int64_t* ent_ptr, const void* ent, int ent_dtype, int64_t n_rows, int32_t wh, const void* x,
                  int x_dtype, int64_t x_rows, int32_t dim, int64_t ldx, float* z, int64_t ldz, void* workspace,
                  size_t ws_bytes, void* stream);
/* hcs_spmm_tile with the warps' chunk ranges weighted by cost = alpha * chunks + entries instead of
 * equal chunk counts (alpha > 0; 0 = hcs_spmm_tile).  Skewed plans (hub windows whose chunks hold
 * hundreds of entries, e.g. R-MAT) otherwise leave the first warps with ~1.8x the mean work.  One
 * small extra launch (k_tile_bounds: one 32-way warp search per range boundary, into the
 * workspace) for plans of >= 8 tile windows per warp group; deterministic for a given alpha.
 * n_chunks > 0: the launched range holds that many 64-column chunks (chunk_ptr[n_tile] - chunk_ptr[0],
 * known to the plan's owner), and the grid shrinks to keep one chunk position per warp group: a
 * small plan then does not occupy every SM (C1: 10.25 -> 8.22 us); 0 = one CTA per SM. */
int hcs_spmm_tile_balanced(const int32_t* tile_list, int64_t n_tile, const int64_t* chunk_ptr, const int32_t* gidx,
                           const int64_t* ent_ptr, const void* ent, int ent_dtype, int64_t n_rows, int32_t wh,
                           const void* x, int x_dtype, int64_t x_rows, int32_t dim, int64_t ldx, float* z, int64_t ldz,
                           void* workspace, size_t ws_bytes, int alpha, int64_t n_chunks, void* stream);

/* ---------------------------------------------------------------- K6 / K7
 * gnn.py:121-159 forward (fused mode) and gnn.py:162-205 backward (fused mode):
 * the SpMM of the listed windows with the feature GEMM fused into the window
 * epilogue:  out[rows] = (A_w X) M,  and z[rows] = A_w X when z != NULL
 * (forward z_cache).  M is an fp32 [dim x d_out] row-major device matrix: W for the
 * forward, W^T for the backward grad_X = (A^T G) W^T.
 * hcs_gcn_tile takes the tile plan of K2 and the K4 workspace (hcs_tile_scratch_floats);
 * d_out <= 64; bf16 plan: dim <= 128 (M^T staged in shared memory as bf16); fp32 plan (tf32):
 * any dim, M RNA-rounded to tf32 by the caller.  Window partials cut by warp ranges are summed
 * in warp order.  hcs_gcn_scalar takes a window list; dim, d_out <= 128.  Larger shapes run
 * unfused: SpMM, then hcs_gemm. */
int hcs_gcn_tile(const int32_t* tile_list, int64_t n_tile, const int64_t* chunk_ptr, const int32_t* gidx,
                 const int64_t* ent_ptr, const void* ent, int ent_dtype, int64_t n_rows, int32_t wh, const void* x,
                 int x_dtype, int64_t x_rows, int32_t dim, int64_t ldx, float* z, int64_t ldz, const float* m,
                 int32_t d_out, float* out, int64_t ldo, void* workspace, size_t ws_bytes, void* stream);
int hcs_gcn_scalar(const int64_t* row_ptr, const int32_t* col_idx, const void* values, int values_dtype,
                   int64_t n_rows, int32_t wh, const int32_t* win_list, int64_t n_list, const void* x, int x_dtype,
                   int64_t x_rows, int32_t dim, int64_t ldx, float* z, int64_t ldz, const float* m, int32_t d_out,
                   float* out, int64_t ldo, void* stream);

/* ---------------------------------------------------------------- K7 grad_W + dense update
 * gnn.py:188 (unfused) / 195-199 (fused, ascending-window accumulation): grad_W = Z^T G.
 * hcs_grad_w: C[M x N] = A^T B for A [K x M] (z_cache), B [K x N] (grad_out), fp32 row-major
 * (lda, ldb multiples of 4, 16-byte aligned); deterministic split-K over K (fixed row slices,
 * partials summed in slice order by a second launch), mma.sync tf32 (RNA) with fp32 accumulate.
 * workspace: hcs_grad_w_workspace_bytes(K, M, N).
 * hcs_gemm: C[K x N] = A[K x M] B[M x N] (gnn.py:142-143, 189, 202 -- the x_next = Z W and
 * G W^T updates of the unfused mode and of shapes beyond the fused epilogues), same numerics. */
int hcs_grad_w_workspace_bytes(int64_t K, int32_t M, int32_t N, size_t* bytes);
int hcs_grad_w(const float* a, int64_t lda, const float* b, int64_t ldb, int64_t K, int32_t M, int32_t N, float* c,
               int64_t ldc, void* workspace, size_t ws_bytes, void* stream);
int hcs_gemm(const float* a, int64_t lda, const float* b, int64_t ldb, int64_t K, int32_t M, int32_t N, float* c,
             int64_t ldc, void* stream);
/* hcs_gemm with a bf16 destination that is the next aggregation's operand (model.Gcn2's
 * update-first layers, A (X W)): C[K x n_store] = bf16_rne((A B) * 1[mask > 0]) for columns < N
 * (mask: optional fp32 [K x N], ld_mask -- the ReLU backward, grad * 1[H > 0]), zeros for columns
 * [N, n_store) (rows padded to whole gather slices).  n_store, ldc even. */
int hcs_gemm_bf16(const float* a, int64_t lda, const float* b, int64_t ldb, int64_t K, int32_t M, int32_t N, void* c,
                  int64_t ldc, int32_t n_store, const float* mask, int64_t ld_mask, void* stream);

/* ---------------------------------------------------------------- training-epoch loss (C3)
 * Not in the reference (its GCN has no loss or optimizer): the C3 epoch's softmax
 * cross-entropy.  *loss = -mean_i log_softmax(logits_i)[labels_i] (device float, reduced in a
 * fixed order); grad [rows x n_store] (ld_grad; bf16 or f32) = grad_scale * (softmax(logits_i) -
 * onehot(labels_i)) for columns < classes, zeros up to n_store.  labels: int64 [rows]; a label
 * outside [0, classes) makes the loss NaN.  workspace: hcs_softmax_xent_workspace_bytes(rows),
 * zero-filled before first use (left zeroed). */
int hcs_softmax_xent_workspace_bytes(int64_t rows, size_t* bytes);
int hcs_softmax_xent(const float* logits, int64_t ld, int64_t rows, int32_t classes, const int64_t* labels,
                     float grad_scale, float* loss, void* grad, int grad_dtype, int64_t ld_grad, int32_t n_store,
                     void* workspace, size_t ws_bytes, void* stream);

/* ---------------------------------------------------------------- K8 LOA
 * layout.py:186-263 build_windows_optimized (paper Alg. 6): greedy 16-vertex groups
 * maximising the window's entries-per-column ratio.  order: the sort_by_min_neighbor
 * permutation (layout.py:99-109, int32 [n], device); outputs out_order int32 [n]
 * (groups concatenated), gptr int64 [n+1] (group offsets) and *ngroups (device
 * int64).  One persistent CTA runs the sequential loop; bit-exact with the reference.
 * workspace: hcs_loa_workspace_bytes (global bitmaps when n is too large for smem). */
int hcs_loa_workspace_bytes(int64_t n, size_t* bytes);
int hcs_loa(const int64_t* row_ptr, const int32_t* col_idx, int64_t n, int32_t vw, int32_t group_size,
            const int32_t* order, int32_t* out_order, int64_t* gptr, int64_t* ngroups, void* workspace,
            size_t ws_bytes, void* stream);

/* ---------------------------------------------------------------- normalisation
 * gnn.py:68-95 normalize_adj values in float64 with the reference's operation
 * order (structure of A + I assembled by the caller).  kind 0 = gcn
 * ((v * d_r^-1/2) * d_c^-1/2, d = row sums in entry order), 1 = row (v / deg).
 * v_out32 (optional) receives the float32 copy used by the kernels. */
int hcs_normalize_values(int kind, const int64_t* row_ptr, const int32_t* col, const double* v_in, int64_t n,
                         double* workspace_deg, double* v_out, float* v_out32, void* stream);

/* elementwise helpers used by the Python layer (fp32 -> bf16 RNE, fp32 -> tf32 RNA) */
int hcs_convert(const float* src, void* dst, int64_t n, int dst_kind, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* HCSPMM_H_ */
