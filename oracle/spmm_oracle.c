/* Exact float64 SpMM for full-size parity checks -- TEST INFRASTRUCTURE ONLY.
 *
 * Z = A X with every product and sum in float64, CSR order per row: the role of the
 * reference's dense oracle spmm_dense_oracle (/root/reference/pkg/src/rowwin/matrices.py:321-325)
 * and of rowwin_oracle.spmm_exact, at sizes (C2: 115 M entries x 128 features) where numpy's
 * gather-then-reduceat would need ~120 GB of temporaries.  Rows are split into contiguous blocks
 * over `nthreads` pthreads; each row is summed by one thread in CSR order, so the result does not
 * depend on the thread count.  X and Z are row-major float64 with leading dimensions ldx / ldz.
 * Only tests/ may call it (see oracle/rowwin_oracle.py header).
 */
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef struct {
  const int64_t* rp;
  const int32_t* ci;
  const double* val;
  const double* x;
  double* z;
  int64_t r0, r1, ldx, ldz;
  int32_t dim;
} spmm_job;

static void* spmm_rows(void* arg) {
  const spmm_job* j = (const spmm_job*)arg;
  for (int64_t r = j->r0; r < j->r1; ++r) {
    double* zr = j->z + r * j->ldz;
    memset(zr, 0, sizeof(double) * (size_t)j->dim);
    for (int64_t e = j->rp[r]; e < j->rp[r + 1]; ++e) {
      const double v = j->val[e];
      const double* xr = j->x + (int64_t)j->ci[e] * j->ldx;
      for (int32_t f = 0; f < j->dim; ++f) zr[f] += v * xr[f];
    }
  }
  return 0;
}

int oracle_spmm_f64(const int64_t* rp, const int32_t* ci, const double* val, int64_t n_rows, const double* x,
                    int64_t ldx, int32_t dim, double* z, int64_t ldz, int32_t nthreads) {
  if (nthreads < 1) nthreads = 1;
  if (nthreads > 256) nthreads = 256;
  pthread_t th[256];
  spmm_job jobs[256];
  const int64_t nnz = rp[n_rows] - rp[0];
  /* equal-entry blocks: thread t starts at the first row whose prefix reaches t * nnz / T */
  int64_t r = 0;
  for (int32_t t = 0; t < nthreads; ++t) {
    const int64_t target = rp[0] + (nnz * (t + 1)) / nthreads;
    int64_t r1 = r;
    while (r1 < n_rows && rp[r1] < target) ++r1;
    if (t == nthreads - 1) r1 = n_rows;
    jobs[t] = (spmm_job){rp, ci, val, x, z, r, r1, ldx, ldz, dim};
    r = r1;
  }
  int32_t started = 0;
  char threaded[256];
  for (int32_t t = 0; t < nthreads; ++t) {
    threaded[t] = pthread_create(&th[t], 0, spmm_rows, &jobs[t]) == 0;
    if (!threaded[t]) spmm_rows(&jobs[t]); /* no thread available: run the block inline */
    started += threaded[t];
  }
  for (int32_t t = 0; t < nthreads; ++t)
    if (threaded[t]) pthread_join(th[t], 0);
  return started;
}
