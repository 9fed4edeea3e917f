/* CPU oracle kernels (TEST INFRASTRUCTURE ONLY).
 *
 * Restates, in plain C, the compiled part of the reference hot path:
 *   - csr._apply_kernel        /root/reference/pkg/src/trihalo/csr.py:143-156
 *     (rows -> nnz -> u with the u loop innermost, accumulator per row)
 *   - HaloExchange.run         /root/reference/pkg/src/trihalo/schemes.py:185-202
 *     (isfinite over the whole source, np.take gather, kernel, np.take scatter)
 *   - linear.tensor_contract   /root/reference/pkg/src/trihalo/linear.py:115-151
 *     (three dense per-axis contractions, normal then t1 then t2)
 * Only tests/, __graft_entry__.smoke() and bench.py's CPU legs call this.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

void oracle_csr_apply(const int64_t* row_offsets, const int64_t* col_indices, const double* values,
                      int64_t n_rows, const double* src, double* out, int64_t u, double* acc) {
  for (int64_t r = 0; r < n_rows; ++r) {
    for (int64_t c = 0; c < u; ++c) acc[c] = 0.0;
    for (int64_t t = row_offsets[r]; t < row_offsets[r + 1]; ++t) {
      const double w = values[t];
      const double* s = src + col_indices[t] * u;
      for (int64_t c = 0; c < u; ++c) acc[c] += w * s[c];
    }
    double* o = out + r * u;
    for (int64_t c = 0; c < u; ++c) o[c] = acc[c];
  }
}

static int all_finite(const double* v, int64_t n) {
  for (int64_t i = 0; i < n; ++i)
    if (!isfinite(v[i])) return 0;
  return 1;
}

/* one dense contraction along the innermost "cell" axis of a (outer, n, u)
 * block: out(outer, m, u) = mat(m, n) @ in(outer, n, u) */
static void contract(const double* mat, int64_t m, int64_t n, const double* in, int64_t outer,
                     int64_t u, double* out) {
  for (int64_t o = 0; o < outer; ++o) {
    const double* ib = in + o * n * u;
    double* ob = out + o * m * u;
    for (int64_t i = 0; i < m; ++i) {
      double* orow = ob + i * u;
      for (int64_t c = 0; c < u; ++c) orow[c] = 0.0;
      for (int64_t j = 0; j < n; ++j) {
        const double w = mat[i * n + j];
        const double* irow = ib + j * u;
        for (int64_t c = 0; c < u; ++c) orow[c] += w * irow[c];
      }
    }
  }
}

/* (a, b, c, u) -> (b, a, c, u) block transpose helper for the axis rotations
 * of tensor_contract: swaps the two leading axes given (A, B, inner) */
static void swap01(const double* in, int64_t A, int64_t B, int64_t inner, double* out) {
  for (int64_t a = 0; a < A; ++a)
    for (int64_t b = 0; b < B; ++b)
      memcpy(out + (b * A + a) * inner, in + (a * B + b) * inner, (size_t)inner * sizeof(double));
}

/* grid (nz, ny, nx, u) -> out (az, ay, ax, u); work must hold
 * 4 * max(nz*ny*max(nx,ax), ...) doubles: callers pass oracle_tensor_work_size() */
int64_t oracle_tensor_work_size(int64_t nz, int64_t ny, int64_t nx __attribute__((unused)), int64_t ax, int64_t ay,
                                int64_t az, int64_t u) {
  int64_t a = nz * ny * ax * u, b = nz * ax * ay * u, c = ax * ay * az * u;
  int64_t m = a > b ? a : b;
  m = m > c ? m : c;
  return 2 * m;
}

void oracle_tensor_apply(const double* mx, int64_t ax, const double* my, int64_t ay, const double* mz,
                         int64_t az, const double* grid, int64_t nz, int64_t ny, int64_t nx, int64_t u,
                         double* work, double* out) {
  int64_t half = oracle_tensor_work_size(nz, ny, nx, ax, ay, az, u) / 2;
  double* w0 = work;
  double* w1 = work + half;
  /* t1 = mx @ grid over x: (nz*ny, ax, u) */
  contract(mx, ax, nx, grid, nz * ny, u, w0);
  /* t1c (nz, ax, ny, u) */
  for (int64_t z = 0; z < nz; ++z) swap01(w0 + z * ny * ax * u, ny, ax, u, w1 + z * ax * ny * u);
  /* t2 = my @ t1c over y: (nz, ax, ay, u) */
  contract(my, ay, ny, w1, nz * ax, u, w0);
  /* t2c (ax, ay, nz, u): (z, a, b) -> (a, b, z) */
  for (int64_t z = 0; z < nz; ++z)
    for (int64_t a = 0; a < ax; ++a)
      for (int64_t b = 0; b < ay; ++b)
        memcpy(w1 + ((a * ay + b) * nz + z) * u, w0 + ((z * ax + a) * ay + b) * u, (size_t)u * sizeof(double));
  /* t3 = mz @ t2c over z: (ax, ay, az, u) */
  contract(mz, az, nz, w1, ax * ay, u, w0);
  /* out (az, ay, ax, u) */
  for (int64_t a = 0; a < ax; ++a)
    for (int64_t b = 0; b < ay; ++b)
      for (int64_t c = 0; c < az; ++c)
        memcpy(out + ((c * ay + b) * ax + a) * u, w0 + ((a * ay + b) * az + c) * u, (size_t)u * sizeof(double));
}

/* One HaloExchange.run (schemes.py:185-202).  Returns 0, or -1 when the
 * source holds a non-finite value (ContractViolationError in the reference).
 * csr != NULL selects the matrix path; otherwise the tensor path with the
 * three axis matrices and the reference-source grid shape (nz, ny, nx). */
typedef struct {
  /* matrix path */
  const int64_t* row_offsets;
  const int64_t* col_indices;
  const double* values;
  int64_t n_rows;
  /* tensor path */
  const double* mx;
  const double* my;
  const double* mz;
  int64_t ax, ay, az, nz, ny, nx;
  /* maps */
  const int64_t* gather;
  int64_t n_src;
  const int64_t* scatter;
  int64_t n_out;
  int64_t u;
} oracle_exchange;

int oracle_exchange_run(const oracle_exchange* ex, const double* src, double* out, double* scratch) {
  if (!all_finite(src, ex->n_src)) return -1;
  double* ref_src = scratch;
  double* ref_out = scratch + ex->n_src;
  double* tail = ref_out + ex->n_out;
  for (int64_t i = 0; i < ex->n_src; ++i) ref_src[i] = src[ex->gather[i]];
  if (ex->row_offsets) {
    oracle_csr_apply(ex->row_offsets, ex->col_indices, ex->values, ex->n_rows, ref_src, ref_out, ex->u, tail);
  } else {
    oracle_tensor_apply(ex->mx, ex->ax, ex->my, ex->ay, ex->mz, ex->az, ref_src, ex->nz, ex->ny, ex->nx, ex->u,
                        tail, ref_out);
  }
  for (int64_t i = 0; i < ex->n_out; ++i) out[i] = ref_out[ex->scatter[i]];
  return 0;
}

int64_t oracle_exchange_scratch(const oracle_exchange* ex) {
  int64_t t = ex->row_offsets ? ex->u
                              : oracle_tensor_work_size(ex->nz, ex->ny, ex->nx, ex->ax, ex->ay, ex->az, ex->u);
  return ex->n_src + ex->n_out + t;
}

/* Many faces, each with its own exchange class, source and output buffer,
 * spread over nthreads OpenMP threads.  status[f] = oracle_exchange_run's result. */
void oracle_exchange_many(const oracle_exchange* const* ex, const double* const* src, double* const* out,
                          int64_t n_faces, int nthreads, int* status) {
  int64_t most = 0;
  for (int64_t f = 0; f < n_faces; ++f) {
    int64_t s = oracle_exchange_scratch(ex[f]);
    most = s > most ? s : most;
  }
#pragma omp parallel num_threads(nthreads)
  {
    double* scratch = (double*)malloc((size_t)most * sizeof(double));
#pragma omp for schedule(dynamic, 4)
    for (int64_t f = 0; f < n_faces; ++f) status[f] = oracle_exchange_run(ex[f], src[f], out[f], scratch);
    free(scratch);
  }
}
