/*
 * TEST INFRASTRUCTURE — CPU oracle for the MoA generalized product.
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
 * legs may load this; the product path never does.
 *
 * A plain-C restatement of the reference's backend hot loops:
 *   oracle_product_rows  <- _ckernel.product_rows   (_ckernel.pyx:75-88)
 *     mul_add branch     <- _rows_mul_add           (_ckernel.pyx:37-52)
 *     generic branch     <- _rows_generic           (_ckernel.pyx:55-72)
 *     combine / reduce   <- _combine / _reduce      (_ckernel.pyx:11-34)
 *   oracle_product_parallel <- parallel.execute_parallel (parallel.py:26-43):
 *     W threads, worker k runs rows k, k+W, ... of one shared result buffer.
 * Same (i, l, j) loop order, same operand order, one IEEE operation at a time
 * (build with -ffp-contract=off, as the reference's setup.py:14 does), so it
 * is bit-identical to the reference; tests/test_oracle_pins.py checks that
 * against golden vectors produced by the reference itself.
 *
 * float32 variants load float32 operands and compute in float64, exactly as the
 * reference's MoaArray upcast (arrays.py:77-78) makes the reference do; the
 * float64 result is what the GPU's float32 output is compared against after a
 * single rounding.
 */
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>

static inline double combine_op(int code, double x, double y) {
  switch (code) {
    case 0: return x + y;
    case 1: return x - y;
    case 2: return x * y;
    case 3: return x / y;
    case 4: return x < y ? x : y;
    default: return x > y ? x : y;
  }
}

static inline double reduce_op(int code, double acc, double v) {
  switch (code) {
    case 0: return acc + v;
    case 1: return acc * v;
    case 2: return acc < v ? acc : v;
    default: return acc > v ? acc : v;
  }
}

/* element loaders: float64 operands or float32 operands upcast */
#define LOAD(p, f32, idx) ((f32) ? (double)((const float*)(p))[idx] : ((const double*)(p))[idx])

static void rows_impl(double* res, const void* a, const void* b, int a_f32, int b_f32,
                      int64_t noproc, int64_t rowsinred, int64_t elsinop, int64_t lstride,
                      int64_t rstride, int64_t restride, int comb, int red, int64_t start,
                      int64_t step) {
  for (int64_t i = start; i < noproc; i += step) {
    double* row = res + i * restride;
    for (int64_t l = 0; l < rowsinred; l++) {
      const double av = LOAD(a, a_f32, l + i * lstride);
      const int64_t lb = l * rstride;
      if (comb == 2 && red == 0) {
        for (int64_t j = 0; j < elsinop; j++) row[j] = row[j] + av * LOAD(b, b_f32, lb + j);
      } else {
        for (int64_t j = 0; j < elsinop; j++)
          row[j] = reduce_op(red, row[j], combine_op(comb, av, LOAD(b, b_f32, lb + j)));
      }
    }
  }
}

/* _ckernel.product_rows: accumulate rows start, start+step, ... into res */
void oracle_product_rows(double* res, const double* a, const double* b, int64_t noproc,
                         int64_t rowsinred, int64_t elsinop, int64_t lstride, int64_t rstride,
                         int64_t restride, int comb, int red, int64_t start, int64_t step) {
  rows_impl(res, a, b, 0, 0, noproc, rowsinred, elsinop, lstride, rstride, restride, comb, red,
            start, step);
}

void oracle_product_rows_f32in(double* res, const float* a, const float* b, int64_t noproc,
                               int64_t rowsinred, int64_t elsinop, int64_t lstride,
                               int64_t rstride, int64_t restride, int comb, int red,
                               int64_t start, int64_t step) {
  rows_impl(res, a, b, 1, 1, noproc, rowsinred, elsinop, lstride, rstride, restride, comb, red,
            start, step);
}

typedef struct {
  double* res;
  const void* a;
  const void* b;
  int f32;
  int64_t noproc, rowsinred, elsinop, lstride, rstride, restride;
  int comb, red;
  int64_t start, step;
} job_t;

static void* worker(void* p) {
  job_t* j = (job_t*)p;
  rows_impl(j->res, j->a, j->b, j->f32, j->f32, j->noproc, j->rowsinred, j->elsinop, j->lstride,
            j->rstride, j->restride, j->comb, j->red, j->start, j->step);
  return NULL;
}

/* parallel.execute_parallel: W fork-join threads, round-robin rows; returns 0 on success */
int oracle_product_parallel(double* res, const void* a, const void* b, int f32, int64_t noproc,
                            int64_t rowsinred, int64_t elsinop, int64_t lstride, int64_t rstride,
                            int64_t restride, int comb, int red, int workers) {
  if (workers < 1) return -1;
  pthread_t* th = (pthread_t*)malloc(sizeof(pthread_t) * workers);
  job_t* jobs = (job_t*)malloc(sizeof(job_t) * workers);
  if (!th || !jobs) { free(th); free(jobs); return -2; }
  int started = 0, rc = 0;
  for (int k = 0; k < workers; k++) {
    job_t j = {res, a, b, f32, noproc, rowsinred, elsinop, lstride, rstride, restride,
               comb, red, k, workers};
    jobs[k] = j;
    if (pthread_create(&th[k], NULL, worker, &jobs[k]) != 0) { rc = -3; break; }
    started++;
  }
  for (int k = 0; k < started; k++) pthread_join(th[k], NULL);
  free(th);
  free(jobs);
  return rc;
}
