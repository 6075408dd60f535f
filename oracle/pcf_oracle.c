/* pcf_oracle.c -- CPU restatement of the reference kernel module.  TEST INFRASTRUCTURE
 * ONLY: used by tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg as the
 * checker / CPU baseline; never linked into or called by the product path.
 *
 * Restates, operation for operation:
 *   _accumulate   pkg/src/pcflib/_sweepkern.pyx:24-59
 *   fill_block    pkg/src/pcflib/_sweepkern.pyx:88-121
 * Build: gcc -O2 -ffp-contract=off (no FMA contraction, SSE2 double) -- the reference is
 * built by Cython/gcc -O2 for plain x86-64 (no FMA), so p=1 and inner-product results are
 * bit-identical to it; pow() is the same glibc libm.
 *
 * Parity is pinned against the reference itself: tests/golden holds outputs of the
 * reference's compiled _sweepkern (tests/golden/make_golden.py), and tests check this
 * oracle against them bit for bit.
 */
#include <math.h>
#include <stdint.h>
#include <pthread.h>
#include <stdlib.h>

#define OP_LP 0
#define OP_INNER 1

/* pyx:24-59 */
double pcf_oracle_accumulate(const double* ft, const double* fv, int64_t nf, const double* gt,
                             const double* gv, int64_t ng, double a, double b, int op,
                             double p) {
  int64_t k = 0, m = 0;
  double acc = 0.0, t = a;
  while (k + 1 < nf && ft[k + 1] <= a) ++k;
  while (m + 1 < ng && gt[m + 1] <= a) ++m;
  for (;;) {
    const double vf = fv[k], vg = gv[m];
    const double tnf = (k + 1 < nf) ? ft[k + 1] : INFINITY;
    const double tng = (m + 1 < ng) ? gt[m + 1] : INFINITY;
    const double tn = tnf < tng ? tnf : tng;
    const double hv = (op == OP_LP) ? pow(fabs(vf - vg), p) : vf * vg;
    if (tn >= b) {
      if (b == INFINITY) {
        if (hv != 0.0) return hv > 0.0 ? INFINITY : -INFINITY;
      } else {
        acc += hv * (b - t);
      }
      return acc;
    }
    acc += hv * (tn - t);
    if (tnf == tn) ++k;
    if (tng == tn) ++m;
    t = tn;
  }
}

/* pyx:88-121 on float64 packed arrays (tcat, vcat, off); out is M x ld float64.
 * Returns 0, or 1 with *ei/*ej = first non-finite pair (row-major within the block). */
int pcf_oracle_fill_block(const double* tcat, const double* vcat, const int64_t* off, int64_t M,
                          int64_t r0, int64_t r1, int op, double p, int apply_root, int diag,
                          double a, double b, double* out, int64_t ld, int64_t* ei,
                          int64_t* ej) {
  const double invp = apply_root ? 1.0 / p : 1.0;
  for (int64_t i = r0; i < r1; ++i) {
    for (int64_t j = diag ? i : i + 1; j < M; ++j) {
      double acc = pcf_oracle_accumulate(tcat + off[i], vcat + off[i], off[i + 1] - off[i],
                                         tcat + off[j], vcat + off[j], off[j + 1] - off[j], a,
                                         b, op, p);
      if (acc == INFINITY || acc == -INFINITY || acc != acc) {
        *ei = i;
        *ej = j;
        return 1;
      }
      if (apply_root) acc = pow(acc, invp);
      out[i * ld + j] = acc;
      out[j * ld + i] = acc;
    }
  }
  return 0;
}

/* Same as fill_block for row i only, into a row-sized sink (out[j] for j in (i, M)): the
 * O(M)-memory form used to sample rows of matrices too large for host RAM. */
int pcf_oracle_row(const double* tcat, const double* vcat, const int64_t* off, int64_t M,
                   int64_t i, int op, double p, int apply_root, double a, double b,
                   double* row) {
  const double invp = apply_root ? 1.0 / p : 1.0;
  for (int64_t j = i + 1; j < M; ++j) {
    double acc = pcf_oracle_accumulate(tcat + off[i], vcat + off[i], off[i + 1] - off[i],
                                       tcat + off[j], vcat + off[j], off[j + 1] - off[j], a, b,
                                       op, p);
    if (acc == INFINITY || acc == -INFINITY || acc != acc) return 1;
    if (apply_root) acc = pow(acc, invp);
    row[j] = acc;
  }
  return 0;
}

/* Threaded row-sample timing harness: rows[0..nrows) each computed against all j > row
 * into per-thread scratch; returns the number of cells (steps) processed. */
typedef struct {
  const double *tcat, *vcat;
  const int64_t* off;
  int64_t M;
  const int64_t* rows;
  int64_t nrows;
  int op;
  double p;
  int apply_root;
  int tid, nthreads;
  double checksum;
} job_t;

static void* worker(void* arg) {
  job_t* J = (job_t*)arg;
  double* row = (double*)calloc((size_t)J->M, sizeof(double));
  double cs = 0.0;
  for (int64_t r = J->tid; r < J->nrows; r += J->nthreads) {
    int64_t i = J->rows[r];
    pcf_oracle_row(J->tcat, J->vcat, J->off, J->M, i, J->op, J->p, J->apply_root, 0.0, INFINITY,
                   row);
    for (int64_t j = i + 1; j < J->M; ++j) cs += row[j];
  }
  J->checksum = cs;
  free(row);
  return NULL;
}

double pcf_oracle_rows_threaded(const double* tcat, const double* vcat, const int64_t* off,
                                int64_t M, const int64_t* rows, int64_t nrows, int op, double p,
                                int apply_root, int nthreads) {
  if (nthreads < 1) nthreads = 1;
  pthread_t* th = (pthread_t*)malloc(sizeof(pthread_t) * (size_t)nthreads);
  job_t* jobs = (job_t*)malloc(sizeof(job_t) * (size_t)nthreads);
  for (int t = 0; t < nthreads; ++t) {
    job_t J = {tcat, vcat, off, M, rows, nrows, op, p, apply_root, t, nthreads, 0.0};
    jobs[t] = J;
    pthread_create(&th[t], NULL, worker, &jobs[t]);
  }
  double cs = 0.0;
  for (int t = 0; t < nthreads; ++t) {
    pthread_join(th[t], NULL);
    cs += jobs[t].checksum;
  }
  free(th);
  free(jobs);
  return cs;
}
