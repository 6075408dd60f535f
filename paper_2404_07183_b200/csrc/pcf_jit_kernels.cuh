// Kernels for user-defined combination integrals, compiled at run time by NVRTC for
// sm_100a (pcf_jit.cpp) after a prefix of user definitions generated from the Python
// integrand by paper_2404_07183_b200/jit.py:
//
//   #define PCF_MODE 0 | 1        0: pointwise integrand h(x, y) (combine_integrate,
//                                 integrate.py:51-78); 1: antiderivative H(x, y, t)
//                                 (combine_integrate_timedep, integrate.py:81-111)
//   #define PCF_HAS_R 0 | 1       functional r applied to the integral (CombinationIntegral.r,
//                                 integrate.py:175-203)
//   __device__ double pcf_h(double x, double y);            (mode 0)
//   __device__ double pcf_H(double x, double y, double t);  (mode 1)
//   __device__ double pcf_r(double x);                      (PCF_HAS_R)
//   __device__ double pcf_u(double v);                      (integrate_single, PCF_HAS_U)
//
// Every pair is walked by ONE thread in exactly the reference's cell order
// (sweep.iterate_rectangles, sweep.py:67-100: start cursors max{i : t_i <= a}, tn = the
// earlier next breakpoint, simultaneous jumps advance both cursors, no zero-width cells)
// and summed left to right as the reference does (acc += h * (r - l), or
// acc += H(., ., r) - H(., ., l)), compiled with --fmad=false: for integrands built from
// + - * / abs min max sqrt the result is bit-identical to the reference's Python float
// arithmetic.  Transcendentals use CUDA's libdevice (<= 2 ulp from glibc).
//
// Records as in pcf_common.cuh: PCF s = 16-byte {t_next, v} records at soff[s] (float64;
// float32 collections are widened exactly).  Status per entry: 0 ok, 1 divergent tail,
// 2 non-finite (NaN tail integrand or non-finite sum) -- the reference's
// DivergentIntegral / NonFinite (integrate.py:63-78, 96-111).

#define PCF_INF __longlong_as_double(0x7ff0000000000000LL)
#define PCF_NAN __longlong_as_double(0x7ff8000000000000LL)

struct PcfRec {
  double t;
  double v;
};

// Python semantics helpers used by the translated expressions
__device__ __forceinline__ double pcf_pymax(double a, double b) { return b > a ? b : a; }
__device__ __forceinline__ double pcf_pymin(double a, double b) { return b < a ? b : a; }
__device__ __forceinline__ double pcf_npmax(double a, double b) {
  return (a != a || b != b) ? PCF_NAN : (b > a ? b : a);
}
__device__ __forceinline__ double pcf_npmin(double a, double b) {
  return (a != a || b != b) ? PCF_NAN : (b < a ? b : a);
}
// CPython float % and // (Objects/floatobject.c float_rem / float_floor_div): the
// remainder takes the divisor's sign (a zero remainder is copysign(0, y)), the quotient is
// (x - mod) / y snapped to the nearest integer, not floor(x / y): 1.0 // 0.1 == 9.0
__device__ __forceinline__ double pcf_pymod(double x, double y) {
  double r = fmod(x, y);
  if (r != 0.0) {
    if ((y < 0.0) != (r < 0.0)) r = __dadd_rn(r, y);
  } else {
    r = copysign(0.0, y);
  }
  return r;
}
__device__ __forceinline__ double pcf_pyfloordiv(double x, double y) {
  double mod = fmod(x, y);
  double div = __ddiv_rn(__dsub_rn(x, mod), y);
  if (mod != 0.0) {
    if ((y < 0.0) != (mod < 0.0)) div = __dsub_rn(div, 1.0);
  }
  double fd;
  if (div != 0.0) {
    fd = floor(div);
    if (__dsub_rn(div, fd) > 0.5) fd = __dadd_rn(fd, 1.0);
  } else {
    fd = copysign(0.0, __ddiv_rn(x, y));
  }
  return fd;
}
__device__ __forceinline__ double pcf_sq(double x) { return __dmul_rn(x, x); }

// max{i < n : key(i) <= a} + 1 style start cursor: number of records whose piece ends at
// or before a (the reference's linear _start_index, sweep.py:59-64)
__device__ __forceinline__ int pcf_start(const PcfRec* __restrict__ F, int n, double a) {
  int lo = 0, hi = n - 1;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (F[mid].t <= a) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}

#if PCF_MODE == 0
__device__ __forceinline__ double pcf_cell(double x, double y, double l, double r) {
  return __dmul_rn(pcf_h(x, y), __dsub_rn(r, l));
}
#else
__device__ __forceinline__ double pcf_cell(double x, double y, double l, double r) {
  return __dsub_rn(pcf_H(x, y, r), pcf_H(x, y, l));
}
#endif

// One pair's integral over [a, b); returns the status, *res the raw sum.
__device__ int pcf_pair(const PcfRec* __restrict__ F, int nf, const PcfRec* __restrict__ G,
                        int ng, double a, double b, double* res) {
  int k = pcf_start(F, nf, a), m = pcf_start(G, ng, a);
  double t = a, acc = 0.0;
  int st = 0;
  for (;;) {
    const double tnf = F[k].t, tng = G[m].t;
    const double tn = tnf < tng ? tnf : tng;
    const double vf = F[k].v, vg = G[m].v;
    if (tn >= b) {
      if (b == PCF_INF) {
#if PCF_MODE == 0
        const double hv = pcf_h(vf, vg);
        if (hv != hv) st = 2;
        else if (hv != 0.0) st = 1;
#else
        const double c = __dsub_rn(pcf_H(vf, vg, PCF_INF), pcf_H(vf, vg, t));
        if (c != 0.0 || c != c) st = 1;
#endif
      } else {
        acc = __dadd_rn(acc, pcf_cell(vf, vg, t, b));
      }
      break;
    }
    acc = __dadd_rn(acc, pcf_cell(vf, vg, t, tn));
    if (tnf == tn) ++k;
    if (tng == tn) ++m;
    t = tn;
  }
  if (st == 0 && !(acc - acc == 0.0)) st = 2;  // NaN or +-inf sum
  *res = acc;
  return st;
}

// Entry value as the reference returns it: _round_to_kind(acc), then r and round again
// (CombinationIntegral.__call__, integrate.py:197-203).
__device__ __forceinline__ double pcf_finish(double acc, int out_f32) {
  double v = out_f32 ? (double)__double2float_rn(acc) : acc;
#if PCF_HAS_R
  v = pcf_r(v);
  if (out_f32) v = (double)__double2float_rn(v);
#endif
  return v;
}

// Pairwise matrix on size-sorted indices: rows [r0, r1) x columns (sym: q >= s, else all);
// out[perm[s], perm[q]] (and the mirror when sym), original order, leading dimension ld.
// errs[0] / errs[1]: atomicMin of the row-major key of the first divergent / non-finite
// entry (original indices; sym keys are (min, max)).
extern "C" __global__ void pcf_jit_matrix(const PcfRec* __restrict__ recs,
                                          const long long* __restrict__ soff,
                                          const int* __restrict__ perm, long long M, int sym,
                                          double a, double b, void* __restrict__ out, int out_f32,
                                          long long ld, long long r0, long long r1,
                                          unsigned long long* __restrict__ errs) {
  for (long long s = r0 + blockIdx.y; s < r1; s += gridDim.y) {
    const PcfRec* F = recs + soff[s];
    const int nf = (int)(soff[s + 1] - soff[s]);
    const long long oi = perm[s];
    const long long q0 = sym ? s : 0;
    for (long long q = q0 + blockIdx.x * (long long)blockDim.x + threadIdx.x; q < M;
         q += (long long)gridDim.x * blockDim.x) {
      const PcfRec* G = recs + soff[q];
      const int ng = (int)(soff[q + 1] - soff[q]);
      const long long oj = perm[q];
      double acc;
      // the reference computes entry (i, j <= ... ) with f = the lower original index
      // (matrix.py:186-193); keep that orientation for symmetric jobs
      const bool swap = sym && oj < oi;
      const int st = swap ? pcf_pair(G, ng, F, nf, a, b, &acc) : pcf_pair(F, nf, G, ng, a, b, &acc);
      if (st) {
        const long long lo = (sym && oj < oi) ? oj : oi, hi = (sym && oj < oi) ? oi : oj;
        atomicMin(&errs[st - 1], (unsigned long long)(lo * M + hi));
      }
      const double v = pcf_finish(acc, out_f32);
      if (out_f32) {
        float* o = (float*)out;
        o[oi * ld + oj] = (float)v;
        if (sym) o[oj * ld + oi] = (float)v;
      } else {
        double* o = (double*)out;
        o[oi * ld + oj] = v;
        if (sym) o[oj * ld + oi] = v;
      }
    }
  }
}

// Explicit pairs (sorted indices): value after rounding and r, and the status.
extern "C" __global__ void pcf_jit_pairs(const PcfRec* __restrict__ recs,
                                         const long long* __restrict__ soff,
                                         const long long* __restrict__ pairs, long long npairs,
                                         double a, double b, int out_f32,
                                         double* __restrict__ res, int* __restrict__ status) {
  for (long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x; k < npairs;
       k += (long long)gridDim.x * blockDim.x) {
    const long long s = pairs[2 * k], q = pairs[2 * k + 1];
    double acc;
    const int st = pcf_pair(recs + soff[s], (int)(soff[s + 1] - soff[s]), recs + soff[q],
                            (int)(soff[q + 1] - soff[q]), a, b, &acc);
    status[k] = st;
    res[k] = pcf_finish(acc, out_f32);
  }
}

#if PCF_HAS_U
// integrate_single (integrate.py:146-171 over sweep.iterate_segments, sweep.py:103-116):
// pieces [t, t_next) while t_next < b, then the last piece [t, b); same tail rules.
extern "C" __global__ void pcf_jit_single(const PcfRec* __restrict__ recs,
                                          const long long* __restrict__ soff, long long M,
                                          double a, double b, int out_f32,
                                          double* __restrict__ res, int* __restrict__ status) {
  for (long long s = blockIdx.x * (long long)blockDim.x + threadIdx.x; s < M;
       s += (long long)gridDim.x * blockDim.x) {
    const PcfRec* F = recs + soff[s];
    const int n = (int)(soff[s + 1] - soff[s]);
    int k = pcf_start(F, n, a);
    double t = a, acc = 0.0;
    int st = 0;
    while (k + 1 < n && F[k].t < b) {
      acc = __dadd_rn(acc, __dmul_rn(pcf_u(F[k].v), __dsub_rn(F[k].t, t)));
      t = F[k].t;
      ++k;
    }
    const double hv = pcf_u(F[k].v);
    if (b == PCF_INF) {
      if (hv != hv) st = 2;
      else if (hv != 0.0) st = 1;
    } else {
      acc = __dadd_rn(acc, __dmul_rn(hv, __dsub_rn(b, t)));
    }
    if (st == 0 && !(acc - acc == 0.0)) st = 2;
    status[s] = st;
    res[s] = out_f32 ? (double)__double2float_rn(acc) : acc;
  }
}
#endif
