// pow(x, y) bit-identical to the host C library the reference links (glibc 2.39, x86-64,
// the FMA variant its ifunc selects on any FMA/AVX2 CPU): the reference evaluates every
// L_p cell as pow(|v_f - v_g|, p) and every root as pow(acc, 1/p) through libm
// (pkg/src/pcflib/_sweepkern.pyx:10,43-46,98,114; SURVEY.md 8a "p=2,3 are not bitwise
// reproducible with x*x"), and pcflib.integrate._integrate_op takes the scalar root with
// CPython's float pow -- the same libm (integrate.py:114-128).
//
// Algorithm (glibc sysdeps/ieee754/dbl-64/e_pow.c, from ARM optimized-routines; restated
// here, not copied): log(x) in double-double from a 128-entry table of (1/c, log c) and a
// degree-8 polynomial, y*log(x) in double-double with one FMA, exp of that from a
// 128-entry table of 2^(k/128) and a degree-5 polynomial, with glibc's special cases for
// zero / subnormal / huge / tiny operands and results.  Every operation is spelled out
// (fma where the FMA build uses one, separate multiply/add elsewhere) so the compiler
// cannot contract differently on the host or the device.
//
// The tables are the C library's own, read out of the installed libm.so.6 at build time
// (__graft_entry__._pow_tables -> pcf_pow_tables.inc); tools/check_pow.c verifies the
// restatement against libm pow bit for bit on hundreds of millions of inputs.
#pragma once
#include <stdint.h>
#include <string.h>
#ifndef __CUDACC__
#include <math.h>
#define PCF_HD
#define PCF_CONST static const
#else
#define PCF_HD __host__ __device__
#define PCF_CONST __device__ const
#endif

#ifndef PCF_POW_CONTRACT
#define PCF_POW_CONTRACT 1
#endif

namespace pcfpow {

#include "pcf_pow_tables.inc"  // kPowLog*, kExp* (generated from libm.so.6)

PCF_HD inline uint64_t asu64(double x) {
#ifdef __CUDA_ARCH__
  return (uint64_t)__double_as_longlong(x);
#else
  uint64_t u;
  memcpy(&u, &x, 8);
  return u;
#endif
}
PCF_HD inline double asdbl(uint64_t u) {
#ifdef __CUDA_ARCH__
  return __longlong_as_double((long long)u);
#else
  double x;
  memcpy(&x, &u, 8);
  return x;
#endif
}
// correctly rounded primitives (no contraction on either compiler)
PCF_HD inline double mul(double a, double b) {
#ifdef __CUDA_ARCH__
  return __dmul_rn(a, b);
#else
  volatile double r = a * b;
  return r;
#endif
}
PCF_HD inline double add(double a, double b) {
#ifdef __CUDA_ARCH__
  return __dadd_rn(a, b);
#else
  volatile double r = a + b;
  return r;
#endif
}
PCF_HD inline double sub(double a, double b) {
#ifdef __CUDA_ARCH__
  return __dsub_rn(a, b);
#else
  volatile double r = a - b;
  return r;
#endif
}
PCF_HD inline double fmad(double a, double b, double c) {
#ifdef __CUDA_ARCH__
  return __fma_rn(a, b, c);
#else
  return fma(a, b, c);
#endif
}

PCF_HD inline uint32_t top12(double x) { return (uint32_t)(asu64(x) >> 52); }

// log(x) as hi + *tail for the normalised bit pattern ix (e_pow.c log_inline)
PCF_HD inline double log_inline(uint64_t ix, double* tail) {
  const uint64_t OFF = 0x3fe6955500000000ull;
  const uint64_t tmp = ix - OFF;
  const int i = (int)((tmp >> (52 - 7)) % 128);
  const int k = (int)((int64_t)tmp >> 52);
  const uint64_t iz = ix - (tmp & (0xfffull << 52));
  const double z = asdbl(iz);
  const double kd = (double)k;
  const double invc = kPowLogTab[4 * i], logc = kPowLogTab[4 * i + 2],
               logctail = kPowLogTab[4 * i + 3];
  const double r = fmad(z, invc, -1.0);
  const double* A = kPowLogPoly;
#if PCF_POW_CONTRACT
  // the FMA build lets the compiler fuse every product whose only use is an addition
  const double t1 = fmad(kd, kPowLogLn2hi, logc);
  const double lo1 = fmad(kd, kPowLogLn2lo, logctail);
#else
  const double t1 = add(mul(kd, kPowLogLn2hi), logc);
  const double lo1 = add(mul(kd, kPowLogLn2lo), logctail);
#endif
  const double t2 = add(t1, r);
  const double lo2 = add(sub(t1, t2), r);
  const double ar = mul(A[0], r);
  const double ar2 = mul(r, ar);
  const double ar3 = mul(r, ar2);
  const double hi = add(t2, ar2);
  const double lo3 = fmad(ar, r, -ar2);
  const double lo4 = add(sub(t2, hi), ar2);
#if PCF_POW_CONTRACT
  const double q = fmad(ar2, fmad(ar2, fmad(r, A[6], A[5]), fmad(r, A[4], A[3])),
                        fmad(r, A[2], A[1]));
  const double lo = fmad(ar3, q, add(add(add(lo1, lo2), lo3), lo4));
#else
  const double q = add(add(A[1], mul(r, A[2])),
                       mul(ar2, add(add(A[3], mul(r, A[4])),
                                    mul(ar2, add(A[5], mul(r, A[6]))))));
  const double lo = add(add(add(add(lo1, lo2), lo3), lo4), mul(ar3, q));
#endif
  const double y = add(hi, lo);
  *tail = add(sub(hi, y), lo);
  return y;
}

// scale + scale * tmp
PCF_HD inline double scale_add(double scale, double tmp) {
#if PCF_POW_CONTRACT
  return fmad(scale, tmp, scale);
#else
  return add(scale, mul(scale, tmp));
#endif
}

PCF_HD inline double oflow(uint32_t sign) { return sign ? -INFINITY : INFINITY; }
PCF_HD inline double uflow(uint32_t sign) { return sign ? -0.0 : 0.0; }

// results near the overflow / subnormal range (e_exp.c specialcase)
PCF_HD inline double specialcase(double tmp, uint64_t sbits, uint64_t ki) {
  double scale, y;
  if ((ki & 0x80000000ull) == 0) {
    sbits -= 1009ull << 52;
    scale = asdbl(sbits);
    y = mul(0x1p1009, scale_add(scale, tmp));
    return y;
  }
  sbits += 1022ull << 52;
  scale = asdbl(sbits);
  // scale * tmp has two uses here (y and lo): the FMA build keeps it a product
  // (verified bitwise against libm by tools/check_pow.cc)
  const double st = mul(scale, tmp);
  y = add(scale, st);
  if (fabs(y) < 1.0) {
    double one = 1.0;
    if (y < 0.0) one = -1.0;
    double lo = add(sub(scale, y), st);
    const double hi = add(one, y);
    lo = add(add(sub(one, hi), y), lo);
    y = sub(add(hi, lo), one);
    if (y == 0) y = asdbl(sbits & 0x8000000000000000ull);
  }
  return mul(0x1p-1022, y);
}

// exp(x + xtail) with the sign bias of a negative base (e_pow.c exp_inline)
PCF_HD inline double exp_inline(double x, double xtail, uint32_t sign_bias) {
  uint32_t abstop = top12(x) & 0x7ff;
  if (abstop - top12(0x1p-54) >= top12(512.0) - top12(0x1p-54)) {
    if ((int32_t)(abstop - top12(0x1p-54)) < 0) return sign_bias ? -1.0 : 1.0;
    if (abstop >= top12(1024.0)) return (asu64(x) >> 63) ? uflow(sign_bias) : oflow(sign_bias);
    abstop = 0;  // large |x| handled by specialcase below
  }
#if PCF_POW_CONTRACT
  double kd = fmad(kExpInvLn2N, x, kExpShift);
#else
  double kd = add(mul(kExpInvLn2N, x), kExpShift);
#endif
  const uint64_t ki = asu64(kd);
  kd = sub(kd, kExpShift);
#if PCF_POW_CONTRACT
  double r = fmad(kd, kExpNegLn2loN, fmad(kd, kExpNegLn2hiN, x));
#else
  double r = add(add(x, mul(kd, kExpNegLn2hiN)), mul(kd, kExpNegLn2loN));
#endif
  r = add(r, xtail);
  const uint64_t idx = 2 * (ki % 128);
  const uint64_t top = (ki + sign_bias) << (52 - 7);
  const double tail = asdbl(kExpTab[idx]);
  const uint64_t sbits = kExpTab[idx + 1] + top;
  const double r2 = mul(r, r);
  const double* C = kExpPoly;  // C2 .. C5
#if PCF_POW_CONTRACT
  const double tmp = fmad(mul(r2, r2), fmad(r, C[3], C[2]), fmad(r2, fmad(r, C[1], C[0]),
                                                                  add(tail, r)));
#else
  const double tmp = add(add(add(tail, r), mul(r2, add(C[0], mul(r, C[1])))),
                         mul(mul(r2, r2), add(C[2], mul(r, C[3]))));
#endif
  if (abstop == 0) return specialcase(tmp, sbits, ki);
  const double scale = asdbl(sbits);
  return scale_add(scale, tmp);
}

// 0: y not an integer, 1: odd integer, 2: even integer
PCF_HD inline int checkint(uint64_t iy) {
  const int e = (int)(iy >> 52 & 0x7ff);
  if (e < 0x3ff) return 0;
  if (e > 0x3ff + 52) return 2;
  if (iy & ((1ull << (0x3ff + 52 - e)) - 1)) return 0;
  if (iy & (1ull << (0x3ff + 52 - e))) return 1;
  return 2;
}
PCF_HD inline bool zeroinfnan(uint64_t i) { return 2 * i - 1 >= 2 * asu64(INFINITY) - 1; }

PCF_HD inline double pow(double x, double y) {
  uint32_t sign_bias = 0;
  uint64_t ix = asu64(x), iy = asu64(y);
  uint32_t topx = top12(x), topy = top12(y);
  const uint32_t SmallPowX = 0x001, ThresPowX = 0x7ff, SmallPowY = 0x3be, ThresPowY = 0x43e;
  if (topx - SmallPowX >= ThresPowX - SmallPowX ||
      (topy & 0x7ff) - SmallPowY >= ThresPowY - SmallPowY) {
    if (zeroinfnan(iy)) {
      if (2 * iy == 0) return 1.0;
      if (ix == asu64(1.0)) return 1.0;
      if (2 * ix > 2 * asu64(INFINITY) || 2 * iy > 2 * asu64(INFINITY)) return add(x, y);
      if (2 * ix == 2 * asu64(1.0)) return 1.0;
      if ((2 * ix < 2 * asu64(1.0)) == !(iy >> 63)) return 0.0;
      return mul(y, y);
    }
    if (zeroinfnan(ix)) {
      double x2 = mul(x, x);
      if ((ix >> 63) && checkint(iy) == 1) x2 = -x2;
      return (iy >> 63) ? 1.0 / x2 : x2;
    }
    if (ix >> 63) {
      const int yint = checkint(iy);
      if (yint == 0) return NAN;
      if (yint == 1) sign_bias = 0x800 << 7;
      ix &= 0x7fffffffffffffffull;
      topx &= 0x7ff;
    }
    if ((topy & 0x7ff) - SmallPowY >= ThresPowY - SmallPowY) {
      if (ix == asu64(1.0)) return 1.0;
      if ((topy & 0x7ff) < SmallPowY) return ix > asu64(1.0) ? add(1.0, y) : sub(1.0, y);
      return (ix > asu64(1.0)) == (topy < 0x800) ? oflow(0) : uflow(0);
    }
    if (topx == 0) {  // subnormal x: normalise so the exponent becomes negative
      ix = asu64(mul(x, 0x1p52));
      ix &= 0x7fffffffffffffffull;
      ix -= 52ull << 52;
    }
  }
  double lo;
  const double hi = log_inline(ix, &lo);
  const double ehi = mul(y, hi);
#if PCF_POW_CONTRACT
  const double elo = fmad(y, lo, fmad(y, hi, -ehi));
#else
  const double elo = add(mul(y, lo), fmad(y, hi, -ehi));
#endif
  return exp_inline(ehi, elo, sign_bias);
}

}  // namespace pcfpow
