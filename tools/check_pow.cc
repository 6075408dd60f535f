// Bit-exact check of csrc/pcf_pow.cuh (the glibc pow restatement the device kernels use)
// against the host libm pow, on random and structured inputs covering the ranges the
// engine feeds it: |v_f - v_g| for p in {1.5, 2, 2.5, 3, 3.5, 4, 7.25} and roots
// pow(acc, 1/p) of accumulated integrals, plus subnormal / huge / tiny edge cases.
//   g++ -O2 -ffp-contract=off -I paper_2404_07183_b200/csrc tools/check_pow.cc -o /tmp/cp -lm
//   /tmp/cp [n_millions]          -> prints mismatches per class, exit 1 on any mismatch
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <random>
#include "pcf_pow.cuh"

static uint64_t bits(double x) { uint64_t u; memcpy(&u, &x, 8); return u; }

int main(int argc, char** argv) {
  const long n = (argc > 1 ? atol(argv[1]) : 20) * 1000000L;
  std::mt19937_64 rng(2404);
  std::uniform_real_distribution<double> U(0.0, 1.0);
  const double ys[] = {1.5, 2.0, 2.5, 3.0, 3.5, 4.0, 7.25, 1.0 / 1.5, 0.5, 1.0 / 2.5,
                       1.0 / 3.0, 1.0 / 3.5, 0.25, 1.0 / 7.25, 1.0};
  long bad = 0, total = 0;
  double (*volatile libm_pow)(double, double) = static_cast<double (*)(double, double)>(::pow);
  for (double y : ys) {
    long b = 0;
    for (long i = 0; i < n / 15; ++i) {
      double x;
      const int cls = (int)(i % 4);
      if (cls == 0) x = U(rng) * 8.0;                                 // |dv| of N(0,1) values
      else if (cls == 1) x = ldexp(U(rng) + 0.5, (int)(rng() % 200) - 100);  // wide range
      else if (cls == 2) x = (double)(rng() % 20000) * 0.5;          // integer-valued (ECC)
      else if (i % 8 == 3) x = ldexp(U(rng) + 0.5, (int)(rng() % 2200) - 1100);  // extremes
      else x = ldexp(U(rng) + 0.5, -(int)(rng() % 500) - 150);  // tiny / subnormal results
      const double a = libm_pow(x, y), c = pcfpow::pow(x, y);
      if (bits(a) != bits(c) && !(a != a && c != c)) {
        if (b < 5) printf("  y=%a x=%a libm=%a ours=%a\n", y, x, a, c);
        ++b;
      }
    }
    printf("y=%g: %ld mismatches of %ld\n", y, b, n / 15);
    bad += b;
    total += n / 15;
  }
  const double edge[] = {0.0, -0.0, 1.0, INFINITY, 0x1p-1074, 0x1p-1022, 0x1.fffffffffffffp1023,
                         0x1p-537, 0x1p537, 1e-310, 1e300};
  for (double x : edge)
    for (double y : ys) {
      const double a = libm_pow(x, y), c = pcfpow::pow(x, y);
      ++total;
      if (bits(a) != bits(c)) {
        printf("  edge x=%a y=%a libm=%a ours=%a\n", x, y, a, c);
        ++bad;
      }
    }
  printf("%s: %ld mismatches of %ld\n", bad ? "FAIL" : "OK", bad, total);
  return bad ? 1 : 0;
}
