/* Checks the division by a constant used by the lean kernel's Eq. (3) terms (sim_kernel.cuh cdiv): with
 * y = RN(1/b), q0 = RN(a y), two residual corrections q_{i+1} = RN(q_i + RN(a - b q_i) y) (the residual from one FMA)
 * must give RN(a / b) bit for bit.  Divisors: the cost models' flops / bw / link_bw / tp plus random ones; numerators:
 * the integer-valued doubles the terms divide (0 and 1 .. 2^63, log-uniform) and random normal doubles.
 *   gcc -O2 -ffp-contract=off tools/check_cdiv.c -lm && ./a.out [samples]                                        */
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

static uint64_t s = 0x9E3779B97F4A7C15ull;
static uint64_t next(void) { s ^= s << 13; s ^= s >> 7; s ^= s << 17; return s; }
static double cdiv(double a, double b, double y) {
  double q = a * y;
  q = fma(fma(-b, q, a), y, q);
  return fma(fma(-b, q, a), y, q);
}
int main(int argc, char** argv) {
  const long n = argc > 1 ? atol(argv[1]) : 2000000;
  double bs[64] = {312e12, 2039e9, 300e9, 989e12, 3350e9, 450e9, 1248e12, 8156e9, 3956e12, 13400e9, 1, 2, 3, 4, 7, 8};
  int nb = 16;
  while (nb < 64) {  /* random divisors: integers and general doubles */
    const uint64_t r = next();
    bs[nb++] = (nb & 1) ? (double)(r >> (next() % 60)) + 1.0 : ldexp((double)(r >> 11), (int)(next() % 200) - 100);
  }
  long bad = 0, tot = 0;
  for (int i = 0; i < nb; i++) {
    const double b = bs[i], y = 1.0 / b;
    for (long t = 0; t < n; t++) {
      double a;
      const uint64_t r = next();
      if (t % 3 == 0) a = (double)(r >> (next() % 64));  /* integer-valued, log-uniform magnitude */
      else if (t % 3 == 1) a = (double)((next() % 100000) * (next() % 100000000));
      else a = ldexp((double)(r >> 11) + 4503599627370496.0, (int)(next() % 120) - 60);
      const double q = cdiv(a, b, y), e = a / b;
      if (memcmp(&q, &e, 8)) {
        if (bad < 5) printf("MISMATCH a=%.17g b=%.17g got %.17g want %.17g\n", a, b, q, e);
        bad++;
      }
      tot++;
    }
  }
  printf("%ld of %ld quotients differ from RN(a/b)\n", bad, tot);
  return bad != 0;
}
