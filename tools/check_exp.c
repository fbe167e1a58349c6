// Bit-exactness check of tf_glibc_exp against the system libm exp().
// gcc -O2 -ffp-contract=off -I paper_2510_02758_b200/csrc tools/check_exp.c -lm
#include <stdio.h>
#include <stdlib.h>
#include <math.h>
#include "tf_glibc_exp.h"

static uint64_t s = 88172645463325252ull;
static uint64_t rnd(void) { s ^= s << 13; s ^= s >> 7; s ^= s << 17; return s; }

int main(int argc, char** argv) {
  long n = argc > 1 ? atol(argv[1]) : 10000000;
  long bad = 0;
  for (long i = 0; i < n; i++) {
    double x;
    int mode = i % 4;
    if (mode == 0) x = -(double)(rnd() >> 11) / (double)(1ull << 53) * 1100.0;      // [-1100, 0]
    else if (mode == 1) x = -(double)(rnd() >> 11) / (double)(1ull << 53) * 40.0;   // typical phi range
    else if (mode == 2) x = ((double)(rnd() >> 11) / (double)(1ull << 53) - 0.5) * 1500.0;
    else { uint64_t b = rnd(); double d; memcpy(&d, &b, 8); x = d; }              // any bit pattern
    if (isnan(x)) continue;
    double a = exp(x), b = tf_glibc_exp(x);
    if (memcmp(&a, &b, 8) != 0) {
      if (bad < 10) printf("x=%a libm=%a port=%a\n", x, a, b);
      bad++;
    }
  }
  // quotients exactly as the policy forms them: -b / (rate * interval)
  for (int b = 0; b <= 20000; b++)
    for (int ri = 0; ri < 6; ri++) {
      double rates[6] = {15.0, 20.0, 25.0, 30.0, 12.5, 40.0};
      double iv[3] = {0.5, 1.0, 0.25};
      for (int k = 0; k < 3; k++) {
        double sc = rates[ri] * iv[k];
        double x = -((double)b) / (sc > 1e-9 ? sc : 1e-9);
        double p = exp(x), q = tf_glibc_exp(x);
        if (memcmp(&p, &q, 8) != 0) { if (bad < 10) printf("b=%d x=%a\n", b, x); bad++; }
      }
    }
  printf("checked %ld random + 360k structured arguments: %ld mismatches\n", n, bad);
  return bad != 0;
}
