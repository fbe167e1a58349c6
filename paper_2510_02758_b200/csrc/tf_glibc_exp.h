// exp(x) reproducing the x86-64 glibc (>= 2.28) FMA code path bit for bit.
//
// The reference's buffer penalty phi = exp(-b / (r * dt)) is evaluated by
// CPython's math.exp, i.e. glibc's exp (scheduler.py:86-93).  On x86-64 CPUs
// with FMA+AVX2 (the build box and the B200 hosts) glibc's ifunc selects the
// FMA build of sysdeps/ieee754/dbl-64/e_exp.c, whose contractions are:
//     kd  = fma(x, InvLn2N, Shift)          r = fma(kd, NegLn2hiN, x)
//     r   = fma(kd, NegLn2loN, r)            r2 = r * r
//     tmp = fma(fma(r, C3, C2), r2, r + tail)
//     tmp = fma(r2 * r2, fma(r, C5, C4), tmp)
//     y   = fma(scale, tmp, scale)
// (read off the shipped libm's machine code; the table is generated from
// first principles by tools/gen_exp_table.py).  CUDA's own exp() differs by
// up to 1 ulp, which would flip near-tie priority sorts, so the selector
// kernel uses this port instead.  tools/check_exp.c verifies it against
// libm over 10^8 random arguments.
#pragma once
#include <stdint.h>
#include <string.h>
#include "tf_exp_table.h"

#include <math.h>
#if defined(__CUDACC__)
#define TF_HD __host__ __device__ __forceinline__
#else
#define TF_HD static inline
#endif
// Host passes must be compiled with -ffp-contract=off (no implicit FMA).
#if defined(__CUDA_ARCH__)
#define TF_FMA(a, b, c) __fma_rn((a), (b), (c))
#define TF_MUL(a, b) __dmul_rn((a), (b))
#define TF_ADD(a, b) __dadd_rn((a), (b))
#define TF_SUB(a, b) __dsub_rn((a), (b))
#else
#define TF_FMA(a, b, c) fma((a), (b), (c))
#define TF_MUL(a, b) ((a) * (b))
#define TF_ADD(a, b) ((a) + (b))
#define TF_SUB(a, b) ((a) - (b))
#endif

TF_HD double tf_asdouble(uint64_t u) {
#if defined(__CUDA_ARCH__)
  return __longlong_as_double((long long)u);
#else
  double d;
  memcpy(&d, &u, 8);
  return d;
#endif
}

TF_HD uint64_t tf_asuint64(double d) {
#if defined(__CUDA_ARCH__)
  return (uint64_t)__double_as_longlong(d);
#else
  uint64_t u;
  memcpy(&u, &d, 8);
  return u;
#endif
}

#if defined(__CUDACC__)
__device__ __constant__ static const uint64_t tf_exp_tab_dev[256] = TF_EXP_TABLE_INIT;
#endif
static const uint64_t tf_exp_tab_host[256] = TF_EXP_TABLE_INIT;

TF_HD const uint64_t* tf_exp_tab() {
#if defined(__CUDA_ARCH__)
  return tf_exp_tab_dev;
#else
  return tf_exp_tab_host;
#endif
}

// Out-of-range tail (|k| large): scale the exponent in two steps.
TF_HD double tf_exp_special(double tmp, uint64_t sbits, uint64_t ki) {
  if ((ki & 0x80000000u) == 0) {
    sbits -= 1009ull << 52;
    double scale = tf_asdouble(sbits);
    return TF_MUL(TF_FMA(scale, tmp, scale), 0x1p1009);
  }
  sbits += 1022ull << 52;
  double scale = tf_asdouble(sbits);
  double st = TF_MUL(scale, tmp);
  double y = TF_ADD(scale, st);
  if (y < 1.0) {
    double lo = TF_ADD(TF_SUB(scale, y), st);
    double hi = TF_ADD(y, 1.0);
    double t = TF_ADD(TF_ADD(TF_SUB(1.0, hi), y), lo);
    y = TF_SUB(TF_ADD(t, hi), 1.0);
    if (y == 0.0) y = 0.0;
  }
  return TF_MUL(y, 0x1p-1022);
}

TF_HD double tf_glibc_exp(double x) {
  const double InvLn2N = 0x1.71547652b82fep7;
  const double Shift = 0x1.8p52;
  const double NegLn2hiN = -0x1.62e42fefa0000p-8;
  const double NegLn2loN = -0x1.cf79abc9e3b3ap-47;
  const double C2 = 0x1.ffffffffffdbdp-2;
  const double C3 = 0x1.555555555543cp-3;
  const double C4 = 0x1.55555cf172b91p-5;
  const double C5 = 0x1.1111167a4d017p-7;
  uint64_t ix = tf_asuint64(x);
  uint32_t abstop = (uint32_t)((ix >> 52) & 0x7ff);
  int special = 0;
  if (abstop - 0x3c9u > 0x3eu) {
    if ((int32_t)(abstop - 0x3c9u) < 0) return TF_ADD(1.0, x);  // |x| < 2^-54
    if (abstop >= 0x409) {                                      // |x| >= 1024
      if (ix == 0xfff0000000000000ull) return 0.0;
      if (abstop >= 0x7ff) return TF_ADD(1.0, x);
      return (ix >> 63) ? 0.0 : __builtin_huge_val();
    }
    special = 1;  // 512 <= |x| < 1024
  }
  double kd = TF_FMA(x, InvLn2N, Shift);
  uint64_t ki = tf_asuint64(kd);
  kd = TF_SUB(kd, Shift);
  double r = TF_FMA(kd, NegLn2hiN, x);
  r = TF_FMA(kd, NegLn2loN, r);
  uint64_t idx = 2 * (ki & 127);
  uint64_t top = ki << 45;
  const uint64_t* T = tf_exp_tab();
  double tail = tf_asdouble(T[idx]);
  uint64_t sbits = T[idx + 1] + top;
  double r2 = TF_MUL(r, r);
  double tmp = TF_FMA(TF_FMA(r, C3, C2), r2, TF_ADD(r, tail));
  tmp = TF_FMA(TF_MUL(r2, r2), TF_FMA(r, C5, C4), tmp);
  if (special) return tf_exp_special(tmp, sbits, ki);
  double scale = tf_asdouble(sbits);
  return TF_FMA(scale, tmp, scale);
}
