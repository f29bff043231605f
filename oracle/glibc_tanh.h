/*
 * glibc_tanh.h — TEST INFRASTRUCTURE ONLY (oracle restatement).
 *
 * Bit-exact restatement of glibc 2.39 x86_64 `tanh` (sysdeps/ieee754/dbl-64
 * s_tanh.c, fdlibm-derived) and of the two `expm1` variants its IFUNC selects
 * between: the SSE2 build and the build compiled with -mfma -mavx2, where GCC
 * contracted several a*b+c expressions into fused multiply-adds.  The exact
 * operation sequences were read off the disassembly of this image's
 * /lib/x86_64-linux-gnu/libm.so.6 (expm1 IFUNC resolver at 0x2ef20, SSE2 body
 * at 0x2eaf0, FMA body at 0x7ac30, tanh at 0x31620). The reference MLP calls
 * std::tanh (mlp.cpp:155, :161), so this is the function the oracle must
 * reproduce; tests/test_oracle.py pins it against libm bit for bit.
 */
#ifndef ORACLE_GLIBC_TANH_H_
#define ORACLE_GLIBC_TANH_H_

#include <math.h>
#include <stdint.h>
#include <string.h>

static inline uint64_t gt_bits(double x) { uint64_t u; memcpy(&u, &x, 8); return u; }
static inline double gt_from(uint64_t u) { double x; memcpy(&x, &u, 8); return x; }

/* y with k added to its binary exponent by integer arithmetic on the high
 * word (the `add %ecx,%edx` sequence of both expm1 bodies). */
static inline double gt_add_exp(double y, int32_t k) {
  uint64_t b = gt_bits(y);
  uint32_t hi = (uint32_t)(b >> 32) + ((uint32_t)k << 20);
  return gt_from(((uint64_t)hi << 32) | (b & 0xffffffffull));
}

static const double GT_INVLN2 = 1.4426950408889634;       /* 0x3ff71547652b82fe */
static const double GT_LN2HI = 0.6931471803691238;        /* 0x3fe62e42fee00000 */
static const double GT_LN2LO = 1.9082149292705877e-10;    /* 0x3dea39ef35793c76 */
static const double GT_Q1 = -3.33333333333331316428e-02;  /* 0xbfa11111111110f4 */
static const double GT_Q2 = 1.58730158725481460165e-03;   /* 0x3f5a01a019fe5585 */
static const double GT_Q3 = -7.93650757867487942473e-05;  /* 0xbf14ce199eaadbb7 */
static const double GT_Q4 = 4.00821782732936239552e-06;   /* 0x3ed0cfca86e65239 */
static const double GT_Q5 = -2.01099218183624371326e-07;  /* 0xbe8afdb76e09c32d */

/* expm1, variant selected by `use_fma`.  Only finite |x| < 709.78 and the
 * tiny/negative-saturation branches are reachable from tanh; the overflow /
 * non-finite branches are reproduced for completeness. */
static inline double gt_expm1(double x, int use_fma) {
  const uint64_t bx = gt_bits(x);
  const uint32_t hx = (uint32_t)(bx >> 32) & 0x7fffffffu;
  const int neg = (int)((bx >> 63) & 1);
  double hi, lo, c = 0.0;
  int32_t k;
  if (hx >= 0x4043687Au) {               /* |x| >= 56 ln2 */
    if (hx >= 0x40862E42u) {             /* |x| >= 709.78 or non-finite */
      if (hx >= 0x7ff00000u) {
        if (((hx & 0xfffff) | (uint32_t)bx) != 0) return x + x; /* NaN */
        return neg ? -1.0 : x;
      }
      if (x > 7.09782712893383973096e+02) return 1e300 * 1e300; /* overflow */
    }
    if (neg) return 1e-300 - 1.0;        /* -1 with inexact */
  }
  if (hx > 0x3fd62e42u) {                /* |x| > 0.5 ln2 */
    if (hx < 0x3FF0A2B2u) {              /* and |x| < 1.5 ln2 */
      if (!neg) { hi = x - GT_LN2HI; lo = GT_LN2LO; k = 1; }
      else { hi = x + GT_LN2HI; lo = -GT_LN2LO; k = -1; }
    } else {
      double kf = GT_INVLN2 * x;
      kf = (neg ? -0.5 : 0.5) + kf;
      k = (int32_t)kf;                   /* cvttsd2si: truncation */
      const double t = (double)k;
      if (use_fma) hi = fma(-t, GT_LN2HI, x);
      else hi = x - GT_LN2HI * t;
      lo = t * GT_LN2LO;
    }
    x = hi - lo;
    c = (hi - x) - lo;
  } else if (hx < 0x3c900000u) {         /* |x| < 2^-54 */
    return x;
  } else {
    k = 0;
  }
  const double hfx = x * 0.5;
  const double hxs = x * hfx;
  double r1, t, e;
  if (use_fma) {
    const double R2 = fma(hxs, GT_Q3, GT_Q2);
    const double R3 = fma(hxs, GT_Q5, GT_Q4);
    const double h2 = hxs * hxs;
    const double R1 = fma(hxs, GT_Q1, 1.0);
    const double h4 = h2 * h2;
    r1 = fma(h4, R3, fma(h2, R2, R1));
    t = fma(-r1, hfx, 3.0);
    e = (r1 - t) / fma(-x, t, 6.0);
    e = e * hxs;
    if (k == 0) return x - fma(e, x, -hxs);
    e = fma(e - c, x, -c);
    e = e - hxs;
    if (k == -1) return fma(0.5, x - e, -0.5);
    if (k == 1) {
      if (x < -0.25) return (e - (x + 0.5)) * -2.0;
      return fma(x - e, 2.0, 1.0);
    }
  } else {
    const double h2 = hxs * hxs;
    const double R2 = GT_Q3 * hxs + GT_Q2;
    const double R1 = GT_Q1 * hxs + 1.0;
    const double h4 = h2 * h2;
    const double R3 = GT_Q5 * hxs + GT_Q4;
    r1 = (R2 * h2 + R1) + R3 * h4;
    t = 3.0 - hfx * r1;
    e = (r1 - t) / (6.0 - t * x);
    e = e * hxs;
    if (k == 0) return x - (e * x - hxs);
    e = (e - c) * x - c;
    e = e - hxs;
    if (k == -1) return (x - e) * 0.5 - 0.5;
    if (k == 1) {
      if (x < -0.25) return (e - (x + 0.5)) * -2.0;
      return 1.0 + 2.0 * (x - e);
    }
  }
  if (k <= -2 || k > 56) {
    const double y = 1.0 - (e - x);
    return gt_add_exp(y, k) - 1.0;
  }
  if (k < 20) {
    const double tt = gt_from((uint64_t)(0x3ff00000u - (0x200000u >> k)) << 32);
    return gt_add_exp(tt - (e - x), k);
  }
  {
    const double tt = gt_from((uint64_t)((uint32_t)(0x3ff - k) << 20) << 32);
    return gt_add_exp((x - (e + tt)) + 1.0, k);
  }
}

/* tanh (s_tanh.c; plain SSE2 build, calls the IFUNC-selected expm1). */
static inline double gt_tanh(double x, int use_fma) {
  const uint64_t bx = gt_bits(x);
  const uint32_t jx = (uint32_t)(bx >> 32);
  const uint32_t ix = jx & 0x7fffffffu;
  const int neg = (int)(jx >> 31);
  double z;
  if (ix >= 0x7ff00000u) return neg ? 1.0 / x - 1.0 : 1.0 / x + 1.0;
  if (ix < 0x40360000u) {                /* |x| < 22 */
    if ((ix | (uint32_t)bx) == 0) return x;
    if (ix < 0x3c800000u) return x * (1.0 + x);
    const double ax = fabs(x);
    if (ix >= 0x3ff00000u) {
      const double t = gt_expm1(ax + ax, use_fma);
      z = 1.0 - 2.0 / (t + 2.0);
    } else {
      const double t = gt_expm1(-2.0 * ax, use_fma);
      z = -t / (t + 2.0);
    }
  } else {
    z = 1.0 - 1e-300;
  }
  return neg ? -z : z;
}

#endif
