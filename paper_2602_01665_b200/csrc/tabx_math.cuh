// Scalar math with the reference's rounding.
//
// * libm_sin/libm_cos: numpy's float64 cos/sin (called at
//   perception.py:61-62,118-119; combat.py:31-32; heuristics.py:91,192) are
//   the host glibc's, which is NOT correctly rounded (0.07% of arguments
//   differ from the correctly rounded value by one ulp).  CUDA's sin/cos
//   differ by up to 2 ulp.  To reproduce the reference bit for bit the
//   device runs a restatement of glibc 2.39's algorithm, including the
//   exact fused multiply-adds of its x86-64 FMA build.
//   Provenance / attribution: the range reduction constants, the
//   polynomial coefficients and the branch structure of __sin / __cos follow
//   the GNU C Library's sysdeps/ieee754/dbl-64/s_sin.c and usncs.h (glibc
//   2.39, Copyright (C) 2001-2024 Free Software Foundation, Inc., licensed
//   under the GNU Lesser General Public License v2.1 or later; originally
//   contributed by IBM).  The table sincos_table.inc is regenerated from its
//   definition (sin/cos of i/128 in 70-digit arithmetic,
//   tools/gen_sincos_table.py), not copied.
// * np_max/np_min/np_clip/np_remainder: numpy's ufunc definitions.
// * pairwise_sum: numpy's pairwise add.reduce (8 accumulators, blocks of
//   128, recursive split), used for the team health ratio sums
//   (arrays.py:395) and the lava burn sum (environment.py:273).
//
// Everything here is compiled with -fmad=false; the only fused multiply-adds
// are the explicit fma() calls of the libm restatement.
#pragma once
#include <math.h>
#include <stdint.h>

#if defined(__CUDACC__)
#define TABX_HD __host__ __device__ __forceinline__
#define TABX_HD_CALL static __host__ __device__ __noinline__
#define TABX_SC_TABLE_QUAL __device__ const
#else
#define TABX_HD static inline
#define TABX_HD_CALL static
#define TABX_SC_TABLE_QUAL static const
#endif

#include "sincos_table.inc"

namespace tabx {

// ---------------------------------------------------------------------------
// libm restatement: glibc 2.39 dbl-64 sin/cos, x86-64 FMA multiarch build
// (sysdeps/ieee754/dbl-64/s_sin.c + usncs.h constants).  The fused
// multiply-adds below are the ones GCC emits for that build (-mfma, contract
// on); every other operation is an unfused IEEE double op (-fmad=false).
// Valid for |x| < 105414350; larger arguments (never produced by headings)
// fall back to CUDA's sin/cos.
// ---------------------------------------------------------------------------
TABX_HD double bits_to_d(uint64_t b) {
  union { uint64_t u; double d; } v;
  v.u = b;
  return v.d;
}
TABX_HD uint64_t d_to_bits(double d) {
  union { uint64_t u; double d; } v;
  v.d = d;
  return v.u;
}

#define TABX_BIG bits_to_d(0x42c8000000000000ULL)   /* 52776558133248 = 1.5*2^45 */
#define TABX_HP0 bits_to_d(0x3FF921FB54442D18ULL)   /* pi/2 hi */
#define TABX_HP1 bits_to_d(0x3C91A62633145C07ULL)   /* pi/2 lo */
#define TABX_MP1 bits_to_d(0x3FF921FB58000000ULL)
#define TABX_MP2 bits_to_d(0xBE4DDE973C000000ULL)
#define TABX_PP3 bits_to_d(0xBC8CB3B398000000ULL)
#define TABX_PP4 bits_to_d(0xBACD747F23E32ED7ULL)
#define TABX_HPINV bits_to_d(0x3FE45F306DC9C883ULL) /* 2/pi */
#define TABX_TOINT bits_to_d(0x4338000000000000ULL) /* 1.5*2^52 */

struct libm_consts {
  static constexpr double sn3 = -1.66666666666664880952546298448555E-01;
  static constexpr double sn5 = 8.33333214285722277379541354343671E-03;
  static constexpr double cs2 = 4.99999999999999999999950396842453E-01;
  static constexpr double cs4 = -4.16666666666664434524222570944589E-02;
  static constexpr double cs6 = 1.38888874007937613028114285595617E-03;
  static constexpr double s1 = -1.6666666666666666e-01;
  static constexpr double s2 = 8.3333333333323288e-03;
  static constexpr double s3 = -1.9841269834414642e-04;
  static constexpr double s4 = 2.755729806860771e-06;
  static constexpr double s5 = -2.5022014848318398e-08;
};

TABX_HD const double* sc_entry(double u) {
  return &tabx_sc_table[0][0] + 4 * (int)(uint32_t)d_to_bits(u);
}

TABX_HD double taylor_sin(double xx, double a, double da) {
  typedef libm_consts K;
  double poly = fma(fma(fma(fma(K::s5, xx, K::s4), xx, K::s3), xx, K::s2), xx, K::s1);
  double t = fma(fma(poly, a, -(0.5 * da)), xx, da);
  return a + t;
}

TABX_HD double libm_do_cos(double x, double dx) {
  typedef libm_consts K;
  if (x < 0) dx = -dx;
  double u = TABX_BIG + fabs(x);
  x = fabs(x) - (u - TABX_BIG) + dx;
  double xx = x * x;
  double s = fma(x * xx, fma(xx, K::sn5, K::sn3), x);
  double c = xx * fma(fma(xx, K::cs6, K::cs4), xx, K::cs2);
  const double* e = sc_entry(u);  // SN, SSN, CS, CCS
  double cor = fma(-e[0], s, fma(-e[2], c, fma(-s, e[1], e[3])));
  return e[2] + cor;
}

TABX_HD double libm_do_sin(double x, double dx) {
  typedef libm_consts K;
  double xold = x;
  if (fabs(x) < 0.126) return taylor_sin(x * x, x, dx);
  if (x <= 0) dx = -dx;
  double u = TABX_BIG + fabs(x);
  x = fabs(x) - (u - TABX_BIG);
  double xx = x * x;
  double s = x + fma(x * xx, fma(xx, K::sn5, K::sn3), dx);
  double c = fma(x, dx, xx * fma(fma(xx, K::cs6, K::cs4), xx, K::cs2));
  const double* e = sc_entry(u);
  double cor = fma(e[2], s, fma(-e[0], c, fma(s, e[3], e[1])));
  return copysign(e[0] + cor, xold);
}

TABX_HD int libm_reduce(double x, double* a, double* da) {
  double t = fma(x, TABX_HPINV, TABX_TOINT);
  double xn = t - TABX_TOINT;
  double y = fma(-xn, TABX_MP2, fma(-xn, TABX_MP1, x));
  int n = (int)(d_to_bits(t) & 3);
  double t2 = fma(-xn, TABX_PP3, y);
  double db = fma(-xn, TABX_PP3, y - t2);
  double b = fma(-xn, TABX_PP4, t2);
  db = db + fma(-xn, TABX_PP4, t2 - b);
  *a = b;
  *da = db;
  return n;
}

TABX_HD double libm_do_sincos(double a, double da, int n) {
  double r = (n & 1) ? libm_do_cos(a, da) : libm_do_sin(a, da);
  return (n & 2) ? -r : r;
}

TABX_HD_CALL double libm_sin(double x) {
  uint32_t k = (uint32_t)(d_to_bits(x) >> 32) & 0x7fffffffu;
  if (k < 0x3e500000u) return x;
  if (k < 0x3feb6000u) return libm_do_sin(x, 0.0);
  if (k < 0x400368fdu) return copysign(libm_do_cos(TABX_HP0 - fabs(x), TABX_HP1), x);
  if (k < 0x419921FBu) {
    double a, da;
    int n = libm_reduce(x, &a, &da);
    return libm_do_sincos(a, da, n);
  }
  return sin(x);
}

TABX_HD_CALL double libm_cos(double x) {
  uint32_t k = (uint32_t)(d_to_bits(x) >> 32) & 0x7fffffffu;
  if (k < 0x3e400000u) return 1.0;
  if (k < 0x3feb6000u) return libm_do_cos(x, 0.0);
  if (k < 0x400368fdu) {
    double y = TABX_HP0 - fabs(x);
    double a = y + TABX_HP1;
    double da = (y - a) + TABX_HP1;
    return libm_do_sin(a, da);
  }
  if (k < 0x419921FBu) {
    double a, da;
    int n = libm_reduce(x, &a, &da);
    return libm_do_sincos(a, da, n + 1);
  }
  return cos(x);
}

// do_sin with its small-argument Taylor branch evaluated alongside the table
// path and selected, so lanes of a warp never diverge on it.
TABX_HD double libm_do_sin_sel(double x, double dx) {
  typedef libm_consts K;
  const double tay = taylor_sin(x * x, x, dx);
  const double ax = fabs(x);
  const double d = x <= 0 ? -dx : dx;
  const double u = TABX_BIG + ax;
  const double xr = ax - (u - TABX_BIG);
  const double xx = xr * xr;
  const double s = xr + fma(xr * xx, fma(xx, K::sn5, K::sn3), d);
  const double c = fma(xr, d, xx * fma(fma(xx, K::cs6, K::cs4), xx, K::cs2));
  const double* e = sc_entry(u);
  const double cor = fma(e[2], s, fma(-e[0], c, fma(s, e[3], e[1])));
  const double tab = copysign(e[0] + cor, x);
  return ax < 0.126 ? tay : tab;
}

// (sin x, cos x), each component exactly libm_sin(x) / libm_cos(x), with
// warp-uniform control flow: glibc picks, by |x|, the arguments of one
// do_sin and one do_cos evaluation (|x| < 0.855: (x, 0) for both; < 2.426:
// cos-of-complement arguments; else the Cody-Waite reduction, quadrant n)
// and how their results map to sin and cos.  Here every lane computes the
// three argument sets, selects its own, runs do_sin and do_cos once, and
// selects the outputs -- the same float64 operations per lane as the
// branchy reference, without serialising a warp over its lanes' ranges.
struct sincos_t {
  double s, c;
};
#if defined(__CUDACC__) && defined(TABX_INLINE_SINCOS)
static __host__ __device__ __forceinline__ sincos_t libm_sincos(double x) {
#else
TABX_HD_CALL sincos_t libm_sincos(double x) {
#endif
  sincos_t r;
  const uint32_t k = (uint32_t)(d_to_bits(x) >> 32) & 0x7fffffffu;
  if (k >= 0x419921FBu) {  // outside the restated range (never a heading)
    r.s = libm_sin(x);
    r.c = libm_cos(x);
    return r;
  }
  const bool r1 = k < 0x3feb6000u, r2 = !r1 && k < 0x400368fdu;
  double a3, da3;
  const int n = libm_reduce(x, &a3, &da3);
  const double y = TABX_HP0 - fabs(x);
  const double a2 = y + TABX_HP1;
  const double da2 = (y - a2) + TABX_HP1;
  const double sa = r1 ? x : (r2 ? a2 : a3), sda = r1 ? 0.0 : (r2 ? da2 : da3);
  const double ca = r1 ? x : (r2 ? y : a3), cda = r1 ? 0.0 : (r2 ? TABX_HP1 : da3);
  const double vs = libm_do_sin_sel(sa, sda);
  const double vc = libm_do_cos(ca, cda);
  if (r1) {
    r.s = vs;
    r.c = vc;
  } else if (r2) {
    r.s = copysign(vc, x);
    r.c = vs;
  } else {
    const double s0 = (n & 1) ? vc : vs;
    const double c0 = ((n + 1) & 1) ? vc : vs;
    r.s = (n & 2) ? -s0 : s0;
    r.c = ((n + 1) & 2) ? -c0 : c0;
  }
  if (k < 0x3e500000u) r.s = x;
  if (k < 0x3e400000u) r.c = 1.0;
  return r;
}

// numpy.maximum / numpy.minimum for non-NaN operands (loops_minmax: in1 >= in2 ? in1 : in2)
TABX_HD double np_max(double a, double b) { return a >= b ? a : b; }
TABX_HD double np_min(double a, double b) { return a <= b ? a : b; }
// numpy.clip: minimum(maximum(x, lo), hi)
TABX_HD double np_clip(double x, double lo, double hi) { return np_min(np_max(x, lo), hi); }

// numpy.remainder for doubles (npy_divmod): sign follows the divisor.
TABX_HD double np_remainder(double a, double b) {
  double m = fmod(a, b);
  if (m != 0.0) {
    if ((b < 0.0) != (m < 0.0)) m += b;
  } else {
    m = copysign(0.0, b);
  }
  return m;
}

// numpy pairwise_sum over v[0..n) starting from 0.0 (n <= 128 block form).
TABX_HD double pairwise_block(const double* v, int n) {
  if (n < 8) {
    double r = 0.0;
    for (int i = 0; i < n; ++i) r += v[i];
    return r;
  }
  double r0 = v[0], r1 = v[1], r2 = v[2], r3 = v[3];
  double r4 = v[4], r5 = v[5], r6 = v[6], r7 = v[7];
  int i = 8;
  int lim = n - (n % 8);
  for (; i < lim; i += 8) {
    r0 += v[i + 0]; r1 += v[i + 1]; r2 += v[i + 2]; r3 += v[i + 3];
    r4 += v[i + 4]; r5 += v[i + 5]; r6 += v[i + 6]; r7 += v[i + 7];
  }
  double r = ((r0 + r1) + (r2 + r3)) + ((r4 + r5) + (r6 + r7));
  for (; i < n; ++i) r += v[i];
  return r;
}

// Full pairwise rule for n <= 256 (TABX_MAX_UNITS): the top split leaves a
// head of <= 128 and a tail of <= 135, which splits once more.
TABX_HD double pairwise_sum(const double* v, int n) {
  if (n <= 128) return pairwise_block(v, n);
  int h = n / 2;
  h -= h % 8;
  double a, b;
  if (h <= 128) {
    a = pairwise_block(v, h);
  } else {
    int h2 = h / 2;
    h2 -= h2 % 8;
    a = pairwise_block(v, h2) + pairwise_block(v + h2, h - h2);
  }
  int m = n - h;
  if (m <= 128) {
    b = pairwise_block(v + h, m);
  } else {
    int h2 = m / 2;
    h2 -= h2 % 8;
    b = pairwise_block(v + h, h2) + pairwise_block(v + h + h2, m - h2);
  }
  return a + b;
}

}  // namespace tabx
