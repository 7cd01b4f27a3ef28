// Bit-exact numpy float64 arctan2 / tanh / sin / cos for the coherence
// directions (guide.eigen_2x2, guide.py:123-136: phi = 0.5 * arctan2(2b, a - c),
// v = (-sin phi, cos phi); guide.py:350 / make_spline: tanh((hi - lo) / lam)).
//
// The coherence fill order hinges on these: at deadlock shells of the smart
// order the top-two confidences can differ by 1 ulp, so g must be the very
// bits numpy produces.  What numpy runs on the
// reference's x86-64 AVX512_SKX hosts, and what is restated here:
//
//   np.arctan2  Intel SVML __svml_atan28_ha: |y| / |x| split at 7/16, 11/16,
//               19/16, 39/16 into atan(c) + atan((|y| - c|x|) / (|x| + c|y|)),
//               the quotient from vrcp14pd + two Newton steps + a remainder
//               correction, an even/odd split degree-20 polynomial, and the
//               quadrant fix-up with pi in two parts.  vrcp14pd itself is a
//               table of the top 16 mantissa bits (rcp14_np).
//   np.tanh     SVML __svml_tanh8: 16 intervals selected by the exponent and
//               top 3 mantissa bits, degree-16 polynomial in |x| - centre.
//   np.sin/cos  glibc 2.39 libm (sysdeps/ieee754/dbl-64/s_sin.c, FMA build):
//               |x| < 2^-26 / 2^-27 shortcuts, TAYLOR_SIN below 0.126,
//               do_sin / do_cos on the 1/128-spaced __sincostab double-double
//               table, and pi/2 - |x| (hp0 + hp1) up to 2.426265.
//
// Constants and FMA placement follow the machine code of those builds; the
// tables are captured by tools/gen_np_tables.py (gf_np_tables.h).  Checked
// against numpy on >= 10 M inputs per function by tests/test_exactmath.py.
// Domain notes: sin_np / cos_np cover |x| <= 2.426 (phi is in [-pi/2, pi/2]);
// beyond that they fall back to the C library's sin / cos.  atan2_np restates
// the vector path and the IEEE special cases (zeros, infinities, NaN); finite
// inputs outside 2^-1020 <= |v| < 2^993 are rescaled by a power of two first.
//
// Like gf_math.cuh: compile without FP contraction; fma() is written out.
#pragma once

#include "gf_math.cuh"
#include "gf_np_tables.h"

namespace gf {

#if defined(__CUDACC__)
__device__ static const uint32_t d_rcp14_words[4096] = GF_RCP14_WORDS;
__device__ static const uint16_t d_rcp14_anchors[1024] = GF_RCP14_ANCHORS;
__device__ static const uint64_t d_tanh_tab[18 * 16] = GF_TANH_TABLE;
__device__ static const uint64_t d_sincos_tab[440] = GF_SINCOS_TABLE;
#endif
static const uint32_t h_rcp14_words[4096] = GF_RCP14_WORDS;
static const uint16_t h_rcp14_anchors[1024] = GF_RCP14_ANCHORS;
static const uint64_t h_tanh_tab[18 * 16] = GF_TANH_TABLE;
static const uint64_t h_sincos_tab[440] = GF_SINCOS_TABLE;

GF_HD uint32_t rcp14_word(int k) {
#if defined(__CUDA_ARCH__)
  return __ldg(&d_rcp14_words[k]);
#else
  return h_rcp14_words[k];
#endif
}
GF_HD int rcp14_anchor(int b) {
#if defined(__CUDA_ARCH__)
  return (int)d_rcp14_anchors[b];
#else
  return (int)h_rcp14_anchors[b];
#endif
}
GF_HD double tanh_tab(int row, int i) {
#if defined(__CUDA_ARCH__)
  return as_d(__ldg(reinterpret_cast<const unsigned long long*>(&d_tanh_tab[16 * row + i])));
#else
  return as_d(h_tanh_tab[16 * row + i]);
#endif
}
GF_HD double sincos_tab(int i) {
#if defined(__CUDA_ARCH__)
  return as_d(__ldg(reinterpret_cast<const unsigned long long*>(&d_sincos_tab[i])));
#else
  return as_d(h_sincos_tab[i]);
#endif
}
GF_HD int popc32(uint32_t v) {
#if defined(__CUDA_ARCH__)
  return __popc(v);
#else
  return __builtin_popcount(v);
#endif
}

// vrcp14pd for a positive normal d: exact for powers of two, otherwise a
// 16-bit mantissa that depends only on the top 16 mantissa bits of d.
GF_HD double rcp14_np(double d) {
  const uint64_t u = as_u(d);
  const uint64_t m = u & 0xfffffffffffffULL;
  const int e = (int)((u >> 52) & 0x7ff);
  if (m == 0) return as_d((uint64_t)(2046 - e) << 52);
  const int i = (int)(m >> 36);
  int g = rcp14_anchor(i >> 6);
  const int n = i & 63;  // differences d[64 b .. i - 1]
  for (int w = 0; w < 4; ++w) {
    const int cnt = n - 16 * w;
    if (cnt <= 0) break;
    uint32_t word = rcp14_word((i >> 6) * 4 + w);
    if (cnt < 16) word &= (1u << (2 * cnt)) - 1u;
    g -= popc32(word & 0x55555555u) + 2 * popc32(word & 0xaaaaaaaau);
  }
  return as_d(((uint64_t)(2045 - e) << 52) | ((uint64_t)g << 36));
}

// __svml_atan28_ha vector path; needs 2^-1020 <= |x|, |y| < 2^993.
GF_HD double atan2_np_main(double y, double x) {
  const double ax = fabs(x), ay = fabs(y);
  const uint64_t sx = as_u(x) & 0x8000000000000000ULL;
  const uint64_t sy = as_u(y) & 0x8000000000000000ULL;
  const bool k1 = 0.6875 * ax < ay, k5 = 0.4375 * ax < ay;
  const bool k2 = 1.1875 * ax < ay, k3 = 2.4375 * ax < ay;
  double c, hi, lo;
  if (k2) {
    c = k3 ? 1.0 : 1.5;
    hi = k3 ? as_d(0x3ff921fb54442d18ULL) : as_d(0x3fef730bd281f69bULL);  // pi/2, atan 1.5
    lo = k3 ? as_d(0x3c91a62633145c07ULL) : as_d(0x3c7007887af0cbbdULL);
  } else {
    c = k1 ? 1.0 : 0.5;
    hi = k1 ? as_d(0x3fe921fb54442d18ULL) : as_d(0x3fddac670561bb4fULL);  // pi/4, atan 0.5
    lo = k1 ? as_d(0x3c81a62633145c07ULL) : as_d(0x3c7a2b7f222f65e2ULL);
  }
  double d = k3 ? 0.0 : ax;
  double n = k3 ? 0.0 : ay;
  if (k5) {
    d = fma_rn(c, ay, d);
    n = fma_rn(-c, ax, n);
  }
  const double r0 = rcp14_np(d);
  const double e0 = fma_rn(-d, r0, 1.0);
  const double r1 = fma_rn(e0, r0, r0);
  const double e1 = fma_rn(-r1, d, 1.0);
  const double r2 = fma_rn(e1, r1, r1);
  const double q = n * r2;
  const double q2 = q * q;
  const double rem = fma_rn(-q, d, n);
  const double q4 = q2 * q2;
  double corr = rem * r2;
  if (k5) corr = corr + lo;
  double A = fma_rn(as_d(0x3f8be4fbe6733718ULL), q4, as_d(0x3fa6ad5558fe19c9ULL));
  double B = fma_rn(as_d(0xbfa04cd71f92185eULL), q4, as_d(0xbfaa9e755ca13d23ULL));
  A = fma_rn(q4, A, as_d(0x3fae12f1edf7c393ULL));
  B = fma_rn(q4, B, as_d(0xbfb1108d326c68edULL));
  A = fma_rn(q4, A, as_d(0x3fb3b132b731e73aULL));
  B = fma_rn(q4, B, as_d(0xbfb745d119677a4fULL));
  A = fma_rn(q4, A, as_d(0x3fbc71c719f99f96ULL));
  B = fma_rn(q4, B, as_d(0xbfc2492492441a21ULL));
  A = fma_rn(q4, A, as_d(0x3fc9999999998f43ULL));
  B = fma_rn(q4, B, as_d(0xbfd5555555555552ULL));
  const double P = fma_rn(q2, A, B);
  const double Pq2 = P * q2;
  if (sx) corr = corr + as_d(0x3ca1a64000000000ULL ^ sx);  // -pi lo
  const double t = fma_rn(q, Pq2, corr);
  double s = q + t;
  if (k5) s = s + hi;
  s = as_d(as_u(s) ^ sx);
  if (sx) s = s + as_d(0x400921fb54442d18ULL);  // pi hi
  return as_d(as_u(s) | sy);
}

GF_HD bool atan2_in_range(double v) {
  const uint32_t h = (uint32_t)(as_u(v) >> 32) & 0x7fffffffu;
  return h >= 0x00300000u && h < 0x7e000000u;
}

// numpy float64 arctan2 (SVML __svml_atan28_ha), bit-exact.
GF_HD double atan2_np(double y, double x) {
  if (atan2_in_range(x) && atan2_in_range(y)) return atan2_np_main(y, x);
  const double PI = as_d(0x400921fb54442d18ULL), PI2 = as_d(0x3ff921fb54442d18ULL);
  if (x != x || y != y) return x + y;
  const uint64_t sy = as_u(y) & 0x8000000000000000ULL;
  const bool xneg = (as_u(x) >> 63) != 0;
  const double ax = fabs(x), ay = fabs(y);
  double r;
  if (ay == 0.0) {
    r = xneg ? PI : 0.0;
  } else if (ax == 0.0) {
    r = PI2;
  } else if (isinf(ay)) {
    r = isinf(ax) ? (xneg ? as_d(0x4002d97c7f3321d2ULL) : as_d(0x3fe921fb54442d18ULL)) : PI2;
  } else if (isinf(ax)) {
    r = xneg ? PI : 0.0;
  } else {
    // finite, non-zero, outside the vector path's exponent window: scale both
    const int ex = (int)((as_u(ax) >> 52) & 0x7ff), ey = (int)((as_u(ay) >> 52) & 0x7ff);
    const int shift = 1023 - (ex > ey ? ex : ey);  // |shift| <= 1076: two exact steps
    const int s1 = shift / 2, s2 = shift - s1;
    const double xs = (x * pow2i(s1)) * pow2i(s2), ys = (y * pow2i(s1)) * pow2i(s2);
    if (atan2_in_range(xs) && atan2_in_range(ys)) return atan2_np_main(ys, xs);
    // one operand is negligible next to the other
    if (fabs(ys) > fabs(xs)) {
      r = PI2;
    } else {
      const double q = fabs(ys) / fabs(xs);
      r = xneg ? PI - q : q;
    }
  }
  return as_d(as_u(r) | sy);
}

// numpy float64 tanh (SVML __svml_tanh8), bit-exact.
GF_HD double tanh_np(double x) {
  const uint64_t u = as_u(x);
  const uint32_t h = (uint32_t)(u >> 32) & 0x7ff80000u;
  if (h > 0x7fe00000u) {
    if (x != x) return x + x;
    return as_d(0x3ff0000000000000ULL | (u & 0x8000000000000000ULL));
  }
  int idx = (int)h - 0x3fc00000;
  idx = idx < 0 ? 0 : (idx > 0x780000 ? 0x780000 : idx);
  idx >>= 19;
  const double t = as_d(u & 0x7fffffffffffffffULL) - tanh_tab(0, idx);
  double p = tanh_tab(17, idx);
  for (int k = 16; k >= 1; --k) p = fma_rn(p, t, tanh_tab(k, idx));
  return as_d(as_u(p) | (u & 0x8000000000000000ULL));
}

// ---- glibc dbl-64 s_sin.c (FMA build) ----
namespace libm {
constexpr uint64_t kBig = 0x42c8000000000000ULL;  // 52776558133248.0
constexpr uint64_t kHp0 = 0x3ff921fb54442d18ULL, kHp1 = 0x3c91a62633145c07ULL;
constexpr uint64_t kS1 = 0xbfc5555555555555ULL, kS2 = 0x3f81111111110eceULL,
                   kS3 = 0xbf2a01a019db08b8ULL, kS4 = 0x3ec71de27b9a7ed9ULL,
                   kS5 = 0xbe5addffc2fcdf59ULL;
constexpr uint64_t kSn3 = 0xbfc5555555555515ULL, kSn5 = 0x3f811110e829872fULL;
constexpr uint64_t kCs2 = 0x3fe0000000000000ULL, kCs4 = 0xbfa5555555555535ULL,
                   kCs6 = 0x3f56c16bedd9e239ULL;
constexpr uint64_t kTaylorMax = 0x3fc020c49ba5e354ULL;  // 0.126
}  // namespace libm

GF_HD double taylor_sin(double xx, double a, double da) {
  using namespace libm;
  double p = fma_rn(xx, as_d(kS5), as_d(kS4));
  p = fma_rn(xx, p, as_d(kS3));
  p = fma_rn(xx, p, as_d(kS2));
  p = fma_rn(xx, p, as_d(kS1));
  const double t = fma_rn(p, a, -(0.5 * da));
  return a + fma_rn(xx, t, da);
}

GF_HD double libm_do_sin(double x, double dx) {
  using namespace libm;
  if (x <= 0.0) dx = -dx;
  const double ax = fabs(x);
  const double ux = ax + as_d(kBig);
  const int k = (int)((uint32_t)as_u(ux) << 2);
  const double xr = ax - (ux - as_d(kBig));
  const double xx = xr * xr;
  const double s = xr + fma_rn(xr * xx, fma_rn(xx, as_d(kSn5), as_d(kSn3)), dx);
  const double c =
      fma_rn(xr, dx, xx * fma_rn(xx, fma_rn(xx, as_d(kCs6), as_d(kCs4)), as_d(kCs2)));
  const double sn = sincos_tab(k), ssn = sincos_tab(k + 1), cs = sincos_tab(k + 2),
               ccs = sincos_tab(k + 3);
  double cor = fma_rn(s, ccs, ssn);
  cor = fma_rn(-c, sn, cor);
  cor = fma_rn(s, cs, cor);
  return copysign(sn + cor, x);
}

GF_HD double libm_do_cos(double x, double dx) {
  using namespace libm;
  if (x < 0.0) dx = -dx;
  const double ax = fabs(x);
  const double ux = ax + as_d(kBig);
  const int k = (int)((uint32_t)as_u(ux) << 2);
  const double xr = (ax - (ux - as_d(kBig))) + dx;
  const double xx = xr * xr;
  const double s = fma_rn(xr * xx, fma_rn(xx, as_d(kSn5), as_d(kSn3)), xr);
  const double c = xx * fma_rn(xx, fma_rn(xx, as_d(kCs6), as_d(kCs4)), as_d(kCs2));
  const double sn = sincos_tab(k), ssn = sincos_tab(k + 1), cs = sincos_tab(k + 2),
               ccs = sincos_tab(k + 3);
  double cor = fma_rn(-s, ssn, ccs);
  cor = fma_rn(-c, cs, cor);
  cor = fma_rn(-s, sn, cor);
  return cs + cor;
}

// numpy float64 sin (glibc libm), bit-exact for |x| <= 2.426265.
GF_HD double sin_np(double x) {
  using namespace libm;
  const uint32_t k = (uint32_t)(as_u(x) >> 32) & 0x7fffffffu;
  if (k < 0x3e500000u) return x;
  if (k < 0x3feb6000u) {
    if (fabs(x) < as_d(kTaylorMax)) return taylor_sin(x * x, x, 0.0);
    return libm_do_sin(x, 0.0);
  }
  if (k < 0x400368fdu) return copysign(libm_do_cos(as_d(kHp0) - fabs(x), as_d(kHp1)), x);
  return sin(x);  // outside the coherence domain
}

// numpy float64 cos (glibc libm), bit-exact for |x| <= 2.426265.
GF_HD double cos_np(double x) {
  using namespace libm;
  const uint32_t k = (uint32_t)(as_u(x) >> 32) & 0x7fffffffu;
  if (k < 0x3e400000u) return 1.0;
  if (k < 0x3feb6000u) return libm_do_cos(x, 0.0);
  if (k < 0x400368fdu) {
    const double y = as_d(kHp0) - fabs(x);
    const double a = y + as_d(kHp1);
    const double da = (y - a) + as_d(kHp1);
    if (fabs(a) < as_d(kTaylorMax)) return taylor_sin(a * a, a, da);
    return libm_do_sin(a, da);
  }
  return cos(x);  // outside the coherence domain
}

}  // namespace gf
