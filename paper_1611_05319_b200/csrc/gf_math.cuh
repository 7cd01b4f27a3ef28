// Bit-exact fp64 primitives of the reference's numpy decision path.
//
// The fill order of Guidefill hinges on fp64 comparisons (C > c, rw > 0,
// argmax C), so the weights must be bit-identical to what numpy computes
// on the host that runs the reference:
//
//   * np.exp(float64) on AVX512_SKX hosts dispatches to Intel SVML
//     __svml_exp8_ha (DOUBLE_exp_AVX512_SKX).  exp_np() restates its vector
//     path (fma round-toward-zero range reduction, 16-entry 2^(j/16) table,
//     degree-6 polynomial, vscalefpd) and its scalar rare path for
//     |x| >= 707.70327... (64-entry table, gradual-underflow splitting).
//   * np.hypot(float64) calls glibc hypot; glibc 2.39 on x86_64 uses the
//     Borges kernel without FMA.  hypot_np() restates it.
//   * np.sum over the K ball samples of one row uses numpy's pairwise
//     summation: blocks of <=128 with 8 interleaved accumulators combined as
//     ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7)) plus a sequential tail; longer
//     rows split recursively at n/2 rounded down to a multiple of 8.
//     PairwisePlan describes that tree for a given K.
//
// Every function here is __host__ __device__ so tests/test_exactmath.py can
// check the very same source against numpy on the CPU.  The translation
// unit must be compiled without FP contraction (nvcc --fmad=false,
// gcc -ffp-contract=off): every a*b+c below is meant as two roundings unless
// written as fma().
#pragma once

#include <stdint.h>
#include <math.h>
#include <string.h>
#include <fenv.h>

#include "gf_exp_tables.h"

#if defined(__CUDACC__)
#define GF_HD __host__ __device__ __forceinline__
#else
#define GF_HD inline
#endif

namespace gf {

#if defined(__CUDACC__)
__device__ static const uint64_t d_exp16[32] = GF_EXP16_TABLE;
__device__ static const uint64_t d_exp64[128] = GF_EXP64_TABLE;
#endif
static const uint64_t h_exp16[32] = GF_EXP16_TABLE;
static const uint64_t h_exp64[128] = GF_EXP64_TABLE;

GF_HD double as_d(uint64_t u) {
#if defined(__CUDA_ARCH__)
  return __longlong_as_double((long long)u);
#else
  double d; memcpy(&d, &u, 8); return d;
#endif
}
GF_HD uint64_t as_u(double d) {
#if defined(__CUDA_ARCH__)
  return (uint64_t)__double_as_longlong(d);
#else
  uint64_t u; memcpy(&u, &d, 8); return u;
#endif
}

GF_HD double tab16(int i) {
#if defined(__CUDA_ARCH__)
  return as_d(__ldg(reinterpret_cast<const unsigned long long*>(&d_exp16[i])));
#else
  return as_d(h_exp16[i]);
#endif
}
GF_HD double tab64(int i) {
#if defined(__CUDA_ARCH__)
  return as_d(__ldg(reinterpret_cast<const unsigned long long*>(&d_exp64[i])));
#else
  return as_d(h_exp64[i]);
#endif
}

GF_HD double fma_rn(double a, double b, double c) {
#if defined(__CUDA_ARCH__)
  return __fma_rn(a, b, c);
#else
  return fma(a, b, c);
#endif
}

GF_HD double fma_rz(double a, double b, double c) {
#if defined(__CUDA_ARCH__)
  return __fma_rz(a, b, c);
#else
  int old = fegetround();
  fesetround(FE_TOWARDZERO);
  volatile double r = fma(a, b, c);
  fesetround(old);
  return r;
#endif
}

// 2^e for e in the normal exponent range [-1022, 1023]
GF_HD double pow2i(int e) { return as_d((uint64_t)(e + 1023) << 52); }

// SVML scalar rare path (__svml_dexp_ha_cout_rare_internal)
GF_HD double exp_np_rare(double x) {
  const uint64_t ux = as_u(x);
  const int e = (int)((ux >> 52) & 0x7ff);
  if (e == 0x7ff) {
    if (ux == 0xfff0000000000000ULL) return 0.0;
    return x * x;
  }
  if (e <= 0x3ca) return x + 1.0;
  if (!(as_d(0x40862e42fefa39efULL) >= x)) return as_d(0x7fefffffffffffffULL) * as_d(0x7fefffffffffffffULL);
  if (x < as_d(0xc0874910d52d3051ULL)) {
    const double t = as_d(0x0010000000000001ULL);
    return t * t;
  }
  const double t = x * as_d(0x40571547652b82feULL) + as_d(0x4338000000000000ULL);
  const uint32_t lo32 = (uint32_t)as_u(t);
  const int j = (int)(lo32 & 0x3f);
  const double kd = t - as_d(0x4338000000000000ULL);
  double r = x - kd * as_d(0x3f862e42fefa0000ULL);
  r = r - kd * as_d(0x3d1cf79abc9e3b3aULL);
  double p = as_d(0x3f56c16a1c2a3ffdULL) * r;
  p = p + as_d(0x3f8111123aaf20d3ULL);
  p = p * r;
  p = p + as_d(0x3fa5555555558fccULL);
  p = p * r;
  p = p + as_d(0x3fc55555555548f8ULL);
  p = p * r;
  p = p + as_d(0x3fe0000000000000ULL);
  p = p * r;
  p = p * r;
  p = p + r;
  const double thi = tab64(2 * j), tlo = tab64(2 * j + 1);
  p = p + tlo;
  p = p * thi;
  const uint32_t n = lo32 >> 6;
  if (x < as_d(0xc086232bdd7abcd2ULL)) {
    const uint32_t ec = (n + 0x43b) & 0x7ff;
    const double sc = as_d((uint64_t)ec << 52);
    const double a = p * sc;
    const double b = sc * thi;
    const double s = b + a;
    if (ec <= 0x32) return s * as_d(0x3c30000000000000ULL);
    const double lo = (b - s) + a;
    const double tt = s * as_d(0x41f8000000000000ULL);
    const double h = (s + tt) - tt;
    const double l = lo + (s - h);
    return h * as_d(0x3c30000000000000ULL) + l * as_d(0x3c30000000000000ULL);
  }
  const uint32_t ed = (n + 0x3ff) & 0x7ff;
  p = p + thi;
  if (ed > 0x7fe) {
    const uint32_t e2 = (ed - 1) & 0x7ff;
    return (p * as_d((uint64_t)e2 << 52)) * 2.0;
  }
  return p * as_d((uint64_t)ed << 52);
}

// numpy float64 exp on AVX512_SKX hosts (SVML __svml_exp8_ha), bit-exact.
GF_HD double exp_np(double x) {
  const double ax = fabs(x);
  if (ax >= as_d(0x40861da04cbafe44ULL)) return exp_np_rare(x);
  if (x != x) return x + x;
  const double shifter = as_d(0x42f8000000003ff0ULL);
  const double z = fma_rz(x, as_d(0x3ff71547652b82feULL), shifter);
  const double N = z - shifter;
  const int j = (int)(as_u(z) & 15);
  double r = fma_rn(-N, as_d(0x3fe62e42fefa39efULL), x);
  r = fma_rn(-as_d(0x3c7abc9e3b39803fULL), N, r);
  r = as_d(as_u(r) & 0xbfffffffffffffffULL);
  const double r2 = r * r;
  const double p1 = fma_rn(as_d(0x3f57411836940c04ULL), r, as_d(0x3f81101cbbc265c0ULL));
  const double p2 = fma_rn(as_d(0x3fa55557242d68feULL), r, as_d(0x3fc5555553939732ULL));
  const double p3 = fma_rn(as_d(0x3fe000000000d008ULL), r, as_d(0x3fefffffffffff70ULL));
  double q = fma_rn(r2, p1, p2);
  q = fma_rn(r2, q, p3);
  const double thi = tab16(j), tlo = tab16(16 + j);
  double s = fma_rn(q, r, tlo);
  s = fma_rn(thi, s, thi);
  return s * pow2i((int)floor(N));
}

// glibc 2.39 hypot (sysdeps/ieee754/dbl-64/e_hypot.c, non-FMA kernel).
GF_HD double hypot_kernel(double ax, double ay) {
  double h = sqrt(ax * ax + ay * ay);
  double t1, t2;
  if (h <= 2.0 * ay) {
    const double delta = h - ay;
    t1 = ax * (2.0 * delta - ax);
    t2 = (delta - 2.0 * (ax - ay)) * delta;
  } else {
    const double delta = h - ax;
    t1 = 2.0 * delta * (ax - 2.0 * ay);
    t2 = (4.0 * delta - ay) * ay + delta * delta;
  }
  h -= (t1 + t2) / (2.0 * h);
  return h;
}

GF_HD double hypot_np(double x, double y) {
  if (!isfinite(x) || !isfinite(y)) {
    if (isinf(x) || isinf(y)) return INFINITY;
    return x + y;
  }
  x = fabs(x);
  y = fabs(y);
  double ax = x < y ? y : x;
  double ay = x < y ? x : y;
  const double SCALE = 0x1p-600, LARGE = 0x1p+511, TINY = 0x1p-511, EPS = 0x1p-54;
  if (ax > LARGE) {
    if (ay <= ax * EPS) return ax + ay;
    return hypot_kernel(ax * SCALE, ay * SCALE) / SCALE;
  }
  if (ay < TINY) {
    if (ax >= ay / EPS) return ax + ay;
    return hypot_kernel(ax / SCALE, ay / SCALE) * SCALE;
  }
  if (ay <= ax * EPS) return ax + ay;
  return hypot_kernel(ax, ay);
}

// ------------------------------------------------------------------------
// numpy pairwise summation tree for one row of K elements.
//
// Leaves are either "blocked" (n >= 8: 8 interleaved accumulators, tree,
// then sequential tail) or "short" (n < 8: sequential from 0.0).  Leaf
// starts are multiples of 8, so element k always belongs to accumulator
// lane k % 8.  The combine tree is a postfix program over leaf results.
constexpr int kMaxLeaves = 4;
constexpr int kMaxProg = 2 * kMaxLeaves;

struct PairwisePlan {
  int n_leaves;
  int leaf_lo[kMaxLeaves];
  int leaf_n[kMaxLeaves];
  int n_prog;
  int prog[kMaxProg];  // >= 0: push leaf i; -1: pop two, push (a + b)
};

inline void plan_rec(PairwisePlan& p, int lo, int n) {
  if (n <= 128) {
    p.leaf_lo[p.n_leaves] = lo;
    p.leaf_n[p.n_leaves] = n;
    p.prog[p.n_prog++] = p.n_leaves++;
    return;
  }
  int n2 = n / 2;
  n2 -= n2 % 8;
  plan_rec(p, lo, n2);
  plan_rec(p, lo + n2, n - n2);
  p.prog[p.n_prog++] = -1;
}

inline PairwisePlan make_plan(int K) {
  PairwisePlan p;
  memset(&p, 0, sizeof(p));
  plan_rec(p, 0, K);
  return p;
}

// Sequential reference implementation of the plan (host tests and
// single-thread device use).  a[] holds the K row elements.
GF_HD double leaf_sum(const double* a, int lo, int n) {
  if (n < 8) {
    double res = 0.0;
    for (int i = 0; i < n; ++i) res += a[lo + i];
    return res;
  }
  double r[8];
  for (int l = 0; l < 8; ++l) r[l] = a[lo + l];
  int i = 8;
  for (; i < n - (n % 8); i += 8)
    for (int l = 0; l < 8; ++l) r[l] += a[lo + i + l];
  double res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
  for (; i < n; ++i) res += a[lo + i];
  return res;
}

GF_HD double plan_sum(const PairwisePlan& p, const double* a) {
  double stack[kMaxLeaves];
  int sp = 0;
  for (int i = 0; i < p.n_prog; ++i) {
    const int op = p.prog[i];
    if (op >= 0) {
      stack[sp++] = leaf_sum(a, p.leaf_lo[op], p.leaf_n[op]);
    } else {
      const double b = stack[--sp];
      const double a0 = stack[--sp];
      stack[sp++] = a0 + b;
    }
  }
  return stack[0];
}

}  // namespace gf
