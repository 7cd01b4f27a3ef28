// Radius-specialised ball evaluators for the shell loop (r <= 6, K <= 128:
// one numpy pairwise leaf).  With K a compile-time constant every loop is
// unrolled, so the fetches of an item are issued before any of them is
// consumed and the weight arithmetic overlaps their latency.
//
// Both produce exactly engine._BallSampler.gather's rw / tw bits
// (engine.py:175-199); colours are weighted averages in fp64 (stored fp32).
#pragma once

#include "gf_sampler.cuh"

namespace gf {

__host__ __device__ constexpr int disk_count(int r) {
  int k = 0;
  for (int m = -r; m <= r; ++m)
    for (int n = -r; n <= r; ++n)
      if (n * n + m * m <= r * r && (n != 0 || m != 0)) ++k;
  return k;
}

template <int R>
struct Ball {
  static constexpr int K = disk_count(R);
  static constexpr int KPL = (K + kGroup - 1) / kGroup;  // samples per lane, 8-lane item
  static constexpr int KPW = (K + 31) / 32;              // samples per lane, warp item
  static constexpr int N8 = K - K % 8;                   // pairwise: 8-accumulator part
  static constexpr int NT = K % 8;                       // pairwise: sequential tail
  static_assert(K <= 128, "one pairwise leaf");
};

// Lattice item (g = 0, integral centre) on a group of LG = 8 or 4 lanes.
// Lane j owns samples j, j+LG, j+2LG, ...; numpy's accumulator of sample k
// is k % 8, so with LG = 8 a lane holds accumulator j, with LG = 4 it holds
// accumulators j (even slots) and j+4 (odd slots), each summed in sample
// order in registers.  The accumulator tree ((r0+r1)+(r2+r3))+((r4+r5)+
// (r6+r7)) is three xor levels (LG = 8) or two plus the lane-local pair
// (LG = 4); the tail samples (k >= N8) are added in order from ballots of
// their readability.  tw is the host's constant P.tw0.
template <int R, int LG>
__device__ __forceinline__ void eval_lattice(const BallParams& P, const BallTables& T,
                                             const WorkSource& src, int glane, int sub, bool valid,
                                             int pi, int pj, SampleResult& out) {
  using B = Ball<R>;
  static_assert(LG == 8 || LG == 4, "8 or 4 lanes per item");
  constexpr int KPL = (B::K + LG - 1) / LG;
  int q[KPL];
  float4 v[KPL];
  // a ball that lies inside the lattice (the usual case) indexes its samples
  // by flat offset; near the border each sample is bounds-checked / wrapped
  const bool inner = pi >= R && pi + R < src.W && pj >= R && pj + R < src.H;
  const int p = pj * src.W + pi;
  if (__all_sync(0xffffffffu, inner || !valid)) {
    // the whole warp's items lie inside the lattice (warp-uniform branch)
#pragma unroll
    for (int t = 0; t < KPL; ++t) {
      const int k = glane + LG * t;
      q[t] = (valid && k < B::K) ? p + T.off[k] : -1;
    }
  } else {
#pragma unroll
    for (int t = 0; t < KPL; ++t) {
      const int k = glane + LG * t;
      q[t] = (valid && k < B::K)
                 ? (inner ? p + T.off[k]
                          : lattice_index(pi + T.ni[k], pj + T.mi[k], src.H, src.W, P.periodic))
                 : -1;
    }
  }
#ifdef GF_FINE_TRACE
  {
    if (q[0] == -2) asm volatile("trap;");
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(out.t0));
  }
#endif
#pragma unroll
  for (int t = 0; t < KPL; ++t)
    if (q[t] >= 0) v[t] = src.work[q[t]];
#ifdef GF_FINE_TRACE
  {
    if (__float_as_int(v[0].w) == -2 && q[0] >= 0) asm volatile("trap;");
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(out.t1));
  }
#endif
  unsigned okm = 0;  // bit t: sample glane + LG t readable
#pragma unroll
  for (int t = 0; t < KPL; ++t)
    if (q[t] >= 0 && __float_as_int(v[t].w) <= src.shell) okm |= 1u << t;
  // the 8-neighbours this lane sampled that are Inpaint and not yet in a
  // frontier: only those can be activated by a fill (tracker.py:42-79)
  unsigned inact = 0;
#pragma unroll
  for (int t = 0; t < KPL; ++t) {
    const int k = glane + LG * t;
    if (k < B::K && q[t] >= 0) {
      const int o = T.kn[k];
      if (o >= 0 && (__float_as_int(v[t].w) & ~kRotBit) == kStampInactive) inact |= 1u << o;
    }
  }
#pragma unroll
  for (int o = 1; o < LG; o <<= 1) inact |= __shfl_xor_sync(0xffffffffu, inact, o, LG);
  out.nb = inact | P.nb_unknown;
  double acc0 = 0.0, acc1 = 0.0;  // accumulators glane (and glane + 4 when LG == 4)
#pragma unroll
  for (int t = 0; t < B::N8 / LG; ++t)
    if ((okm >> t) & 1u) {  // + 0.0 for an unreadable sample would be the identity
      const double w = T.w0[glane + LG * t];
      if (LG == 8 || (t & 1) == 0) acc0 += w;
      else acc1 += w;
    }
  double acc;
  if constexpr (LG == 8) {
    acc = group_sum_tree(acc0);
  } else {
    acc0 = acc0 + __shfl_xor_sync(0xffffffffu, acc0, 1, LG);
    acc1 = acc1 + __shfl_xor_sync(0xffffffffu, acc1, 1, LG);
    acc0 = acc0 + __shfl_xor_sync(0xffffffffu, acc0, 2, LG);
    acc1 = acc1 + __shfl_xor_sync(0xffffffffu, acc1, 2, LG);
    acc = acc0 + acc1;
  }
  if constexpr (B::NT > 0) {
    constexpr int ts0 = B::N8 / LG, ts1 = (B::K - 1) / LG;  // slots holding the tail
    unsigned tb0 = (__ballot_sync(0xffffffffu, (okm >> ts0) & 1u) >> (LG * sub)) & ((1u << LG) - 1);
    unsigned tb1 = tb0;
    if constexpr (ts1 != ts0)
      tb1 = (__ballot_sync(0xffffffffu, (okm >> ts1) & 1u) >> (LG * sub)) & ((1u << LG) - 1);
#pragma unroll
    for (int e = 0; e < B::NT; ++e) {
      const int k = B::N8 + e;
      const unsigned tb = (k / LG == ts0) ? tb0 : tb1;
      if ((tb >> (k % LG)) & 1u) acc = acc + T.w0[k];
    }
  }
  // colour numerators: off the decision path (values only need 1e-4 and are
  // stored fp32), so they accumulate in fp32 with explicit FMAs -- the fp64
  // masses above keep numpy's exact bits
  float num[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
  for (int t = 0; t < KPL; ++t)
    if ((okm >> t) & 1u) {
      const float w = T.w0f[glane + LG * t];
      num[0] = __fmaf_rn(w, v[t].x, num[0]);
      num[1] = __fmaf_rn(w, v[t].y, num[1]);
      num[2] = __fmaf_rn(w, v[t].z, num[2]);
    }
  if (src.c3) {
#pragma unroll
    for (int t = 0; t < KPL; ++t)
      if ((okm >> t) & 1u) num[3] = __fmaf_rn(T.w0f[glane + LG * t], src.c3[q[t]], num[3]);
  }
  const double inv = (acc != 0.0) ? 1.0 / acc : 0.0;
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    float s = 0.f;
    if (c < 3 || src.c3) {
      s = num[c];
#pragma unroll
      for (int o = 1; o < LG; o <<= 1) s += __shfl_xor_sync(0xffffffffu, s, o, LG);
    }
    out.v[c] = (double)s * inv;
  }
  out.rw = acc;
  out.tw = P.tw0;
}

// Column wrap for the fill's ghost corners: |x| stays within r + 1 of the
// lattice, so a couple of conditional adds replace the 64-bit modulo.
__device__ __forceinline__ int wrap_col(int x, int W) {
  while (x < 0) x += W;
  while (x >= W) x -= W;
  return x;
}

// Rotated-ball item (g != 0) on a whole warp.  Sample k lives in lane
// k % 32, slot k / 32.  (ux, uy) = g / hypot(g) comes precomputed with g.
// Per slot: rotated offset -> ghost corners -> corner fetches issued ->
// weight (glibc hypot, SVML exp, division) computed while they fly.
// numpy's accumulator j = a_j + a_{j+8} + ... is rebuilt by lane j pulling
// a_{j+8t} from lane j + 8 (t % 4), slot t / 4.
template <int R>
__device__ __forceinline__ void eval_rot_warp(const BallParams& P, const BallTables& T,
                                              const WorkSource& src, int lane, double fi, double fj,
                                              double gx, double gy, double ux, double uy,
                                              SampleResult& out) {
  using B = Ball<R>;
  constexpr int KPW = B::KPW;
  double safe = 1.0, thr = 0.0;
  if (P.mu_inf) {
    const double nr2 = sqrt(gx * gx + gy * gy);
    safe = (nr2 == 0.0) ? 1.0 : nr2;
    double mloc = INFINITY;
#pragma unroll
    for (int s = 0; s < KPW; ++s) {
      const int k = lane + 32 * s;
      if (k < B::K) {
        double px = T.n[k], py = T.m[k];
        if (P.rotated) {
          px = T.n[k] * uy + T.m[k] * ux;
          py = (-T.n[k]) * ux + T.m[k] * uy;
        }
        const double d = ((-gy) * px + gx * py) / safe;
        mloc = min_prop(mloc, d * d);
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mloc = min_prop(mloc, __shfl_xor_sync(0xffffffffu, mloc, o));
    thr = mloc + P.tol_inf;
  }
  double w[KPW], wr[KPW];
  // colour path in fp32 (off the decision path, tolerance 1e-4): the sample
  // colour sv and, after the warp knows its largest readable weight, the
  // numerators with weights scaled by a power of two so the largest is in
  // [1, 2) -- tiny Eq. 3.2 weights (1e-61 in test_engine.py:77-139) never
  // underflow the dominant terms
  float sv[KPW][4];
#pragma unroll
  for (int s = 0; s < KPW; ++s) {
    const int k = lane + 32 * s;
    w[s] = 0.0;
    wr[s] = 0.0;
#pragma unroll
    for (int c = 0; c < 4; ++c) sv[s][c] = 0.f;
    if (k < B::K) {
      double px = T.n[k], py = T.m[k];
      if (P.rotated) {
        px = T.n[k] * uy + T.m[k] * ux;
        py = (-T.n[k]) * ux + T.m[k] * uy;
      }
      // ghost corners (grid.py:186-209), fetches issued before the weight
      const double X = fi + px, Y = fj + py;
      const double fx0 = floor(X), fy0 = floor(Y);
      const double tx = X - fx0, ty = Y - fy0;
      const int x0 = (int)fx0, y0 = (int)fy0;
      unsigned live = 0;  // bit c: corner c has weight and lies in the lattice
      bool outside = false;
      float4 v[4];
      float c3v[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const int a = c >> 1, b = c & 1;  // (x0,y0),(x0,y0+1),(x0+1,y0),(x0+1,y0+1)
        const double wc = (a ? tx : 1.0 - tx) * (b ? ty : 1.0 - ty);
        if (wc != 0.0) {
          const int cy = y0 + b;
          int cx = x0 + a;
          bool inside = cy >= 0 && cy < src.H;
          if (P.periodic) cx = wrap_col(cx, src.W);
          else inside = inside && cx >= 0 && cx < src.W;
          if (inside) {
            const int q = cy * src.W + cx;
            v[c] = src.work[q];
            if (src.c3) c3v[c] = src.c3[q];
            live |= 1u << c;
          } else {
            outside = true;
          }
        }
      }
      const double dist = hypot_np(px, py);
      double ws;
      if (P.mu_inf) {
        const double d = ((-gy) * px + gx * py) / safe;
        ws = (d * d <= thr) ? 1.0 / dist : 0.0;
      } else {
        const double d = (-gy) * px + gx * py;
        ws = exp_np((P.coef * d) * d) / dist;
      }
      w[s] = ws;
      bool ok = !outside;
#pragma unroll
      for (int c = 0; c < 4; ++c)
        if ((live >> c) & 1u) {
          const int a = c >> 1, b = c & 1;
          const float wc = (float)((a ? tx : 1.0 - tx) * (b ? ty : 1.0 - ty));
          ok = ok && __float_as_int(v[c].w) <= src.shell;
          sv[s][0] = __fmaf_rn(wc, v[c].x, sv[s][0]);
          sv[s][1] = __fmaf_rn(wc, v[c].y, sv[s][1]);
          sv[s][2] = __fmaf_rn(wc, v[c].z, sv[s][2]);
          sv[s][3] = __fmaf_rn(wc, c3v[c], sv[s][3]);
        }
      wr[s] = ok ? ws : 0.0;
    }
  }
  // binary exponent of the warp's largest readable weight (0 when none)
  int e_loc = -2000;
#pragma unroll
  for (int s = 0; s < KPW; ++s)
    if (wr[s] > 0.0) e_loc = max(e_loc, ilogb(wr[s]));
  const int e_max = __reduce_max_sync(0xffffffffu, e_loc);
  const int e_use = e_max < -1100 ? 0 : e_max;
  const double down = scalbn(1.0, -e_use);  // exact power of two
  float num[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
  for (int s = 0; s < KPW; ++s)
    if (wr[s] != 0.0) {
      const float wsf = (float)(wr[s] * down);
#pragma unroll
      for (int c = 0; c < 4; ++c) num[c] = __fmaf_rn(wsf, sv[s][c], num[c]);
    }
  double acc_rw = 0.0, acc_tw = 0.0;
#pragma unroll
  for (int t = 0; t < B::N8 / 8; ++t) {
    const int src_lane = (lane & 7) + 8 * (t & 3);
    acc_rw += __shfl_sync(0xffffffffu, wr[t >> 2], src_lane);
    acc_tw += __shfl_sync(0xffffffffu, w[t >> 2], src_lane);
  }
  double rw = group_sum_tree(acc_rw);
  double tw = group_sum_tree(acc_tw);
#pragma unroll
  for (int e = 0; e < B::NT; ++e) {
    const int i = B::N8 + e;
    rw = rw + __shfl_sync(0xffffffffu, wr[i >> 5], i & 31);
    tw = tw + __shfl_sync(0xffffffffu, w[i >> 5], i & 31);
  }
  if (e_max < -1000 && e_max > -2000) {
    // every readable weight is near the bottom of the fp64 range (high mu,
    // tiny r: Eq. 3.2 weights of ~1e-320): the scaling above would leave
    // the double range, and numpy's own products wr * v round to multiples
    // of 2^-1074 there.  Form those products in fp64 as numpy does; sums of
    // such tiny values are exact in any order.
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      double part = 0.0;
#pragma unroll
      for (int s = 0; s < KPW; ++s)
        if (wr[s] != 0.0) part += wr[s] * (double)sv[s][c];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
      out.v[c] = (c < 3 || src.c3) ? part / rw : 0.0;
    }
    out.rw = rw;
    out.tw = tw;
    return;
  }
  const double inv = (rw != 0.0) ? 1.0 / rw : 0.0;
  const double up = scalbn(1.0, e_use);
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    float sacc = 0.f;
    if (c < 3 || src.c3) {
      sacc = num[c];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) sacc += __shfl_xor_sync(0xffffffffu, sacc, o);
    }
    out.v[c] = ((double)sacc * up) * inv;
  }
  out.rw = rw;
  out.tw = tw;
}

}  // namespace gf
