// Ball sampler shared by the fill engine and the point-evaluation kernels.
//
// One item (frontier pixel) is evaluated by a group of 8 lanes.  Lane l owns
// ball samples k = l, l+8, l+16, ... which is exactly numpy's pairwise-sum
// accumulator assignment (element k -> accumulator k % 8), so the readable
// and total weight masses come out bit-identical to
// engine._BallSampler.gather (engine.py:175-199).  Geometry, weights and
// masses are fp64 without contraction; colours are accumulated in fp64 from
// the stored fp32 values.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>
#include <math.h>

#include "gf_math.cuh"

namespace gf {

constexpr int kMaxK = 440;  // disk of radius 12, centre excluded
constexpr int kGroup = 8;   // lanes per item

// stamp encoding (int32, one per pixel): readable at shell k <=> stamp <= k.
// Unfilled Inpaint pixels carry a marker whose bit 0 (kRotBit) records
// g != 0 (the item takes the rotated-ball path), so frontier entries know
// their path without reading the guide field.
constexpr int kStampReadable = 0;
constexpr int kRotBit = 1;
constexpr int kStampInactive = 0x7ffffff8;  // Inpaint, not in the frontier (| kRotBit)
constexpr int kStampActive = 0x7ffffffa;    // Inpaint, in the frontier (| kRotBit)
constexpr int kStampBystander = 0x7fffffff;
// frontier list entries: pixel index | kEntryRot when g != 0
constexpr uint32_t kEntryRot = 0x80000000u;
constexpr uint32_t kEntryPix = 0x7fffffffu;

__host__ __device__ __forceinline__ bool stamp_unfilled(int st) {
  return st >= kStampInactive && st < kStampBystander;
}

struct BallParams {
  int r, K;
  unsigned nb_unknown;  // 8-neighbours (NEIGHBOR_OFFSETS order) that are not ball samples
  double tw0;      // numpy pairwise sum of the g = 0 weights (the lattice-path tw)
  int rotated;   // rotated_ball (engine.py:150-164) vs axis_ball
  int periodic;  // periodic_x
  int mu_inf;
  double coef;     // -(mu*mu) / (2.0*float(r*r))      engine.py:147
  double tol_inf;  // 1e-12 * max(1.0, float(r*r))    engine.py:143
  PairwisePlan plan;
};

// Ball tables (offsets and the g = 0 weights 1/hypot(n, m) computed by the
// host with numpy), staged in shared memory by the kernels.
struct BallTables {
  double n[kMaxK];
  double m[kMaxK];
  double w0[kMaxK];
  float w0f[kMaxK];  // (float)w0: the fp32 colour numerators' weights
  int ni[kMaxK];  // the same offsets as integers (lattice path)
  int mi[kMaxK];
  signed char kn[kMaxK];  // sample k is 8-neighbour kn[k] of the centre, or -1
  int off[kMaxK];         // n + m * W (shell kernel's shared copy only): flat offsets
};

struct SampleResult {
  double rw, tw;  // readable / total weight mass (exact numpy bits)
  double v[4];    // weighted average colour, 0 where rw == 0
  unsigned nb;    // 8-neighbours that may need activation (lattice path: the
                  // ones Inpaint-inactive at the shell's start, plus those
                  // the ball does not sample); 0xff when unknown
#ifdef GF_FINE_TRACE
  unsigned long long t0, t1;  // fetch issued / first fetch arrived (phase trace)
#endif
};

// --------------------------------------------------------------- sources

// Working frame of the fill engine: float4 (c0, c1, c2, stamp bits) per
// pixel plus an optional 4th channel plane.
struct Px {
  float4 v;  // c0, c1, c2, stamp bits (WorkSource) / c0..c2, unused (RawSource)
  float c3;
};

struct WorkSource {
  const float4* work;  // frame base
  const float* c3;     // frame base or nullptr
  int H, W, C;
  int shell;
  __device__ __forceinline__ Px fetch(int q) const {
    Px r;
    r.v = work[q];
    r.c3 = c3 ? c3[q] : 0.f;
    return r;
  }
  __device__ __forceinline__ bool readable(const Px& x) const {
    return __float_as_int(x.v.w) <= shell;
  }
  __device__ __forceinline__ void accumulate(const Px& x, double wc, double* sv) const {
    sv[0] += wc * (double)x.v.x;
    sv[1] += wc * (double)x.v.y;
    sv[2] += wc * (double)x.v.z;
    sv[3] += wc * (double)x.c3;
  }
  __device__ __forceinline__ bool load(int q, double* v) const {
    const float4 px = work[q];
    if (__float_as_int(px.w) > shell) return false;
    v[0] = px.x;
    v[1] = px.y;
    v[2] = px.z;
    v[3] = c3 ? (double)c3[q] : 0.0;
    return true;
  }
};

// Raw float64 image + label lattice (point-evaluation API).
struct RawSource {
  const double* img;
  const uint8_t* lab;
  int H, W, C;
  struct RawPx {
    double c[4];
    bool ok;
  };
  __device__ __forceinline__ RawPx fetch(int q) const {
    RawPx r;
    r.ok = lab[q] == 0;
    const double* p = img + (size_t)q * C;
    for (int c = 0; c < 4; ++c) r.c[c] = c < C ? p[c] : 0.0;
    return r;
  }
  __device__ __forceinline__ bool readable(const RawPx& x) const { return x.ok; }
  __device__ __forceinline__ void accumulate(const RawPx& x, double wc, double* sv) const {
    for (int c = 0; c < 4; ++c) sv[c] += wc * x.c[c];
  }
  __device__ __forceinline__ bool load(int q, double* v) const {
    if (lab[q] != 0) return false;
    const double* p = img + (size_t)q * C;
    for (int c = 0; c < 4; ++c) v[c] = c < C ? p[c] : 0.0;
    return true;
  }
};

__device__ __forceinline__ int pos_mod(long long a, int W) {
  long long r = a % W;
  return (int)(r < 0 ? r + W : r);
}
__device__ __forceinline__ int pos_mod32(int a, int W) {
  const int r = a % W;
  return r < 0 ? r + W : r;
}

// Strict bilinear ghost sample at (X, Y), grid.py:186-210.  Returns ok; adds
// the interpolated colour into sv[] (only meaningful when ok).
template <class Src>
__device__ __forceinline__ bool ghost_sample(const Src& src, double X, double Y, int periodic,
                                             double* sv) {
  const double fx0 = floor(X), fy0 = floor(Y);
  const double tx = X - fx0, ty = Y - fy0;
  const long long x0 = (long long)fx0, y0 = (long long)fy0;
  const double wxs[2] = {1.0 - tx, tx};
  const double wys[2] = {1.0 - ty, ty};
  bool ok = true;
#pragma unroll
  for (int a = 0; a < 2; ++a) {
#pragma unroll
    for (int b = 0; b < 2; ++b) {
      const double wc = wxs[a] * wys[b];
      if (wc == 0.0 || !ok) continue;
      const long long cx = x0 + a, cy = y0 + b;
      int col;
      bool inside;
      if (periodic) {
        inside = (cy >= 0) && (cy < src.H);
        col = pos_mod(cx, src.W);
      } else {
        inside = (cx >= 0) && (cx < src.W) && (cy >= 0) && (cy < src.H);
        col = (int)cx;
      }
      if (!inside) {
        ok = false;
        continue;
      }
      double v[4];
      if (!src.load((int)cy * src.W + col, v)) {
        ok = false;
        continue;
      }
#pragma unroll
      for (int c = 0; c < 4; ++c) sv[c] += wc * v[c];
    }
  }
  return ok;
}

// Lattice sample (g = 0): the only live corner is (x, y) itself.
template <class Src>
__device__ __forceinline__ bool lattice_sample(const Src& src, int x, int y, int periodic,
                                               double* sv) {
  if (y < 0 || y >= src.H) return false;
  if (periodic) {
    x = pos_mod(x, src.W);
  } else if (x < 0 || x >= src.W) {
    return false;
  }
  double v[4];
  if (!src.load(y * src.W + x, v)) return false;
#pragma unroll
  for (int c = 0; c < 4; ++c) sv[c] += v[c];
  return true;
}

__device__ __forceinline__ double group_sum_tree(double v) {
  // ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7)) lands in lane 0 of the group
  v = v + __shfl_xor_sync(0xffffffffu, v, 1, kGroup);
  v = v + __shfl_xor_sync(0xffffffffu, v, 2, kGroup);
  v = v + __shfl_xor_sync(0xffffffffu, v, 4, kGroup);
  return v;
}

__device__ __forceinline__ double min_prop(double a, double b) {
  return (a != a || b != b) ? (a + b) : fmin(a, b);
}

// Corner set of one ghost sample (grid.py:186-209): index of each corner to
// fetch (-1: not live, nothing to read) and whether a live corner falls
// outside the lattice (the sample is then unreadable).  No loads here, so
// the fetches of all corners of all samples can be issued back to back.
struct Corners {
  int q[4];
  double w[4];
  bool outside;
};

__device__ __forceinline__ void ghost_corners(double X, double Y, int H, int W, int periodic,
                                              Corners& c) {
  const double fx0 = floor(X), fy0 = floor(Y);
  const double tx = X - fx0, ty = Y - fy0;
  const long long x0 = (long long)fx0, y0 = (long long)fy0;
  const double wxs[2] = {1.0 - tx, tx};
  const double wys[2] = {1.0 - ty, ty};
  c.outside = false;
#pragma unroll
  for (int a = 0; a < 2; ++a) {
#pragma unroll
    for (int b = 0; b < 2; ++b) {
      const int i = 2 * a + b;  // reference corner order (x0,y0),(x0,y0+1),(x0+1,y0),(x0+1,y0+1)
      const double wc = wxs[a] * wys[b];
      c.w[i] = wc;
      c.q[i] = -1;
      if (wc != 0.0) {
        const long long cx = x0 + a, cy = y0 + b;
        bool inside;
        int col;
        if (periodic) {
          inside = (cy >= 0) && (cy < H);
          col = pos_mod(cx, W);
        } else {
          inside = (cx >= 0) && (cx < W) && (cy >= 0) && (cy < H);
          col = (int)cx;
        }
        if (inside) c.q[i] = (int)cy * W + col;
        else c.outside = true;
      }
    }
  }
}

// Lattice sample index for g = 0 at an integer centre: -1 when out of lattice.
__device__ __forceinline__ int lattice_index(int x, int y, int H, int W, int periodic) {
  if (y < 0 || y >= H) return -1;
  if (periodic) x = pos_mod32(x, W);
  else if (x < 0 || x >= W) return -1;
  return y * W + x;
}

// numpy pairwise accumulation of sample k (lane-local part)
template <int NL>
__device__ __forceinline__ void acc_sample(const BallParams& P, int k, double w, double wr,
                                           double* acc_rw, double* acc_tw, double* tl_rw,
                                           double* tl_tw) {
#pragma unroll
  for (int L = 0; L < NL; ++L) {
    const int lo = NL == 1 ? 0 : P.plan.leaf_lo[L];
    const int n = P.plan.leaf_n[L];
    const int kk = k - lo;
    if ((NL == 1 || (L < P.plan.n_leaves && kk >= 0)) && kk < n) {
      if (kk < n - (n % 8)) {
        acc_rw[L] += wr;
        acc_tw[L] += w;
      } else {
        tl_rw[L] = wr;
        tl_tw[L] = w;
      }
    }
  }
}

// Weight of ball sample k for a g != 0 guide (engine.py:131-164); also
// returns the rotated offset.
__device__ __forceinline__ double sample_weight(const BallParams& P, const BallTables& T, int k,
                                                double gx, double gy, double ux, double uy,
                                                double safe, double thr, double& px, double& py) {
  px = T.n[k];
  py = T.m[k];
  if (P.rotated) {
    px = T.n[k] * uy + T.m[k] * ux;
    py = (-T.n[k]) * ux + T.m[k] * uy;
  }
  const double dist = hypot_np(px, py);
  if (P.mu_inf) {
    const double d = ((-gy) * px + gx * py) / safe;
    return (d * d <= thr) ? 1.0 / dist : 0.0;
  }
  const double d = (-gy) * px + gx * py;
  return exp_np((P.coef * d) * d) / dist;
}

// Evaluate one item.  Must be called by all 32 lanes of the warp
// (groups with valid == false compute on dummy data and never write).
// NL  = pairwise leaves the kernel was specialised for (1 covers K <= 128);
// KPL = samples per lane (ceil(K / 8)) as a compile-time bound so every
//       fetch of a lane is issued before the first one is consumed, or 0
//       for a runtime loop (large radii).
// axis_dist: optional hypot(n_k, m_k) table (EXACTV path, axis ball).
// EXACTV: the colour numerator in numpy's einsum("fk,fkc->fc") order
//       (engine.py:196) instead of per-lane partial sums, so the values are
//       bit-exact in fp64 (the coherence path feeds them back into the
//       structure tensor).  For C >= 2 einsum adds the products w_k * v_kc
//       in k order; for C == 1 both operands are contiguous and its SSE2
//       loop keeps two lanes (even / odd k), folding each block of 8 from
//       the top (k+6, k+4, k+2, k) and the tail upwards, then adds the lanes.
// The result is valid in every lane of the group.
template <int NL, int KPL, bool EXACTV = false, class Src>
__device__ __forceinline__ void eval_item(const BallParams& P, const BallTables& T,
                                          const Src& src, int lane, bool valid, double fi,
                                          double fj, bool integral, double gx, double gy,
                                          SampleResult& out, const double* axis_dist = nullptr) {
  const int K = P.K;
  const bool gzero = (gx == 0.0) && (gy == 0.0);
  double ux = 0.0, uy = 1.0;
  if (P.rotated && !gzero) {
    const double nr = hypot_np(gx, gy);
    ux = gx / nr;
    uy = gy / nr;
  }
  double safe = 1.0, thr = 0.0;
  if (P.mu_inf) {
    const double nr2 = sqrt(gx * gx + gy * gy);
    safe = (nr2 == 0.0) ? 1.0 : nr2;
    double mloc = INFINITY;
    for (int k = lane; k < K; k += kGroup) {
      double px = T.n[k], py = T.m[k];
      if (P.rotated && !gzero) {
        px = T.n[k] * uy + T.m[k] * ux;
        py = (-T.n[k]) * ux + T.m[k] * uy;
      }
      const double d = ((-gy) * px + gx * py) / safe;
      mloc = min_prop(mloc, d * d);
    }
    mloc = min_prop(mloc, __shfl_xor_sync(0xffffffffu, mloc, 1, kGroup));
    mloc = min_prop(mloc, __shfl_xor_sync(0xffffffffu, mloc, 2, kGroup));
    mloc = min_prop(mloc, __shfl_xor_sync(0xffffffffu, mloc, 4, kGroup));
    thr = mloc + P.tol_inf;
  }

  double acc_rw[NL], acc_tw[NL], tl_rw[NL], tl_tw[NL];
#pragma unroll
  for (int L = 0; L < NL; ++L) acc_rw[L] = acc_tw[L] = tl_rw[L] = tl_tw[L] = 0.0;
  double num[4] = {0.0, 0.0, 0.0, 0.0};
  const int pi = (int)fi, pj = (int)fj;

  double ex_s[4] = {0.0, 0.0, 0.0, 0.0};  // EXACTV: C >= 2 sums / C == 1 lanes 0, 1
  if constexpr (EXACTV) {
    // numpy einsum order for the numerator: block of kGroup samples folded
    // in k order (lanes hold consecutive k; the fold is warp-uniform)
    auto fold = [&](const double (&p)[4], int rem) {
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        double q[kGroup];
#pragma unroll
        for (int l = 0; l < kGroup; ++l) q[l] = __shfl_sync(0xffffffffu, p[c], l, kGroup);
        if (c >= src.C) continue;
        if (src.C == 1) {
          if (rem >= 8) {
            ex_s[0] = q[6] + ex_s[0];
            ex_s[0] = q[4] + ex_s[0];
            ex_s[0] = q[2] + ex_s[0];
            ex_s[0] = q[0] + ex_s[0];
            ex_s[1] = q[7] + ex_s[1];
            ex_s[1] = q[5] + ex_s[1];
            ex_s[1] = q[3] + ex_s[1];
            ex_s[1] = q[1] + ex_s[1];
          } else {
#pragma unroll
            for (int l = 0; l < 8; l += 2) {
              if (l < rem) {
                ex_s[0] = q[l] + ex_s[0];
                ex_s[1] = (l + 1 < rem ? q[l + 1] : 0.0) + ex_s[1];
              }
            }
          }
        } else {
#pragma unroll
          for (int l = 0; l < kGroup; ++l)
            if (l < rem) ex_s[c] = ex_s[c] + q[l];
        }
      }
    };
    // weight of sample k at offset (px, py) (engine.py:131-147); an axis
    // ball's distances hypot(n, m) may come from the axis_dist table
    auto weight = [&](int k, double px, double py) {
      if (gzero) return T.w0[k];
      const double dist = (axis_dist && !P.rotated) ? axis_dist[k] : hypot_np(px, py);
      if (P.mu_inf) {
        const double d = ((-gy) * px + gx * py) / safe;
        return (d * d <= thr) ? 1.0 / dist : 0.0;
      }
      const double d = (-gy) * px + gx * py;
      return exp_np((P.coef * d) * d) / dist;
    };
    if (integral && (gzero || !P.rotated)) {
      // an integral centre with lattice offsets (g = 0, or the axis ball at
      // any g) samples one pixel with bilinear weight 1: grid.py's ghost
      // gather reduces to the lattice value (the other corners are not
      // live).  Two blocks per iteration: both fetches and both weight
      // chains in flight together.
#pragma unroll 1
      for (int kb = 0; kb < K; kb += 2 * kGroup) {
        int kk[2], q[2];
        decltype(src.fetch(0)) v[2];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          kk[h] = kb + h * kGroup + lane;
          const int kc = kk[h] < K ? kk[h] : 0;
          q[h] = (valid && kk[h] < K)
                     ? lattice_index(pi + T.ni[kc], pj + T.mi[kc], src.H, src.W, P.periodic)
                     : -1;
          v[h] = src.fetch(q[h] >= 0 ? q[h] : 0);
        }
        double w[2];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int kc = kk[h] < K ? kk[h] : 0;
          w[h] = weight(kc, T.n[kc], T.m[kc]);
        }
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int b0 = kb + h * kGroup;
          if (b0 >= K) break;  // uniform
          double p[4] = {0.0, 0.0, 0.0, 0.0};
          if (kk[h] < K) {
            double sv[4] = {0.0, 0.0, 0.0, 0.0};
            const bool ok = q[h] >= 0 && src.readable(v[h]);
            if (ok) src.accumulate(v[h], 1.0, sv);
            const double wr = ok ? w[h] : 0.0;
            if (ok) {
#pragma unroll
              for (int c = 0; c < 4; ++c) p[c] = wr * sv[c];
            }
            acc_sample<NL>(P, kk[h], w[h], wr, acc_rw, acc_tw, tl_rw, tl_tw);
          }
          fold(p, K - b0);
        }
      }
    } else {
      // ghost samples: one per lane per block of kGroup
#pragma unroll 1
      for (int kb = 0; kb < K; kb += kGroup) {
        const int k = kb + lane;
        double p[4] = {0.0, 0.0, 0.0, 0.0};
        if (k < K) {
          double px = T.n[k], py = T.m[k];
          if (!gzero && P.rotated) {
            px = T.n[k] * uy + T.m[k] * ux;
            py = (-T.n[k]) * ux + T.m[k] * uy;
          }
          Corners cn;
          ghost_corners(fi + px, fj + py, src.H, src.W, P.periodic, cn);
          decltype(src.fetch(0)) v[4];
#pragma unroll
          for (int c = 0; c < 4; ++c) v[c] = src.fetch(cn.q[c] >= 0 ? cn.q[c] : 0);
          const double w = weight(k, px, py);
          double sv[4] = {0.0, 0.0, 0.0, 0.0};
          bool ok = valid && !cn.outside;
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            if (cn.q[c] >= 0 && valid) {
              ok = ok && src.readable(v[c]);
              src.accumulate(v[c], cn.w[c], sv);
            }
          }
          const double wr = ok ? w : 0.0;
          if (ok) {
#pragma unroll
            for (int c = 0; c < 4; ++c) p[c] = wr * sv[c];
          }
          acc_sample<NL>(P, k, w, wr, acc_rw, acc_tw, tl_rw, tl_tw);
        }
        fold(p, K - kb);
      }
    }
  } else if (gzero && integral) {
    // lattice path (most Inpaint pixels): weights are the host's
    // 1/hypot(n, m); one fetch per sample, all issued up front
    if constexpr (KPL > 0) {
      int q[KPL];
      decltype(src.fetch(0)) v[KPL];
#pragma unroll
      for (int t = 0; t < KPL; ++t) {
        const int k = lane + kGroup * t;
        q[t] = (valid && k < K)
                   ? lattice_index(pi + (int)T.n[k], pj + (int)T.m[k], src.H, src.W, P.periodic)
                   : -1;
      }
#pragma unroll
      for (int t = 0; t < KPL; ++t)
        if (q[t] >= 0) v[t] = src.fetch(q[t]);
#pragma unroll
      for (int t = 0; t < KPL; ++t) {
        const int k = lane + kGroup * t;
        if (k < K) {
          const double w = T.w0[k];
          const bool ok = q[t] >= 0 && src.readable(v[t]);
          const double wr = ok ? w : 0.0;
          if (ok) {
            double sv[4] = {0.0, 0.0, 0.0, 0.0};
            src.accumulate(v[t], 1.0, sv);
#pragma unroll
            for (int c = 0; c < 4; ++c) num[c] += wr * sv[c];
          }
          acc_sample<NL>(P, k, w, wr, acc_rw, acc_tw, tl_rw, tl_tw);
        }
      }
    } else {
#pragma unroll 1
      for (int k = lane; k < K; k += kGroup) {
        const int q = valid ? lattice_index(pi + (int)T.n[k], pj + (int)T.m[k], src.H, src.W,
                                            P.periodic)
                            : -1;
        const double w = T.w0[k];
        bool ok = false;
        double sv[4] = {0.0, 0.0, 0.0, 0.0};
        if (q >= 0) {
          const auto v = src.fetch(q);
          ok = src.readable(v);
          if (ok) src.accumulate(v, 1.0, sv);
        }
        const double wr = ok ? w : 0.0;
        if (ok) {
#pragma unroll
          for (int c = 0; c < 4; ++c) num[c] += wr * sv[c];
        }
        acc_sample<NL>(P, k, w, wr, acc_rw, acc_tw, tl_rw, tl_tw);
      }
    }
  } else {
    // ghost-pixel path: rotated ball at g, or g = 0 at a non-lattice point
#pragma unroll 1
    for (int k = lane; k < K; k += kGroup) {
      double px, py, w;
      if (gzero) {
        px = T.n[k];
        py = T.m[k];
        w = T.w0[k];
      } else {
        w = sample_weight(P, T, k, gx, gy, ux, uy, safe, thr, px, py);
      }
      Corners cn;
      ghost_corners(fi + px, fj + py, src.H, src.W, P.periodic, cn);
      decltype(src.fetch(0)) v[4];
#pragma unroll
      for (int c = 0; c < 4; ++c)
        if (valid && cn.q[c] >= 0) v[c] = src.fetch(cn.q[c]);
      bool ok = valid && !cn.outside;
      double sv[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        if (cn.q[c] >= 0 && valid) {
          ok = ok && src.readable(v[c]);
          src.accumulate(v[c], cn.w[c], sv);
        }
      }
      const double wr = ok ? w : 0.0;
      if (ok) {
#pragma unroll
        for (int c = 0; c < 4; ++c) num[c] += wr * sv[c];
      }
      acc_sample<NL>(P, k, w, wr, acc_rw, acc_tw, tl_rw, tl_tw);
    }
  }

  // leaf sums: 8-accumulator tree, then the sequential tail (lane 0 exact)
  double leaf_rw[NL], leaf_tw[NL];
#pragma unroll
  for (int L = 0; L < NL; ++L) {
    double srw = group_sum_tree(acc_rw[L]);
    double stw = group_sum_tree(acc_tw[L]);
    const int ntail = (L < P.plan.n_leaves) ? P.plan.leaf_n[L] % 8 : 0;
    for (int t = 0; t < ntail; ++t) {
      srw = srw + __shfl_sync(0xffffffffu, tl_rw[L], t, kGroup);
      stw = stw + __shfl_sync(0xffffffffu, tl_tw[L], t, kGroup);
    }
    leaf_rw[L] = srw;
    leaf_tw[L] = stw;
  }
  double rw, tw;
  if (NL == 1) {
    rw = leaf_rw[0];
    tw = leaf_tw[0];
  } else {
    double st_rw[NL], st_tw[NL];
    int sp = 0;
    for (int i = 0; i < P.plan.n_prog; ++i) {
      const int op = P.plan.prog[i];
      if (op >= 0) {
        double a = 0.0, b = 0.0;
#pragma unroll
        for (int L = 0; L < NL; ++L)
          if (L == op) {
            a = leaf_rw[L];
            b = leaf_tw[L];
          }
#pragma unroll
        for (int s = 0; s < NL; ++s)
          if (s == sp) {
            st_rw[s] = a;
            st_tw[s] = b;
          }
        ++sp;
      } else {
        --sp;
        double a = 0.0, b = 0.0, c = 0.0, d = 0.0;
#pragma unroll
        for (int s = 0; s < NL; ++s) {
          if (s == sp) { a = st_rw[s]; b = st_tw[s]; }
          if (s == sp - 1) { c = st_rw[s]; d = st_tw[s]; }
        }
#pragma unroll
        for (int s = 0; s < NL; ++s)
          if (s == sp - 1) {
            st_rw[s] = c + a;
            st_tw[s] = d + b;
          }
      }
    }
    rw = st_rw[0];
    tw = st_tw[0];
  }
  rw = __shfl_sync(0xffffffffu, rw, 0, kGroup);
  tw = __shfl_sync(0xffffffffu, tw, 0, kGroup);
  if constexpr (EXACTV) {
    if (src.C == 1) ex_s[0] = 0.0 + (ex_s[0] + ex_s[1]);
#pragma unroll
    for (int c = 0; c < 4; ++c) out.v[c] = (c < src.C && rw != 0.0) ? ex_s[c] / rw : 0.0;
  } else {
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      double s = num[c];
      s += __shfl_xor_sync(0xffffffffu, s, 1, kGroup);
      s += __shfl_xor_sync(0xffffffffu, s, 2, kGroup);
      s += __shfl_xor_sync(0xffffffffu, s, 4, kGroup);
      out.v[c] = (rw != 0.0) ? s / rw : 0.0;
    }
  }
  out.rw = rw;
  out.tw = tw;
}

}  // namespace gf
