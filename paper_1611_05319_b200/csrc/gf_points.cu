// Point-evaluation and lattice kernels behind the reference's small public
// operators: engine.confidence / engine.fill_color (engine.py:202-221),
// grid.bilinear_gather / sample_bilinear (grid.py:158-221) and the boundary
// set operators (grid.py:84-106).
#include <cuda_runtime.h>
#include <stdint.h>

#include "gf_internal.cuh"

namespace gf {

constexpr int kPtThreads = 256;

template <int NL>
__global__ void __launch_bounds__(kPtThreads)
    k_sample_points(RawSource src, int n, const double* __restrict__ pts,
                    const double* __restrict__ g, const __grid_constant__ BallParams P,
                    const __grid_constant__ BallTables tab, double* rw, double* tw, double* vals) {
  __shared__ BallTables T;
  for (int i = threadIdx.x; i < P.K; i += blockDim.x) {
    T.n[i] = tab.n[i];
    T.m[i] = tab.m[i];
    T.w0[i] = tab.w0[i];
    T.ni[i] = tab.ni[i];
    T.mi[i] = tab.mi[i];
  }
  __syncthreads();
  const int lane = threadIdx.x & (kGroup - 1);
  const int groups = blockDim.x / kGroup;
  for (int base = blockIdx.x * groups; base < n; base += gridDim.x * groups) {
    const int t = base + threadIdx.x / kGroup;
    const bool valid = t < n;
    const double x = valid ? pts[2 * t] : 0.0, y = valid ? pts[2 * t + 1] : 0.0;
    const double gx = valid ? g[2 * t] : 0.0, gy = valid ? g[2 * t + 1] : 0.0;
    const bool integral = (x == floor(x)) && (y == floor(y)) && fabs(x) < 1e9 && fabs(y) < 1e9;
    SampleResult r;
    eval_item<NL, 0, true>(P, T, src, lane, valid, x, y, integral, gx, gy, r);
    if (valid && lane == 0) {
      rw[t] = r.rw;
      tw[t] = r.tw;
      for (int c = 0; c < src.C; ++c) vals[(size_t)t * src.C + c] = r.v[c];
    }
  }
}

int sample_points_launch(int H, int W, int C, const double* image, const uint8_t* labels, int n,
                         const double* points, const double* g, const BallParams& P,
                         const BallTables& tab, double* rw, double* tw, double* vals,
                         cudaStream_t stream) {
  if (n <= 0) return GF_OK;
  RawSource src{image, labels, H, W, C};
  const int groups = kPtThreads / kGroup;
  const int grid = std::min(4096, (n + groups - 1) / groups);
  if (P.plan.n_leaves > 1)
    k_sample_points<kMaxLeaves><<<grid, kPtThreads, 0, stream>>>(src, n, points, g, P, tab, rw, tw, vals);
  else
    k_sample_points<1><<<grid, kPtThreads, 0, stream>>>(src, n, points, g, P, tab, rw, tw, vals);
  count_launches(1);
  cudaError_t e = cudaPeekAtLastError();
  if (e != cudaSuccess) return set_error(GF_E_CUDA, cudaGetErrorString(e));
  return GF_OK;
}

// ---------------------------------------------------------------------------
// Balls beyond the shell kernels' tables (r > GF_MAX_RADIUS; the reference
// accepts any r >= 1, engine.py:51-52).  The tables live in global memory and
// the numpy pairwise plan has any number of leaves.  One 8-lane group per
// point walks the K samples in blocks of 8 (a leaf starts on a multiple of 8,
// so a block never straddles two): lane 0 keeps numpy's 8 interleaved
// accumulators of the current leaf, reduces a finished leaf with the
// ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7)) tree and its sequential tail, and runs
// the plan's postfix program on a small stack.  The colour numerator is
// folded in numpy's einsum order as in eval_item's EXACTV path.
// ---------------------------------------------------------------------------
constexpr int kBigStack = 48;

__global__ void __launch_bounds__(kPtThreads)
    k_sample_points_big(RawSource src, int n, const double* __restrict__ pts,
                        const double* __restrict__ g, const BigBall B, double* rw, double* tw,
                        double* vals) {
  const int lane = threadIdx.x & (kGroup - 1);
  const int groups = blockDim.x / kGroup;
  const int K = B.K;
  for (int base = blockIdx.x * groups; base < n; base += gridDim.x * groups) {
    const int t = base + threadIdx.x / kGroup;
    const bool valid = t < n;
    const double fi = valid ? pts[2 * t] : 0.0, fj = valid ? pts[2 * t + 1] : 0.0;
    const double gx = valid ? g[2 * t] : 0.0, gy = valid ? g[2 * t + 1] : 0.0;
    const bool integral = (fi == floor(fi)) && (fj == floor(fj)) && fabs(fi) < 1e9 && fabs(fj) < 1e9;
    const int pi = (int)fi, pj = (int)fj;
    const bool gzero = gx == 0.0 && gy == 0.0;
    double ux = 0.0, uy = 1.0;
    if (B.rotated && !gzero) {
      const double nr = hypot_np(gx, gy);
      ux = gx / nr;
      uy = gy / nr;
    }
    auto offset = [&](int k, double& px, double& py) {
      px = B.n[k];
      py = B.m[k];
      if (!gzero && B.rotated) {
        px = B.n[k] * uy + B.m[k] * ux;
        py = (-B.n[k]) * ux + B.m[k] * uy;
      }
    };
    double safe = 1.0, thr = 0.0;
    if (B.mu_inf) {  // argmin-set rule (engine.py:138-144): the smallest d^2 first
      const double nr2 = sqrt(gx * gx + gy * gy);
      safe = (nr2 == 0.0) ? 1.0 : nr2;
      double mloc = INFINITY;
      for (int k = lane; k < K; k += kGroup) {
        double px, py;
        offset(k, px, py);
        const double d = ((-gy) * px + gx * py) / safe;
        mloc = min_prop(mloc, d * d);
      }
      mloc = min_prop(mloc, __shfl_xor_sync(0xffffffffu, mloc, 1, kGroup));
      mloc = min_prop(mloc, __shfl_xor_sync(0xffffffffu, mloc, 2, kGroup));
      mloc = min_prop(mloc, __shfl_xor_sync(0xffffffffu, mloc, 4, kGroup));
      thr = mloc + B.tol_inf;
    }
    const bool lat = integral && (gzero || !B.rotated);
    // lane 0 state: the leaf accumulators, the plan stack, the fold
    double r_rw[kGroup], r_tw[kGroup], st_rw[kBigStack], st_tw[kBigStack];
    int sp = 0, pc = 0, leaf = 0;
    double ex[4] = {0.0, 0.0, 0.0, 0.0};
    auto push_leaf = [&](double a_rw, double a_tw) {
      // prog[pc] is this leaf's push; then every -1 that follows combines
      st_rw[sp] = a_rw;
      st_tw[sp] = a_tw;
      ++sp;
      ++pc;
      while (pc < B.n_prog && B.prog[pc] < 0) {
        st_rw[sp - 2] = st_rw[sp - 2] + st_rw[sp - 1];
        st_tw[sp - 2] = st_tw[sp - 2] + st_tw[sp - 1];
        --sp;
        ++pc;
      }
    };
    for (int kb = 0; kb < K; kb += kGroup) {
      const int k = kb + lane;
      double w = 0.0, wr = 0.0, p[4] = {0.0, 0.0, 0.0, 0.0};
      if (k < K) {
        double px, py;
        offset(k, px, py);
        double sv[4] = {0.0, 0.0, 0.0, 0.0};
        bool ok = false;
        if (lat) {
          const int q = valid ? lattice_index(pi + B.ni[k], pj + B.mi[k], src.H, src.W, B.periodic)
                              : -1;
          if (q >= 0) {
            const auto v = src.fetch(q);
            ok = src.readable(v);
            if (ok) src.accumulate(v, 1.0, sv);
          }
        } else {
          Corners cn;
          ghost_corners(fi + px, fj + py, src.H, src.W, B.periodic, cn);
          ok = valid && !cn.outside;
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            if (cn.q[c] >= 0 && valid) {
              const auto v = src.fetch(cn.q[c]);
              ok = ok && src.readable(v);
              src.accumulate(v, cn.w[c], sv);
            }
          }
        }
        w = B.w0[k];
        if (!gzero) {
          const double dist = hypot_np(px, py);
          if (B.mu_inf) {
            const double d = ((-gy) * px + gx * py) / safe;
            w = (d * d <= thr) ? 1.0 / dist : 0.0;
          } else {
            const double d = (-gy) * px + gx * py;
            w = exp_np((B.coef * d) * d) / dist;
          }
        }
        wr = ok ? w : 0.0;
        if (ok) {
#pragma unroll
          for (int c = 0; c < 4; ++c) p[c] = wr * sv[c];
        }
      }
      // masses: this block's 8 values to lane 0, in k order
      double q_rw[kGroup], q_tw[kGroup];
#pragma unroll
      for (int l = 0; l < kGroup; ++l) {
        q_rw[l] = __shfl_sync(0xffffffffu, wr, l, kGroup);
        q_tw[l] = __shfl_sync(0xffffffffu, w, l, kGroup);
      }
      if (lane == 0) {
        const int lo = B.leaf_lo[leaf], nl = B.leaf_n[leaf];
        const int bend = lo + nl - nl % kGroup;
        if (nl < kGroup) {  // a short leaf: sequential from 0.0
          double a = 0.0, b = 0.0;
          for (int l = 0; l < nl; ++l) {
            a += q_rw[l];
            b += q_tw[l];
          }
          push_leaf(a, b);
          ++leaf;
        } else if (kb < bend) {
#pragma unroll
          for (int l = 0; l < kGroup; ++l) {
            r_rw[l] = kb == lo ? q_rw[l] : r_rw[l] + q_rw[l];
            r_tw[l] = kb == lo ? q_tw[l] : r_tw[l] + q_tw[l];
          }
          if (kb + kGroup == lo + nl) {
            push_leaf(((r_rw[0] + r_rw[1]) + (r_rw[2] + r_rw[3])) + ((r_rw[4] + r_rw[5]) + (r_rw[6] + r_rw[7])),
                      ((r_tw[0] + r_tw[1]) + (r_tw[2] + r_tw[3])) + ((r_tw[4] + r_tw[5]) + (r_tw[6] + r_tw[7])));
            ++leaf;
          }
        } else {  // the leaf's tail block
          double a = ((r_rw[0] + r_rw[1]) + (r_rw[2] + r_rw[3])) + ((r_rw[4] + r_rw[5]) + (r_rw[6] + r_rw[7]));
          double b = ((r_tw[0] + r_tw[1]) + (r_tw[2] + r_tw[3])) + ((r_tw[4] + r_tw[5]) + (r_tw[6] + r_tw[7]));
          for (int l = 0; l < nl % kGroup; ++l) {
            a += q_rw[l];
            b += q_tw[l];
          }
          push_leaf(a, b);
          ++leaf;
        }
      }
      // colour numerator, numpy einsum order (eval_item EXACTV)
      const int rem = K - kb;
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        double q[kGroup];
#pragma unroll
        for (int l = 0; l < kGroup; ++l) q[l] = __shfl_sync(0xffffffffu, p[c], l, kGroup);
        if (c >= src.C) continue;
        if (src.C == 1) {
          if (rem >= 8) {
            ex[0] = q[6] + ex[0];
            ex[0] = q[4] + ex[0];
            ex[0] = q[2] + ex[0];
            ex[0] = q[0] + ex[0];
            ex[1] = q[7] + ex[1];
            ex[1] = q[5] + ex[1];
            ex[1] = q[3] + ex[1];
            ex[1] = q[1] + ex[1];
          } else {
            for (int l = 0; l < 8; l += 2)
              if (l < rem) {
                ex[0] = q[l] + ex[0];
                ex[1] = (l + 1 < rem ? q[l + 1] : 0.0) + ex[1];
              }
          }
        } else {
#pragma unroll
          for (int l = 0; l < kGroup; ++l)
            if (l < rem) ex[c] = ex[c] + q[l];
        }
      }
    }
    if (valid && lane == 0) {
      const double R = st_rw[0], T = st_tw[0];
      rw[t] = R;
      tw[t] = T;
      if (src.C == 1) ex[0] = 0.0 + (ex[0] + ex[1]);
      for (int c = 0; c < src.C; ++c) vals[(size_t)t * src.C + c] = R != 0.0 ? ex[c] / R : 0.0;
    }
  }
}

int sample_points_big_launch(int H, int W, int C, const double* image, const uint8_t* labels,
                             int n, const double* points, const double* g, const BigBall& B,
                             double* rw, double* tw, double* vals, cudaStream_t stream) {
  if (n <= 0) return GF_OK;
  RawSource src{image, labels, H, W, C};
  const int groups = kPtThreads / kGroup;
  const int grid = std::min(4096, (n + groups - 1) / groups);
  k_sample_points_big<<<grid, kPtThreads, 0, stream>>>(src, n, points, g, B, rw, tw, vals);
  count_launches(1);
  cudaError_t e = cudaPeekAtLastError();
  if (e != cudaSuccess) return set_error(GF_E_CUDA, cudaGetErrorString(e));
  return GF_OK;
}

__global__ void k_bilinear(RawSource src, int n, const double* X, const double* Y, int periodic,
                           double* vals, uint8_t* ok) {
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < n; t += gridDim.x * blockDim.x) {
    double sv[4] = {0.0, 0.0, 0.0, 0.0};
    const bool good = ghost_sample(src, X[t], Y[t], periodic, sv);
    ok[t] = good ? 1 : 0;
    for (int c = 0; c < src.C; ++c) vals[(size_t)t * src.C + c] = good ? sv[c] : 0.0;
  }
}

int bilinear_launch(int H, int W, int C, const double* image, const uint8_t* labels, int n,
                    const double* X, const double* Y, int periodic, double* vals, uint8_t* ok,
                    cudaStream_t stream) {
  if (n <= 0) return GF_OK;
  RawSource src{image, labels, H, W, C};
  k_bilinear<<<std::min(4096, (n + 255) / 256), 256, 0, stream>>>(src, n, X, Y, periodic, vals, ok);
  count_launches(1);
  cudaError_t e = cudaPeekAtLastError();
  if (e != cudaSuccess) return set_error(GF_E_CUDA, cudaGetErrorString(e));
  return GF_OK;
}

// One thread per pixel: active / inner / outer boundary flags.
__global__ void k_boundary(int H, int W, const uint8_t* __restrict__ lab, int periodic,
                           uint8_t* active, uint8_t* inner, uint8_t* outer) {
  const int total = H * W;
  for (int p = blockIdx.x * blockDim.x + threadIdx.x; p < total; p += gridDim.x * blockDim.x) {
    const int i = p % W, j = p / W;
    const bool inp = lab[p] == 255;
    bool nb_read = false, nb_noninp = false, nb_inp = false;
    for (int dj = -1; dj <= 1; ++dj) {
      const int jj = j + dj;
      if (jj < 0 || jj >= H) continue;
      for (int di = -1; di <= 1; ++di) {
        if (di == 0 && dj == 0) continue;
        int ii = i + di;
        if (periodic) ii = (ii + W) % W;
        else if (ii < 0 || ii >= W) continue;
        const uint8_t l = lab[jj * W + ii];
        nb_read |= l == 0;
        nb_noninp |= l != 255;
        nb_inp |= l == 255;
      }
    }
    if (active) active[p] = inp && nb_read;
    if (inner) inner[p] = inp && nb_noninp;
    if (outer) outer[p] = !inp && nb_inp;
  }
}

int boundary_launch(int H, int W, const uint8_t* labels, int periodic, uint8_t* active,
                    uint8_t* inner, uint8_t* outer, cudaStream_t stream) {
  const int total = H * W;
  if (total <= 0) return GF_OK;
  k_boundary<<<std::min(8192, (total + 255) / 256), 256, 0, stream>>>(H, W, labels, periodic,
                                                                       active, inner, outer);
  count_launches(1);
  cudaError_t e = cudaPeekAtLastError();
  if (e != cudaSuccess) return set_error(GF_E_CUDA, cudaGetErrorString(e));
  return GF_OK;
}

}  // namespace gf
