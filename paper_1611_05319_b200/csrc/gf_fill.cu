// Guidefill fill engine for sm_100a: prep -> persistent shell loop -> finalize.
//
// Replaces engine._fill_loop (engine.py:286-376) together with the tracker
// hook (tracker.py:42-79, 161-170).  Layout in HBM, per frame f of a batch:
//
//   work[f][H*W]      float4 {c0, c1, c2, stamp}: fp32 colour + int32 stamp
//                     (readable at shell k <=> stamp <= k; filled at shell k
//                     -> stamp = k+1; Inpaint/Bystander -> large markers).
//                     One 128-bit load gives a ball sample's colour and its
//                     snapshot readability, so a shell needs no barrier
//                     between evaluating and writing fills.
//   c3[f][H*W]        4th channel plane (C == 4 only).
//   list[2][f][H*W]   ping-pong compacted frontier lists (uint32 pixel index).
//   conf[f][H*W]      per-item confidence of the current shell (deadlock guard).
//   per-frame counters (frontier sizes, fills, remaining, ...).
//
// The shell loop is ONE cooperative persistent kernel: every shell is
//   A  fill:     8 lanes per frontier pixel evaluate the rotated ball
//                (gf_sampler.cuh) and write fills in place;
//   G  guard:    only if some frame filled nothing: argmax-C (first index on
//                ties, NaN maximal) and the single guarded fill;
//   B  update:   tracked -- survivors + Inpaint 8-neighbours of the filled
//                pixels, deduplicated by an atomic INACTIVE->ACTIVE stamp
//                transition, compacted through shared memory with one global
//                atomic per tile; untracked -- full-lattice rescan;
// separated by grid-wide barriers, so the host never sees a shell.
#include <cooperative_groups.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "gf_internal.cuh"

namespace cg = cooperative_groups;

namespace gf {

constexpr int kThreads = 256;
constexpr int kGroupsPerBlock = kThreads / kGroup;
constexpr int kAppendCap = kThreads * 9;

__device__ __forceinline__ unsigned long long enc_ordered(double d) {
  const unsigned long long b = (unsigned long long)__double_as_longlong(d);
  return (b >> 63) ? ~b : (b | 0x8000000000000000ULL);
}
__host__ __device__ inline double dec_ordered(unsigned long long e) {
  const unsigned long long b = (e >> 63) ? (e & 0x7fffffffffffffffULL) : ~e;
  double d;
  memcpy(&d, &b, 8);
  return d;
}

__device__ __forceinline__ int stamp_of(const float4* work, int q) {
  return __float_as_int(work[q].w);
}
__device__ __forceinline__ int* stamp_ptr(float4* work, int q) {
  return reinterpret_cast<int*>(&work[q].w);
}

// ---------------------------------------------------------------- prep
//
// One pass over every pixel, frame-major grid (blockIdx.y = frame): builds
// the working frame (fp32 colour + stamp), the initial frontier (Inpaint
// with a Readable 8-neighbour, grid.py:104-106), |D|, the value hull
// (min/max of the readable values over all channels, engine.py:291-296)
// and, when splines are given, the guide field g of every Inpaint pixel
// (guide.py:303-327) -- rastered in place, so the field never exists as a
// dense array.  Segments are culled per 256-pixel tile against the tile's
// bounding box inflated by 3 eta: a pixel's g is non-zero only if its
// nearest segment lies within 3 eta, and then that segment (and every tied
// one) survives the cull, so non-zero g values are bit-identical to the
// dense rasteriser; pixels with no candidate get g = +0 (the reference's
// +-0 there is indistinguishable to the fill: every use tests g == 0 or
// |g|).

constexpr int kMaxCand = 512;

__device__ __forceinline__ double seg_dist(double px, double py, const double4 s) {
  const double ax = s.x, ay = s.y, bx = s.z, by = s.w;
  const double abx = bx - ax, aby = by - ay;
  const double L2 = abx * abx + aby * aby;
  if (L2 == 0.0) return hypot_np(px - ax, py - ay);
  double t = ((px - ax) * abx + (py - ay) * aby) / L2;
  t = (t < 0.0) ? 0.0 : t;
  t = (t > 1.0) ? 1.0 : t;
  return hypot_np(px - (ax + t * abx), py - (ay + t * aby));
}

template <typename T>
__global__ void __launch_bounds__(kThreads) k_prep(const __grid_constant__ FillArgs A) {
  const int f = blockIdx.y;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  __shared__ int s_cand[kMaxCand];
  __shared__ int s_ncand;
  __shared__ unsigned long long s_red[2][kThreads / 32];
  __shared__ int s_cnt[kThreads / 32];
  const uint8_t* lab = A.labels + (size_t)f * A.HW;
  const T* img = reinterpret_cast<const T*>(A.image) + (size_t)f * A.HW * A.C;
  float4* work = A.work + (size_t)f * A.HW;
  unsigned long long emin_inv = 0ULL, emax = 0ULL;  // max(~enc) <=> min(enc)
  int n_inp = 0;
  bool anyg = false;
  const bool raster = A.n_seg > 0;
  for (int base = blockIdx.x * kThreads; base < A.HW; base += gridDim.x * kThreads) {
    const int p = base + threadIdx.x;
    const bool in = p < A.HW;
    if (raster) {
      // tile bounding box -> candidate segments (order-free: the fused
      // raster takes the lexicographic min of (distance, spline index))
      const int last = min(A.HW - 1, base + kThreads - 1);
      const int j0 = base / A.W, j1 = last / A.W;
      const double x0 = (j0 == j1) ? (double)(base % A.W) : 0.0;
      const double x1 = (j0 == j1) ? (double)(last % A.W) : (double)(A.W - 1);
      if (threadIdx.x == 0) s_ncand = 0;
      __syncthreads();
      for (int i = threadIdx.x; i < A.n_seg; i += kThreads) {
        const double4 sg = A.seg[i];
        const double lo_x = fmin(sg.x, sg.z) - A.cut, hi_x = fmax(sg.x, sg.z) + A.cut;
        const double lo_y = fmin(sg.y, sg.w) - A.cut, hi_y = fmax(sg.y, sg.w) + A.cut;
        if (hi_x >= x0 && lo_x <= x1 && hi_y >= (double)j0 && lo_y <= (double)j1) {
          const int slot = atomicAdd(&s_ncand, 1);
          if (slot < kMaxCand) s_cand[slot] = i;
        }
      }
      __syncthreads();
    }
    bool active = false;
    if (in) {
      const uint8_t l = lab[p];
      const T* px_in = img + (size_t)p * A.C;
      float4 px;
      px.x = (float)px_in[0];
      px.y = A.C > 1 ? (float)px_in[1] : 0.f;
      px.z = A.C > 2 ? (float)px_in[2] : 0.f;
      if (A.C > 3) A.c3[(size_t)f * A.HW + p] = (float)px_in[3];
      int st;
      if (l == 0) {
        st = kStampReadable;
        for (int c = 0; c < A.C; ++c) {
          const unsigned long long e = enc_ordered((double)px_in[c]);
          emin_inv = (~e > emin_inv) ? ~e : emin_inv;
          emax = (e > emax) ? e : emax;
        }
      } else if (l == 255) {
        ++n_inp;
        const int i = p % A.W, j = p / A.W;
        for (int dj = -1; dj <= 1 && !active; ++dj) {
          const int jj = j + dj;
          if (jj < 0 || jj >= A.H) continue;
          for (int di = -1; di <= 1; ++di) {
            if (di == 0 && dj == 0) continue;
            int ii = i + di;
            if (A.periodic) ii = (ii + A.W) % A.W;
            else if (ii < 0 || ii >= A.W) continue;
            if (lab[jj * A.W + ii] == 0) {
              active = true;
              break;
            }
          }
        }
        st = active ? kStampActive : kStampInactive;
        double gx = 0.0, gy = 0.0;
        if (raster) {
          const bool exhaustive = s_ncand > kMaxCand;
          const int n_eval = exhaustive ? A.n_seg : s_ncand;
          double dmin = INFINITY;
          int near = 0x7fffffff;
          const double fx = (double)i, fy = (double)j;
          for (int c = 0; c < n_eval; ++c) {
            const int sidx = exhaustive ? c : s_cand[c];
            const double d = seg_dist(fx, fy, A.seg[sidx]);
            const int sp = A.seg_spline[sidx];
            if (d < dmin || (d == dmin && sp < near)) {
              dmin = d;
              near = sp;
            }
          }
          if (dmin <= A.cut) {
            const double fall = exp_np((-(dmin * dmin)) / A.c2eta);
            const double2 dir = A.dirs[near];
            gx = dir.x * fall;
            gy = dir.y * fall;
          }
          reinterpret_cast<double2*>(A.gfield)[(size_t)f * A.HW + p] = make_double2(gx, gy);
        } else if (A.g_mode == 2) {
          const double2 g = reinterpret_cast<const double2*>(A.gsrc)[(size_t)f * A.HW + p];
          gx = g.x;
          gy = g.y;
        }
        if (active && (gx != 0.0 || gy != 0.0)) anyg = true;
      } else {
        st = kStampBystander;
      }
      px.w = __int_as_float(st);
      work[p] = px;
      if (A.enter) A.enter[(size_t)f * A.HW + p] = active ? 0 : -1;
    }
    // warp-aggregated append of the initial frontier
    const unsigned mact = __ballot_sync(0xffffffffu, active);
    if (mact) {
      const int leader = __ffs(mact) - 1;
      int b = 0;
      if (lane == leader) b = atomicAdd(&A.cnt[f], __popc(mact));
      b = __shfl_sync(0xffffffffu, b, leader);
      if (active) A.list0[(size_t)f * A.cap + b + __popc(mact & ((1u << lane) - 1))] = (uint32_t)p;
    }
    if (raster) __syncthreads();  // s_cand is rebuilt for the next tile
  }
  // block reductions: hull, |D|, data-term flag -> one atomic each per block
  for (int o = 16; o > 0; o >>= 1) {
    const unsigned long long a = __shfl_xor_sync(0xffffffffu, emin_inv, o);
    const unsigned long long b = __shfl_xor_sync(0xffffffffu, emax, o);
    emin_inv = a > emin_inv ? a : emin_inv;
    emax = b > emax ? b : emax;
    n_inp += __shfl_xor_sync(0xffffffffu, n_inp, o);
  }
  const bool blk_anyg = __syncthreads_or(anyg);
  if (lane == 0) {
    s_red[0][warp] = emin_inv;
    s_red[1][warp] = emax;
    s_cnt[warp] = n_inp;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    int tot = 0;
    for (int w = 0; w < kThreads / 32; ++w) {
      emin_inv = s_red[0][w] > emin_inv ? s_red[0][w] : emin_inv;
      emax = s_red[1][w] > emax ? s_red[1][w] : emax;
      tot += s_cnt[w];
    }
    if (emax != 0ULL) {
      atomicMax(&A.hull[2 * f], emin_inv);
      atomicMax(&A.hull[2 * f + 1], emax);
    }
    if (tot) {
      atomicAdd(&A.remaining[f], tot);
      atomicAdd(&A.inpaint[f], tot);
    }
    if (blk_anyg) A.anyg[f] = 1;
  }
}

// ------------------------------------------------------- shell loop

struct Smem {
  BallTables tab;
  int pref[kMaxFramesPerLaunch + 1];
  unsigned char act[kMaxFramesPerLaunch];
  unsigned char dl[kMaxFramesPerLaunch];
  uint32_t app[kAppendCap];
  int napp;
  int base;
  int red[kThreads / 32];
  unsigned long long redk[kThreads / 32];
  int any_dl;
  int total;
};

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// per-shell phase timestamps (profiling only, A.trace may be null)
__device__ __forceinline__ void trace_set(const FillArgs& A, int k, int slot, unsigned long long v) {
  if (A.trace && k < A.trace_cap && blockIdx.x == 0 && threadIdx.x == 0) A.trace[k * 6 + slot] = v;
}
__device__ __forceinline__ void trace_max(const FillArgs& A, int k, int slot) {
  if (A.trace && k < A.trace_cap && threadIdx.x == 0) atomicMax(&A.trace[k * 6 + slot], gtimer());
}

__device__ __forceinline__ int find_frame(const int* pref, int nF, int t) {
  int lo = 0, hi = nF - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (pref[mid] <= t) lo = mid; else hi = mid - 1;
  }
  return lo;
}

__device__ __forceinline__ int block_sum(int v, Smem& S) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  __syncthreads();
  if ((threadIdx.x & 31) == 0) S.red[threadIdx.x >> 5] = v;
  __syncthreads();
  int t = 0;
  for (int w = 0; w < kThreads / 32; ++w) t += S.red[w];
  return t;
}

__device__ __forceinline__ unsigned long long block_max_u64(unsigned long long v, Smem& S) {
  for (int o = 16; o > 0; o >>= 1) {
    const unsigned long long a = __shfl_xor_sync(0xffffffffu, v, o);
    v = a > v ? a : v;
  }
  __syncthreads();
  if ((threadIdx.x & 31) == 0) S.redk[threadIdx.x >> 5] = v;
  __syncthreads();
  unsigned long long t = 0;
  for (int w = 0; w < kThreads / 32; ++w) t = S.redk[w] > t ? S.redk[w] : t;
  return t;
}

__device__ __forceinline__ unsigned long long conf_key(double c) {
  // numpy argmax: NaN is maximal; confidences are >= +0 otherwise
  return (c != c) ? ~0ULL : (unsigned long long)__double_as_longlong(c);
}

__device__ __forceinline__ void frame_guide(const FillArgs& A, int f, int p, double& gx,
                                            double& gy) {
  if (A.g_mode == 2) {
    const double2 g = reinterpret_cast<const double2*>(A.gsrc)[(size_t)f * A.HW + p];
    gx = g.x;
    gy = g.y;
  } else if (A.g_mode == 1) {
    gx = A.gfx;
    gy = A.gfy;
  } else {
    gx = 0.0;
    gy = 0.0;
  }
}

// Does the frontier of list `which` hold a pixel with g != 0?  (the
// data-term latch test of engine.py:327-329)
__device__ __forceinline__ bool frontier_has_g(const FillArgs& A, int which, int f) {
  if (A.g_mode == 2) return A.anyg[which * A.nF + f] != 0;
  if (A.g_mode == 1) return A.gfx != 0.0 || A.gfy != 0.0;
  return false;
}

// Append buffered pixels of frame f to the next list (one global atomic).
__device__ __forceinline__ void flush_appends(const FillArgs& A, Smem& S, int f, uint32_t* nxt_list,
                                              int nxt) {
  __syncthreads();
  const int n = S.napp;
  if (threadIdx.x == 0 && n > 0) S.base = atomicAdd(&A.cnt[nxt * A.nF + f], n);
  __syncthreads();
  if (n > 0) {
    const int base = S.base;
    bool anyg = false;
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
      const uint32_t q = S.app[i];
      nxt_list[(size_t)f * A.cap + base + i] = q;
      if (A.order == 2 && A.g_mode == 2) {
        const double2 g = reinterpret_cast<const double2*>(A.gsrc)[(size_t)f * A.HW + q];
        anyg |= (g.x != 0.0 || g.y != 0.0);
      }
    }
    if (__syncthreads_or(anyg) && threadIdx.x == 0) A.anyg[nxt * A.nF + f] = 1;
  }
  if (threadIdx.x == 0) S.napp = 0;
  __syncthreads();
}

__device__ __forceinline__ void push_append(Smem& S, bool want, uint32_t q) {
  const unsigned m = __ballot_sync(0xffffffffu, want);
  if (!m) return;
  const int lane = threadIdx.x & 31;
  int base = 0;
  if (lane == __ffs(m) - 1) base = atomicAdd(&S.napp, __popc(m));
  base = __shfl_sync(0xffffffffu, base, __ffs(m) - 1);
  if (want) S.app[base + __popc(m & ((1u << lane) - 1))] = q;
}

// Bookkeeping of shell k-1 (block 0 only): report row, remaining, latch.
__device__ void bookkeep(const FillArgs& A, int k) {
  const int prev = (k - 1) & 1;
  for (int f = threadIdx.x; f < A.nF; f += blockDim.x) {
    const int F = A.cnt[prev * A.nF + f];
    if (F > 0 && A.done[f] == 0) {
      const int filled = A.fills[prev * A.nF + f];
      const int it = A.iters[f];
      if (it < A.rows_cap) {
        A.rows[((size_t)f * A.rows_cap + it) * 2 + 0] = F;
        A.rows[((size_t)f * A.rows_cap + it) * 2 + 1] = filled;
      } else {
        A.overflow[f] = 1;
      }
      A.iters[f] = it + 1;
      A.filled[f] += filled;
      A.remaining[f] -= filled;
      if (A.remaining[f] == 0) A.done[f] = 1;
      if (!A.dt_dead[f] && !frontier_has_g(A, prev, f)) A.dt_dead[f] = 1;
    }
  }
}

template <int NL, bool kTracked>
__global__ void __launch_bounds__(kThreads) k_shells(const __grid_constant__ FillArgs A,
                                                     const __grid_constant__ BallParams P,
                                                     const __grid_constant__ BallTables tables) {
  cg::grid_group grid = cg::this_grid();
  extern __shared__ __align__(16) unsigned char smem_raw[];
  Smem& S = *reinterpret_cast<Smem*>(smem_raw);
  for (int i = threadIdx.x; i < P.K; i += blockDim.x) {
    S.tab.n[i] = tables.n[i];
    S.tab.m[i] = tables.m[i];
    S.tab.w0[i] = tables.w0[i];
  }
  if (threadIdx.x == 0) S.napp = 0;
  __syncthreads();

  const int lane = threadIdx.x & 31;
  const int glane = lane & (kGroup - 1);
  const int group = threadIdx.x / kGroup;

  for (int k = 0;; ++k) {
    const int cur = k & 1, nxt = cur ^ 1;
    uint32_t* cur_list = cur ? A.list1 : A.list0;
    uint32_t* nxt_list = cur ? A.list0 : A.list1;
    // ---- P0: bookkeeping of shell k-1 (block 0), frame activity, prefix
    if (blockIdx.x == 0) {
      if (k > 0) bookkeep(A, k);
      __syncthreads();
      for (int f = threadIdx.x; f < A.nF; f += blockDim.x) {
        if (A.done[f] == 0 && A.cnt[cur * A.nF + f] == 0 && A.remaining[f] > 0) A.done[f] = 2;
        A.cnt[nxt * A.nF + f] = 0;
        A.fills[nxt * A.nF + f] = 0;
        A.anyg[nxt * A.nF + f] = 0;
        A.best_key[f] = 0ULL;
        A.best_p[f] = 0x7fffffff;
      }
    }
    for (int f = threadIdx.x; f < A.nF; f += blockDim.x) {
      const int c = A.cnt[cur * A.nF + f];
      S.act[f] = (c > 0 && A.done[f] == 0) ? 1 : 0;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      int run = 0;
      for (int f = 0; f < A.nF; ++f) {
        S.pref[f] = run;
        if (S.act[f]) run += A.cnt[cur * A.nF + f];
      }
      S.pref[A.nF] = run;
      S.total = run;
    }
    __syncthreads();
    const int T = S.total;
    if (T == 0) break;
    trace_set(A, k, 0, gtimer());
    trace_set(A, k, 5, (unsigned long long)T);
    const int chunk = max(kGroupsPerBlock, (T + gridDim.x - 1) / gridDim.x);
    const int c_lo = min(T, blockIdx.x * chunk), c_hi = min(T, c_lo + chunk);

    // ---- A: fill
    for (int s = c_lo; s < c_hi;) {
      const int f = find_frame(S.pref, A.nF, s);
      const int fe = min(c_hi, S.pref[f + 1]);
      const float4* fw = A.work + (size_t)f * A.HW;
      WorkSource src{fw, A.c3 ? A.c3 + (size_t)f * A.HW : nullptr, A.H, A.W, A.C, k};
      const int dt_eff = (A.order == 2) && !A.dt_dead[f] && frontier_has_g(A, cur, f);
      int my_fills = 0;
      for (int base = s; base < fe; base += kGroupsPerBlock) {
        const int t = base + group;
        const bool valid = t < fe;
        const int j = valid ? t - S.pref[f] : 0;
        const uint32_t p = valid ? cur_list[(size_t)f * A.cap + j] : 0u;
        double gx = 0.0, gy = 0.0;
        if (valid) frame_guide(A, f, (int)p, gx, gy);
        SampleResult r;
        eval_item<NL>(P, S.tab, src, glane, valid, (double)((int)p % A.W), (double)((int)p / A.W), true, gx, gy, r);
        if (valid && glane == 0) {
          const double conf = r.rw / r.tw;
          bool ready;
          if (A.order == 0) {
            ready = true;
          } else if (!dt_eff) {
            ready = conf > A.c;
          } else {
            ready = (hypot_np(gx, gy) > A.c2) && (conf > A.c);
          }
          const bool fill = ready && (r.rw > 0.0);
          A.conf[(size_t)f * A.cap + j] = conf;
          if (fill) {
            float4 o;
            o.x = (float)r.v[0];
            o.y = (float)r.v[1];
            o.z = (float)r.v[2];
            o.w = __int_as_float(k + 1);
            A.work[(size_t)f * A.HW + p] = o;
            if (A.c3) A.c3[(size_t)f * A.HW + p] = (float)r.v[3];
            ++my_fills;
          }
        }
      }
      const int tot = block_sum(my_fills, S);
      if (threadIdx.x == 0 && tot > 0) atomicAdd(&A.fills[cur * A.nF + f], tot);
      s = fe;
    }
    trace_max(A, k, 1);
    grid.sync();
    trace_set(A, k, 2, gtimer());

    // ---- G: deadlock guard (engine.py:334-348), only when some frame stalled
    if (threadIdx.x == 0) {
      int any = 0;
      for (int f = 0; f < A.nF; ++f) {
        const int d = S.act[f] && A.fills[cur * A.nF + f] == 0;
        S.dl[f] = (unsigned char)d;
        any |= d;
      }
      S.any_dl = any;
    }
    __syncthreads();
    if (S.any_dl) {
      // G1: max confidence key per stalled frame
      for (int s = c_lo; s < c_hi;) {
        const int f = find_frame(S.pref, A.nF, s);
        const int fe = min(c_hi, S.pref[f + 1]);
        unsigned long long key = 0ULL;
        if (S.dl[f]) {
          for (int t = s + threadIdx.x; t < fe; t += blockDim.x) {
            const unsigned long long kk = conf_key(A.conf[(size_t)f * A.cap + (t - S.pref[f])]);
            key = kk > key ? kk : key;
          }
        }
        key = block_max_u64(key, S);
        if (threadIdx.x == 0 && S.dl[f]) atomicMax(&A.best_key[f], key);
        s = fe;
      }
      grid.sync();
      // G2: smallest pixel index among the maxima (sorted-frontier argmax)
      for (int s = c_lo; s < c_hi;) {
        const int f = find_frame(S.pref, A.nF, s);
        const int fe = min(c_hi, S.pref[f + 1]);
        if (S.dl[f]) {
          const unsigned long long best = A.best_key[f];
          for (int t = s + threadIdx.x; t < fe; t += blockDim.x) {
            const int j = t - S.pref[f];
            if (conf_key(A.conf[(size_t)f * A.cap + j]) == best)
              atomicMin(&A.best_p[f], (int)cur_list[(size_t)f * A.cap + j]);
          }
        }
        s = fe;
      }
      grid.sync();
      // G3: the guarded fill, one warp-group per stalled frame
      for (int fb = blockIdx.x * kGroupsPerBlock; fb < A.nF; fb += gridDim.x * kGroupsPerBlock) {
        const int f = fb + group;
        const bool valid = f < A.nF && S.dl[f];
        const int p = valid ? A.best_p[f] : 0;
        const int fs = valid ? f : 0;
        double gx = 0.0, gy = 0.0;
        if (valid) frame_guide(A, f, p, gx, gy);
        WorkSource src{A.work + (size_t)fs * A.HW, A.c3 ? A.c3 + (size_t)fs * A.HW : nullptr,
                       A.H, A.W, A.C, k};
        SampleResult r;
        eval_item<NL>(P, S.tab, src, glane, valid, (double)(p % A.W), (double)(p / A.W), true, gx, gy, r);
        if (valid && glane == 0) {
          double v[4] = {r.v[0], r.v[1], r.v[2], r.v[3]};
          bool ok = r.rw > 0.0;
          if (!ok) {
            // mean of readable 8-neighbours, engine.py:252-267
            double acc[4] = {0.0, 0.0, 0.0, 0.0};
            int n = 0;
            const int i = p % A.W, j = p / A.W;
            const int offs[8][2] = {{-1, -1}, {0, -1}, {1, -1}, {-1, 0},
                                    {1, 0},   {-1, 1}, {0, 1},  {1, 1}};
            for (int o = 0; o < 8; ++o) {
              int ii = i + offs[o][0];
              const int jj = j + offs[o][1];
              if (A.periodic) ii = pos_mod(ii, A.W);
              if (ii < 0 || ii >= A.W || jj < 0 || jj >= A.H) continue;
              double cv[4];
              if (src.load(jj * A.W + ii, cv)) {
                for (int c = 0; c < 4; ++c) acc[c] += cv[c];
                ++n;
              }
            }
            if (n > 0) {
              for (int c = 0; c < 4; ++c) v[c] = acc[c] / n;
              ok = true;
            }
          }
          if (ok) {
            float4 o;
            o.x = (float)v[0];
            o.y = (float)v[1];
            o.z = (float)v[2];
            o.w = __int_as_float(k + 1);
            A.work[(size_t)f * A.HW + p] = o;
            if (A.c3) A.c3[(size_t)f * A.HW + p] = (float)v[3];
            A.fills[cur * A.nF + f] = 1;
            A.deadlocks[f] += 1;
          } else {
            A.done[f] = 2;  // unfillable: engine.py:342-345
            A.last_f[f] = A.cnt[cur * A.nF + f];
          }
        }
      }
      grid.sync();
    }

    // ---- B: frontier update
    if (kTracked) {
      for (int s = c_lo; s < c_hi;) {
        const int f = find_frame(S.pref, A.nF, s);
        const int fe = min(c_hi, S.pref[f + 1]);
        const bool live = A.done[f] == 0;
        float4* fw = A.work + (size_t)f * A.HW;
        for (int base = s; base < fe; base += kThreads) {
          const int t = base + threadIdx.x;
          const bool valid = live && t < fe;
          const uint32_t p = valid ? cur_list[(size_t)f * A.cap + (t - S.pref[f])] : 0u;
          const int st = valid ? stamp_of(fw, (int)p) : 0;
          const bool filled = valid && st == k + 1;
          // survivor keeps its slot
          push_append(S, valid && !filled, p);
          const int i = (int)p % A.W, j = (int)p / A.W;
#pragma unroll
          for (int o = 0; o < 8; ++o) {
            const int di = (o < 3) ? o - 1 : (o == 3 ? -1 : (o == 4 ? 1 : o - 6));
            const int dj = (o < 3) ? -1 : (o < 5 ? 0 : 1);
            bool want = false;
            int q = 0;
            if (filled) {
              int ii = i + di;
              const int jj = j + dj;
              if (A.periodic) ii = pos_mod(ii, A.W);
              if (ii >= 0 && ii < A.W && jj >= 0 && jj < A.H) {
                q = jj * A.W + ii;
                if (stamp_of(fw, q) == kStampInactive &&
                    atomicCAS(stamp_ptr(fw, q), kStampInactive, kStampActive) == kStampInactive) {
                  want = true;
                  if (A.enter) A.enter[(size_t)f * A.HW + q] = k + 1;
                }
              }
            }
            push_append(S, want, (uint32_t)q);
          }
          flush_appends(A, S, f, nxt_list, nxt);
        }
        s = fe;
      }
    } else {
      // untracked: rescan every pixel of every active frame (engine.py:357-360)
      int nA = 0;
      for (int f = 0; f < A.nF; ++f) nA += S.act[f] && A.done[f] == 0;
      const long long TP = (long long)nA * A.HW;
      const long long pchunk = ((TP + gridDim.x - 1) / gridDim.x + kThreads - 1) / kThreads * kThreads;
      const long long p_lo = min(TP, (long long)blockIdx.x * pchunk), p_hi = min(TP, p_lo + pchunk);
      for (long long s = p_lo; s < p_hi;) {
        const int a = (int)(s / A.HW);
        int f = -1;
        for (int ff = 0, seen = 0; ff < A.nF; ++ff)
          if (S.act[ff] && A.done[ff] == 0) {
            if (seen == a) { f = ff; break; }
            ++seen;
          }
        const long long fe = min(p_hi, (long long)(a + 1) * A.HW);
        float4* fw = A.work + (size_t)f * A.HW;
        for (long long base = s; base < fe; base += kThreads) {
          const long long t = base + threadIdx.x;
          bool want = false;
          int p = 0;
          if (t < fe) {
            p = (int)(t - (long long)a * A.HW);
            const int st = stamp_of(fw, p);
            if (st == kStampInactive || st == kStampActive) {
              const int i = p % A.W, j = p / A.W;
              for (int dj = -1; dj <= 1 && !want; ++dj) {
                const int jj = j + dj;
                if (jj < 0 || jj >= A.H) continue;
                for (int di = -1; di <= 1; ++di) {
                  if (di == 0 && dj == 0) continue;
                  int ii = i + di;
                  if (A.periodic) ii = pos_mod(ii, A.W);
                  else if (ii < 0 || ii >= A.W) continue;
                  if (stamp_of(fw, jj * A.W + ii) <= k + 1) {
                    want = true;
                    break;
                  }
                }
              }
              if (want && st == kStampInactive) {
                *stamp_ptr(fw, p) = kStampActive;
                if (A.enter) A.enter[(size_t)f * A.HW + p] = k + 1;
              }
            }
          }
          push_append(S, want, (uint32_t)p);
          flush_appends(A, S, f, nxt_list, nxt);
        }
        s = fe;
      }
    }
    trace_max(A, k, 3);
    grid.sync();
    trace_set(A, k, 4, gtimer());
  }
  // final bookkeeping: stats
  if (blockIdx.x == 0) {
    for (int f = threadIdx.x; f < A.nF; f += blockDim.x) {
      int* st = A.stats + (size_t)f * GF_STATS;
      st[GF_STAT_ITERATIONS] = A.iters[f];
      st[GF_STAT_FILLED] = A.filled[f];
      st[GF_STAT_DEADLOCK] = A.deadlocks[f];
      st[GF_STAT_UNFILLABLE] = (A.remaining[f] > 0) ? 1 : 0;
      st[GF_STAT_REMAINING] = A.remaining[f];
      st[GF_STAT_INPAINT] = A.inpaint[f];
      st[GF_STAT_ROWS_OVERFLOW] = A.overflow[f];
      st[GF_STAT_LAST_FRONTIER] = A.last_f[f];
    }
  }
}

// ------------------------------------------------------------ finalize

template <typename T>
__global__ void __launch_bounds__(kThreads) k_finalize(FillArgs A) {
  const long long total = (long long)A.nF * A.HW;
  for (long long g = (long long)blockIdx.x * blockDim.x + threadIdx.x; g < total;
       g += (long long)gridDim.x * blockDim.x) {
    const int f = (int)(g / A.HW);
    const float4 px = A.work[g];
    const int st = __float_as_int(px.w);
    const bool filled = st >= 1 && st < kStampInactive;
    const unsigned long long elo = ~A.hull[2 * f], ehi = A.hull[2 * f + 1];
    const bool has_hull = ehi != 0ULL;
    const double lo = has_hull ? dec_ordered(elo) : 0.0;
    const double hi = has_hull ? dec_ordered(ehi) : 0.0;
    const T* in = reinterpret_cast<const T*>(A.image) + (size_t)g * A.C;
    T* out = reinterpret_cast<T*>(A.out) + (size_t)g * A.C;
    const float fv[4] = {px.x, px.y, px.z, A.c3 ? A.c3[g] : 0.f};
    for (int c = 0; c < A.C; ++c) {
      double v = filled ? (double)fv[c] : (double)in[c];
      if (has_hull) v = (v < lo) ? lo : ((v > hi) ? hi : v);
      out[c] = (T)v;
    }
    if (A.fillshell) A.fillshell[g] = filled ? st - 1 : -1;
  }
}

// ---------------------------------------------------------------- host

static size_t align_up(size_t x) { return (x + 255) & ~size_t(255); }

struct Layout {
  size_t work, c3, list0, list1, conf, gfield, ints, u64, total;
};

static Layout layout_for(int nF, int HW, int C, bool raster) {
  Layout L;
  size_t off = 0;
  const size_t n = (size_t)nF * HW;
  L.work = off; off = align_up(off + n * sizeof(float4));
  L.gfield = off; off = align_up(off + (raster ? n * 2 * sizeof(double) : 0));
  L.c3 = off; off = align_up(off + (C > 3 ? n * sizeof(float) : 0));
  L.list0 = off; off = align_up(off + n * sizeof(uint32_t));
  L.list1 = off; off = align_up(off + n * sizeof(uint32_t));
  L.conf = off; off = align_up(off + n * sizeof(double));
  L.ints = off; off = align_up(off + (size_t)nF * kIntsPerFrame * sizeof(int));
  L.u64 = off; off = align_up(off + (size_t)nF * 4 * sizeof(unsigned long long));
  L.total = off;
  return L;
}

size_t fill_workspace_bytes(int nF, int H, int W, int C, bool raster) {
  if (nF <= 0 || H <= 0 || W <= 0) return 0;
  return layout_for(nF, H * W, C, raster).total;
}

static int coop_grid(const void* fn, size_t smem, int* out_grid) {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return GF_E_CUDA;
  int sms = 0, coop = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, dev);
  if (!coop) return set_error(GF_E_UNSUPPORTED, "device lacks cooperative launch");
  if (cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
    return set_error(GF_E_CUDA, "cudaFuncSetAttribute failed");
  int per_sm = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, kThreads, smem) != cudaSuccess ||
      per_sm <= 0)
    return set_error(GF_E_CUDA, "occupancy query failed");
  *out_grid = sms * per_sm;
  return GF_OK;
}

int fill_launch(const gf_frames* fr, const gf_fill_params* prm, const gf_fill_outputs* out,
                const gf_splines* spl, void* ws, size_t ws_bytes, cudaStream_t stream,
                const BallParams& P, const BallTables& host_tab) {
  const int nF = fr->n_frames, H = fr->height, W = fr->width, C = fr->channels;
  const int HW = H * W;
  const bool raster = spl && spl->n_seg > 0;
  const Layout L = layout_for(nF, HW, C, raster);
  if (ws_bytes < L.total) return set_error(GF_E_WORKSPACE, "workspace too small");
  unsigned char* base = static_cast<unsigned char*>(ws);

  FillArgs A;
  memset(&A, 0, sizeof(A));
  A.nF = nF; A.H = H; A.W = W; A.HW = HW; A.C = C; A.cap = HW;
  A.image = fr->image;
  A.labels = fr->labels;
  A.guide = fr->guide;
  A.gsrc = fr->guide;
  A.out = fr->out;
  if (raster) {
    A.gfield = reinterpret_cast<double*>(base + L.gfield);
    A.gsrc = A.gfield;
    A.n_seg = spl->n_seg;
    A.seg = reinterpret_cast<const double4*>(spl->seg);
    A.seg_spline = spl->seg_spline;
    A.dirs = reinterpret_cast<const double2*>(spl->dirs);
    A.cut = 3.0 * spl->eta;
    A.c2eta = 2.0 * spl->eta * spl->eta;
  }
  A.trace = reinterpret_cast<unsigned long long*>(out->shell_trace);
  A.trace_cap = out->shell_trace ? out->trace_cap : 0;
  A.work = reinterpret_cast<float4*>(base + L.work);
  A.c3 = C > 3 ? reinterpret_cast<float*>(base + L.c3) : nullptr;
  A.list0 = reinterpret_cast<uint32_t*>(base + L.list0);
  A.list1 = reinterpret_cast<uint32_t*>(base + L.list1);
  A.conf = reinterpret_cast<double*>(base + L.conf);
  int* ints = reinterpret_cast<int*>(base + L.ints);
  A.cnt = ints;              ints += 2 * nF;
  A.fills = ints;            ints += 2 * nF;
  A.anyg = ints;             ints += 2 * nF;
  A.remaining = ints;        ints += nF;
  A.iters = ints;            ints += nF;
  A.done = ints;             ints += nF;
  A.deadlocks = ints;        ints += nF;
  A.filled = ints;           ints += nF;
  A.dt_dead = ints;          ints += nF;
  A.best_p = ints;           ints += nF;
  A.inpaint = ints;          ints += nF;
  A.overflow = ints;         ints += nF;
  A.last_f = ints;           ints += nF;
  unsigned long long* u64 = reinterpret_cast<unsigned long long*>(base + L.u64);
  A.best_key = u64;
  A.hull = u64 + nF;
  A.stats = out->frame_stats;
  A.rows = out->rows;
  A.rows_cap = out->rows_cap;
  A.enter = out->enter;
  A.fillshell = out->fillshell;
  A.order = prm->order;
  A.c = prm->c;
  A.c2 = prm->c2;
  A.g_mode = raster ? GF_G_FIELD : prm->g_mode;
  A.gfx = prm->g_fixed[0];
  A.gfy = prm->g_fixed[1];
  A.periodic = prm->periodic_x;
  A.dtype = fr->dtype;

  // per-frame counters start at zero (the hull minimum is stored inverted
  // and the data-term latch as a "dead" flag, so zero is the initial state)
  if (cudaMemsetAsync(base + L.ints, 0, L.u64 + (size_t)nF * 4 * sizeof(unsigned long long) - L.ints,
                      stream) != cudaSuccess)
    return set_error(GF_E_CUDA, "memset failed");
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const long long total = (long long)nF * HW;
  {
    const int bpf = std::max(1, std::min((HW + kThreads - 1) / kThreads,
                                         std::max(1, sms * 8 / std::max(1, nF))));
    const dim3 pgrid(bpf, nF);
    if (fr->dtype == GF_F64)
      k_prep<double><<<pgrid, kThreads, 0, stream>>>(A);
    else
      k_prep<float><<<pgrid, kThreads, 0, stream>>>(A);
  }
  if (cudaPeekAtLastError() != cudaSuccess)
    return set_error(GF_E_CUDA, cudaGetErrorString(cudaGetLastError()));

  const size_t smem = sizeof(Smem);
  const bool multi = P.plan.n_leaves > 1;
  const void* fn;
  if (prm->tracked)
    fn = multi ? (const void*)k_shells<kMaxLeaves, true> : (const void*)k_shells<1, true>;
  else
    fn = multi ? (const void*)k_shells<kMaxLeaves, false> : (const void*)k_shells<1, false>;
  int grid = 0;
  int rc = coop_grid(fn, smem, &grid);
  if (rc != GF_OK) return rc;
  void* args[] = {(void*)&A, (void*)&P, (void*)&host_tab};
  cudaError_t e = cudaLaunchCooperativeKernel(fn, grid, kThreads, args, smem, stream);
  if (e != cudaSuccess) return set_error(GF_E_CUDA, cudaGetErrorString(e));

  const int fgrid = (int)std::min<long long>((total + kThreads - 1) / kThreads, (long long)sms * 16);
  if (fr->dtype == GF_F64)
    k_finalize<double><<<fgrid, kThreads, 0, stream>>>(A);
  else
    k_finalize<float><<<fgrid, kThreads, 0, stream>>>(A);
  e = cudaPeekAtLastError();
  if (e != cudaSuccess) return set_error(GF_E_CUDA, cudaGetErrorString(e));
  return GF_OK;
}

}  // namespace gf
