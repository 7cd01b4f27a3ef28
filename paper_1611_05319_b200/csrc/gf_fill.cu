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
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <stdlib.h>

#include <mutex>
#include <vector>

#include "gf_eval.cuh"
#include "gf_internal.cuh"

namespace cg = cooperative_groups;

namespace gf {

constexpr int kThreads = 256;
constexpr int kGroupsPerBlock = kThreads / kGroup;
#ifndef GF_SHELL_THREADS
#define GF_SHELL_THREADS 256
#endif
constexpr int kShellThreads = GF_SHELL_THREADS;  // block size of the shell loop
constexpr int kAppendCap = kShellThreads * 9;

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

// order-preserving 32-bit code of a float (larger value -> larger code)
__device__ __forceinline__ unsigned enc32(float x) {
  const unsigned b = __float_as_uint(x);
  return (b >> 31) ? ~b : (b | 0x80000000u);
}
__device__ __forceinline__ float dec32(unsigned e) {
  return __uint_as_float((e >> 31) ? (e & 0x7fffffffu) : ~e);
}
// horizontal dilation of a halo row's Inpaint mask: bit c <=> an Inpaint
// pixel in ext columns [c, c + 2R]
__device__ __forceinline__ unsigned int hdilate(unsigned long long m, int R) {
  unsigned long long h = m;
  int w = 1;  // h covers a window of w columns
  while (2 * w <= 2 * R + 1) {
    h |= h >> w;
    w *= 2;
  }
  if (w < 2 * R + 1) h |= h >> (2 * R + 1 - w);
  return (unsigned int)h;
}

// 4 byte-wise test results (0xff / 0x00 per byte) -> 4 bits, byte i -> bit i
__device__ __forceinline__ unsigned nib4(unsigned m) { return ((m & 0x01010101u) * 0x01020408u) >> 24; }

// pixel index -> (column, row) without an integer division: the launch's
// round-up multiplier for W (host: div_magic)
__device__ __forceinline__ int row_of(const FillArgs& A, int p) {
  return A.W == 1 ? p : (int)(__umulhi((unsigned)p, A.w_mul) >> A.w_shr);
}
__device__ __forceinline__ void col_row(const FillArgs& A, int p, int& i, int& j) {
  j = row_of(A, p);
  i = p - j * A.W;
}

__device__ __forceinline__ int stamp_of(const float4* work, int q) {
  return __float_as_int(work[q].w);
}
__device__ __forceinline__ int* stamp_ptr(float4* work, int q) {
  return reinterpret_cast<int*>(&work[q].w);
}

// ---------------------------------------------------------------- prep
//
// One pass over every pixel in 32x32 tiles, frame-major grid
// (blockIdx.z = frame).  Labels of the tile plus an (r+1)-pixel halo are
// staged in shared memory; from them the block derives
//   * which pixels can ever be read by the shell loop -- those within
//     Chebyshev distance r+1 of an Inpaint pixel (a ball sample lies within
//     r of its centre, its bilinear corners within r+1), found with a
//     ballot bitmask dilation -- only these get a working-buffer entry;
//   * the initial frontier (Inpaint with a Readable 8-neighbour,
//     grid.py:104-106), |D|, the value hull (engine.py:291-296);
//   * the guide field g of every Inpaint pixel (guide.py:303-327), rastered
//     in place from the splines when given -- segments are culled against
//     the tile's box inflated by 3 eta; a non-zero g needs its nearest
//     segment within 3 eta, which then survives the cull, so non-zero g
//     are bit-identical to the dense rasteriser (pixels with no candidate
//     get +0; the reference's -0 there is indistinguishable to the fill).
// Readable pixels are copied straight to the output: the final hull clip
// (engine.py:372-375) is the identity on them.  k_finalize writes the rest.

__device__ __forceinline__ unsigned long long gtimer0() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
// pipeline timeline in the last trace row: slots 2i = ~start (max of ~t =
// earliest start), 2i+1 = latest end; i = 0 prep, 1 shell loop, 2 finalize
__device__ __forceinline__ void timeline_mark(const FillArgs& A, int stage, bool start) {
  if (threadIdx.x != 0 || !A.trace || A.trace_cap < 2) return;
  unsigned long long* row = A.trace + (size_t)(A.trace_cap - 1) * 8;
  const unsigned long long t = gtimer0();
  atomicMax(&row[2 * stage + (start ? 0 : 1)], start ? ~t : t);
}

#ifdef GF_PREP_PROF
// experiment builds only: per-block stage stamps of the prep pass
// [0] start, [1..6] stages, [7] smid | flags << 32
__device__ unsigned long long g_prep_prof[16384][12];
// k_shells: first block entry, first / last return from the PDL wait
__device__ unsigned long long g_shell_prof[3];
extern "C" int gf_prep_prof_read(void* host, int n) {
  if (n == -2) return (int)cudaMemcpyToSymbol(g_shell_prof, host, 24);  // reset
  if (n < 0) return (int)cudaMemcpyFromSymbol(host, g_shell_prof, 24);
  return (int)cudaMemcpyFromSymbol(host, g_prep_prof, (size_t)n * 96);
}
#define PREP_PROF_T0 \
  if (threadIdx.x == 0 && tile < 16384) g_prep_prof[tile][0] = gtimer0()
#define PREP_STAGE(k) \
  if (threadIdx.x == 0 && tile < 16384) g_prep_prof[tile][k] = gtimer0()
#define PREP_PROF(flags)                                                      \
  if (threadIdx.x == 0 && tile < 16384) {                                     \
    unsigned sm_;                                                             \
    asm volatile("mov.u32 %0, %%smid;" : "=r"(sm_));                          \
    g_prep_prof[tile][10] = gtimer0();                                        \
    g_prep_prof[tile][11] = sm_ | ((unsigned long long)(flags) << 32);         \
  }
#else
#define PREP_PROF_T0
#define PREP_STAGE(k)
#define PREP_PROF(flags)
#endif

// Programmatic dependent launch: each k_prep block signals at its start, so
// the shell kernel's launch and block set-up overlap the last prep wave; the
// shell kernel waits for k_prep's completion (and memory) before its first
// read.
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;"); }
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

constexpr int kMaxCand = 512;
constexpr int kLabBoxMax = 64;  // label box row: columns tx0 - 16 .. tx0 + 47 (a TMA box
                                // must start on a 16-byte boundary)

// TMA descriptors of one k_prep_tma launch: image / output (W*C, H, nF) in the
// caller's dtype, labels (W, H, nF) u8
struct PrepMaps {
  CUtensorMap img, out, lab;
  int lab_bw;  // label box width in bytes (kLabBoxMax)
};
constexpr int kTile = 32;
constexpr int kMaxHalo = GF_MAX_RADIUS + 1;
constexpr int kTileExt = kTile + 2 * kMaxHalo;  // 58 <= 64: one 64-bit row mask

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

// One pass over every pixel in 32x32 tiles, frame-major grid (blockIdx.z =
// frame).  Every tile copies its pixels to the output (Readable pixels are
// final: the closing hull clip, engine.py:372-375, is the identity on them;
// fills and the Bystander clip overwrite the others later) and reduces the
// value hull of its Readable values (engine.py:291-296).  Tiles with an
// Inpaint pixel within reach go on to the D-tile work below.
template <typename T, int C>
#ifndef GF_PREP_MIN_BLOCKS
#define GF_PREP_MIN_BLOCKS 4
#endif
__global__ void __launch_bounds__(kThreads, GF_PREP_MIN_BLOCKS) k_prep(const __grid_constant__ FillArgs A) {
  // grid (tile column, tile row, frame): no division for the tile index
  const int f = blockIdx.z;
  const int tiles_x = gridDim.x;
  const int tix = blockIdx.x, tiy = blockIdx.y;
  const int tile = tiy * tiles_x + tix;
  const int tx0 = tix * kTile;
  const int ty0 = tiy * kTile;
  timeline_mark(A, 0, true);
  // every prep block is resident once all have passed here: the shell
  // kernel may start launching (it waits for this grid's completion)
  pdl_trigger();
  const int R = A.halo;
  const int ext = kTile + 2 * R;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  __shared__ unsigned int s_hrow[kTileExt];
  __shared__ unsigned int s_vrow[kTile];
  __shared__ unsigned long long s_hrow64[kTileExt];
  __shared__ unsigned long long s_rrow64[kTileExt];
  __shared__ int s_cand[kMaxCand];
  __shared__ int s_ncand;
  __shared__ uint16_t s_inp[kTile * kTile];
  __shared__ unsigned int s_rotb[kTile];
  __shared__ int s_ninp, s_anyg;
  __shared__ int s_cnt[kThreads / 32];
  __shared__ int s_wl[kThreads / 32], s_wr[kThreads / 32];
  __shared__ int s_bL, s_bR;
  __shared__ unsigned long long s_red[4][kThreads / 32];
  const uint8_t* lab = A.labels + (size_t)f * A.HW;
  const T* img = reinterpret_cast<const T*>(A.image) + (size_t)f * A.HW * C;
  float4* work = A.work + (size_t)f * A.HW;
  const bool raster = A.n_seg > 0;
  const int ry = threadIdx.x >> 3;
  const int c0 = (threadIdx.x & 7) * 4;
  const int gy = ty0 + ry;

  // 1. Inpaint / Readable bitmasks of the tile + halo rows (bit x <=> ext
  //    column x; out of lattice = neither, x wraps when periodic).  Interior
  //    tiles read 32-bit words, two rows per warp instruction, and pack each
  //    word's 4 byte tests into a nibble (one multiply); the OR of 16 lanes'
  //    nibbles is one redux.  Edge tiles fall back to byte loads + ballots.
  if (threadIdx.x == 0) {
    s_ncand = 0;
    s_ninp = 0;
    s_anyg = 0;
  }
  if (threadIdx.x < kTile) s_rotb[threadIdx.x] = 0u;
  bool any_inp = false;
  const int sh = (tx0 - R) & 3;       // ext column 0 within its aligned word
  const int ws = tx0 - R - sh;        // first word's global column
  const int nw = (ext + sh + 3) >> 2;  // words per row (<= 16)
  const unsigned long long ext_mask = ext >= 64 ? ~0ULL : ((1ULL << ext) - 1);
  if ((A.W & 3) == 0 && ws >= 0 && ws + 4 * nw <= A.W) {
    // four threads per ext row (all warps busy), four aligned words each,
    // combined with two xor shuffles
    const int y = threadIdx.x >> 2, part = threadIdx.x & 3;
    const int gyy = ty0 - R + y;
    unsigned long long im = 0ULL, rm = 0ULL;
    if (y < ext && gyy >= 0 && gyy < A.H) {
      const unsigned* row = reinterpret_cast<const unsigned*>(lab + (size_t)gyy * A.W + ws);
      unsigned w[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) w[i] = 4 * part + i < nw ? __ldg(row + 4 * part + i) : 0x80808080u;
      // for the label values 0 / 128 / 255: Inpaint <=> bit 0 set, Readable
      // <=> bit 7 clear (any other value flags the frame as invalid above and
      // its result is discarded)
      unsigned ib = 0, rb = 0;
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        ib |= nib4(w[i]) << (4 * i);
        rb |= nib4(~w[i] >> 7) << (4 * i);
      }
      im = (unsigned long long)ib << (16 * part);
      rm = (unsigned long long)rb << (16 * part);
    }
    im |= __shfl_xor_sync(0xffffffffu, im, 1);
    rm |= __shfl_xor_sync(0xffffffffu, rm, 1);
    im |= __shfl_xor_sync(0xffffffffu, im, 2);
    rm |= __shfl_xor_sync(0xffffffffu, rm, 2);
    if (part == 0 && y < ext) {
      im = (im >> sh) & ext_mask;
      rm = (rm >> sh) & ext_mask;
      s_hrow64[y] = im;
      s_rrow64[y] = rm;
      s_hrow[y] = hdilate(im, R);
      any_inp = im != 0ULL;
    }
  } else {
    constexpr int kRowsPerWarp = (kTileExt + kThreads / 32 - 1) / (kThreads / 32);
    uint8_t l2[kRowsPerWarp][2];
#pragma unroll
    for (int i = 0; i < kRowsPerWarp; ++i) {
      const int y = warp + i * (kThreads / 32);
      const int gyy = ty0 - R + y;
      const bool row_ok = y < ext && gyy >= 0 && gyy < A.H;
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int x = lane + 32 * h;
        int gxx = tx0 - R + x;
        if (A.periodic) gxx = gxx < 0 ? gxx + A.W : (gxx >= A.W ? gxx - A.W : gxx);
        const bool in = x < ext && row_ok && gxx >= 0 && gxx < A.W;
        l2[i][h] = in ? __ldg(lab + gyy * A.W + gxx) : (uint8_t)128;
      }
    }
#pragma unroll
    for (int i = 0; i < kRowsPerWarp; ++i) {
      const int y = warp + i * (kThreads / 32);
      const unsigned lo = __ballot_sync(0xffffffffu, y < ext && l2[i][0] == 255);
      const unsigned hi = __ballot_sync(0xffffffffu, y < ext && l2[i][1] == 255);
      const unsigned rlo = __ballot_sync(0xffffffffu, y < ext && l2[i][0] == 0);
      const unsigned rhi = __ballot_sync(0xffffffffu, y < ext && l2[i][1] == 0);
      any_inp |= (lo | hi) != 0;
      if (lane == 0 && y < ext) {
        s_hrow64[y] = ((unsigned long long)hi << 32) | lo;
        s_rrow64[y] = ((unsigned long long)rhi << 32) | rlo;
        s_hrow[y] = hdilate(((unsigned long long)hi << 32) | lo, R);
      }
    }
  }
  // labels of the thread's own 4 pixels (byte u = column c0 + u)
  uint32_t own4 = 0x80808080u;
  if (gy < A.H) {
    if ((A.W & 3) == 0 && tx0 + c0 < A.W) {
      own4 = __ldg(reinterpret_cast<const uint32_t*>(lab + (size_t)gy * A.W + tx0 + c0));
    } else {
#pragma unroll
      for (int u = 0; u < 4; ++u)
        if (tx0 + c0 + u < A.W)
          own4 = (own4 & ~(0xffu << (8 * u))) | ((uint32_t)lab[(size_t)gy * A.W + tx0 + c0 + u] << (8 * u));
    }
  }
  // the thread's 4 pixels: loads issued before the label sync
  const int gx0 = tx0 + c0;
  constexpr int nv = (4 * C * (int)sizeof(T)) / 16;
  constexpr bool vec_ok = (4 * C * (int)sizeof(T)) % 16 == 0;
  const bool row_in = gy < A.H;
  const bool vec = vec_ok && (A.W % 4 == 0) && row_in && gx0 < A.W;
  union {
    T t[4 * C];
    uint4 q[nv > 0 ? nv : 1];
  } px;
  if (vec) {
    const uint4* src = reinterpret_cast<const uint4*>(img + ((size_t)gy * A.W + gx0) * C);
#pragma unroll
    for (int i = 0; i < nv; ++i) px.q[i] = __ldg(src + i);
  } else {
#pragma unroll
    for (int u = 0; u < 4; ++u)
#pragma unroll
      for (int ch = 0; ch < C; ++ch)
        px.t[u * C + ch] = (row_in && gx0 + u < A.W) ? __ldg(img + ((size_t)gy * A.W + gx0 + u) * C + ch) : T(0);
  }
  // label validation (grid.py:36-46) rides on the own-pixel load: any byte
  // outside {0, 128, 255} flags the frame
  {
    const unsigned bad = ~(__vcmpeq4(own4, 0u) | __vcmpeq4(own4, 0x80808080u) |
                           __vcmpeq4(own4, 0xffffffffu));
    if (bad && gy < A.H) {
      unsigned valid = 0;  // bytes of in-lattice columns
#pragma unroll
      for (int u = 0; u < 4; ++u)
        if (tx0 + c0 + u < A.W) valid |= 0xffu << (8 * u);
      if (bad & valid) A.badlab[f] = 1;
    }
  }
  const bool tile_d = __syncthreads_or(any_inp);
  // copy to the output + value hull of the Readable pixels
  {
    T* out = reinterpret_cast<T*>(A.out) + (size_t)f * A.HW * C;
    if (vec) {
      uint4* dst = reinterpret_cast<uint4*>(out + ((size_t)gy * A.W + gx0) * C);
#pragma unroll
      for (int i = 0; i < nv; ++i) dst[i] = px.q[i];
    } else {
#pragma unroll
      for (int u = 0; u < 4; ++u)
        if (row_in && gx0 + u < A.W)
#pragma unroll
          for (int ch = 0; ch < C; ++ch) out[((size_t)gy * A.W + gx0 + u) * C + ch] = px.t[u * C + ch];
    }
    // [0] value hull of the Readable pixels, [1] range of the Bystanders
    // per pixel: channel min / max, then merged into its class (branch-free)
    T vlo[2] = {T(INFINITY), T(INFINITY)}, vhi[2] = {T(-INFINITY), T(-INFINITY)};
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const uint8_t l = (uint8_t)(own4 >> (8 * u));
      T mn = px.t[u * C], mx = px.t[u * C];
#pragma unroll
      for (int ch = 1; ch < C; ++ch) {
        mn = fmin(mn, px.t[u * C + ch]);
        mx = fmax(mx, px.t[u * C + ch]);
      }
      const bool in = row_in && gx0 + u < A.W;
      const bool rd = in && l == 0, by = in && l == 128;
      vlo[0] = rd ? fmin(vlo[0], mn) : vlo[0];
      vhi[0] = rd ? fmax(vhi[0], mx) : vhi[0];
      vlo[1] = by ? fmin(vlo[1], mn) : vlo[1];
      vhi[1] = by ? fmax(vhi[1], mx) : vhi[1];
    }
    unsigned long long ered[4];  // max(~enc) <=> min(enc)
    if constexpr (sizeof(T) == 4) {
      // fp32 values: order-preserving 32-bit codes, one redux per quantity
      unsigned m[4];
#pragma unroll
      for (int b = 0; b < 2; ++b) {
        const bool any = vlo[b] <= vhi[b];
        m[2 * b] = __reduce_max_sync(0xffffffffu, any ? ~enc32((float)vlo[b]) : 0u);
        m[2 * b + 1] = __reduce_max_sync(0xffffffffu, any ? enc32((float)vhi[b]) : 0u);
      }
      // the block reduces the 32-bit codes; the fp64 codes are made once
      // per block below
#pragma unroll
      for (int i = 0; i < 4; ++i) ered[i] = m[i];
    } else {
#pragma unroll
      for (int b = 0; b < 2; ++b) {
        ered[2 * b] = vlo[b] <= vhi[b] ? ~enc_ordered((double)vlo[b]) : 0ULL;
        ered[2 * b + 1] = vlo[b] <= vhi[b] ? enc_ordered((double)vhi[b]) : 0ULL;
      }
#pragma unroll
      for (int i = 0; i < 4; ++i)
        for (int o = 16; o > 0; o >>= 1) {
          const unsigned long long a = __shfl_xor_sync(0xffffffffu, ered[i], o);
          ered[i] = a > ered[i] ? a : ered[i];
        }
    }
#pragma unroll
    for (int i = 0; i < 4; ++i)
      if (lane == 0) s_red[i][warp] = ered[i];
    if (A.fillshell && row_in) {
      int* fsh = A.fillshell + (size_t)f * A.HW + (size_t)gy * A.W + gx0;
#pragma unroll
      for (int u = 0; u < 4; ++u)
        if (gx0 + u < A.W) fsh[u] = -1;
    }
    __syncthreads();
    if (threadIdx.x < 4) {
      const int i = threadIdx.x;
      unsigned long long e = 0ULL;
      for (int w = 0; w < kThreads / 32; ++w) e = s_red[i][w] > e ? s_red[i][w] : e;
      if constexpr (sizeof(T) == 4) {
        // 32-bit order codes of fp32 values -> the fp64 codes of the hull
        const unsigned m = (unsigned)e;
        e = (i & 1) ? (m ? enc_ordered((double)dec32(m)) : 0ULL)
                    : (m ? ~enc_ordered((double)dec32(~m)) : 0ULL);
      }
      // i < 2: the frame's hull (most tiles cannot move it any more: skip
      // their atomics); i >= 2: the tile's Bystander range, read by the
      // shell loop's clip, and the frame's
      unsigned long long* fr = i < 2 ? &A.hull[2 * f + i] : &A.bys_frame[2 * f + i - 2];
      if (e != 0ULL && e > *(volatile unsigned long long*)fr) atomicMax(fr, e);
      if (i >= 2) A.bys[((size_t)f * A.ntiles + tile) * 2 + i - 2] = e;
    }
  }
  if (!tile_d) {
    // no Inpaint pixel within reach: nothing of this tile is ever sampled
    if (A.enter && row_in) {
      int* en = A.enter + (size_t)f * A.HW + (size_t)gy * A.W + gx0;
#pragma unroll
      for (int u = 0; u < 4; ++u)
        if (gx0 + u < A.W) en[u] = -1;
    }
    timeline_mark(A, 0, false);
    return;
  }
  if (raster) {
    const double x0 = (double)tx0, x1 = (double)min(A.W - 1, tx0 + kTile - 1);
    const double y0 = (double)ty0, y1 = (double)min(A.H - 1, ty0 + kTile - 1);
    const int s0 = A.frame_seg ? A.frame_seg[f] : 0;
    const int s1 = A.frame_seg ? A.frame_seg[f + 1] : A.n_seg;
    for (int i = s0 + threadIdx.x; i < s1; i += kThreads) {
      const double4 sg = A.seg[i];
      const double lo_x = fmin(sg.x, sg.z) - A.cut, hi_x = fmax(sg.x, sg.z) + A.cut;
      const double lo_y = fmin(sg.y, sg.w) - A.cut, hi_y = fmax(sg.y, sg.w) + A.cut;
      if (hi_x >= x0 && lo_x <= x1 && hi_y >= y0 && lo_y <= y1) {
        const int slot = atomicAdd(&s_ncand, 1);
        if (slot < kMaxCand) s_cand[slot] = i;
      }
    }
  }
  // 2. dilation of the Inpaint indicator (the rows were dilated horizontally
  //    when they were built; visible since the label barrier)
  // ... and vertical: bit c of s_vrow[y] <=> an Inpaint pixel within
  // Chebyshev distance R of tile pixel (c, y)
  if (threadIdx.x < kTile) {
    unsigned int v = 0;
    for (int dy = 0; dy <= 2 * R; ++dy) v |= s_hrow[threadIdx.x + dy];
    s_vrow[threadIdx.x] = v;
  }
  __syncthreads();

  // 3. four consecutive pixels per thread: row ry, columns c0 .. c0+3.
  //    The cheap per-pixel work (stamps, enter map, activity) runs here; the
  //    Inpaint pixels are queued in shared memory for step 4, so the guide
  //    evaluation (raster, exp, hypot in fp64) runs one pixel per thread over
  //    a dense list instead of four serial, divergent pixels per thread.
  const unsigned int vmask = s_vrow[ry];
  int n_inp = 0;
  unsigned act4 = 0;  // bit u: own pixel u is an active Inpaint pixel
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    const int c = c0 + u;
    const int gx = tx0 + c;
    const bool in = gy < A.H && gx < A.W;
    const int p = gy * A.W + gx;
    const uint8_t l = (uint8_t)(own4 >> (8 * u));
    const bool near = (vmask >> c) & 1u;
    bool active = false;
    const bool inp = in && l == 255;
    if (in) {
      if (l == 0) {
        if (near) {
          float cv[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
          for (int ch = 0; ch < C; ++ch) cv[ch] = (float)px.t[u * C + ch];
          work[p] = make_float4(cv[0], cv[1], cv[2], __int_as_float(kStampReadable));
          if (C > 3) A.c3[(size_t)f * A.HW + p] = cv[3];
        }
      } else if (inp) {
        ++n_inp;
        // a Readable 8-neighbour (the pixel itself is not Readable): the
        // three ext columns c+R-1 .. c+R+1 of the rows above, at and below
        const unsigned long long nb = s_rrow64[ry + R - 1] | s_rrow64[ry + R] | s_rrow64[ry + R + 1];
        active = ((nb >> (c + R - 1)) & 7ull) != 0;
      } else if (near) {
        work[p] = make_float4(0.f, 0.f, 0.f, __int_as_float(kStampBystander));
      }
      if (A.enter) A.enter[(size_t)f * A.HW + p] = active ? 0 : -1;
    }
    act4 |= active ? 1u << u : 0u;
    // queue the Inpaint pixel (warp-aggregated slot)
    const unsigned m = __ballot_sync(0xffffffffu, inp);
    if (m) {
      int base = 0;
      if (lane == __ffs(m) - 1) base = atomicAdd(&s_ninp, __popc(m));
      base = __shfl_sync(0xffffffffu, base, __ffs(m) - 1);
      if (inp) s_inp[base + __popc(m & ((1u << lane) - 1))] = (uint16_t)((ry << 5) | c | (active ? 0x8000 : 0));
    }
  }
  __syncthreads();
  // 4. the guide at every Inpaint pixel of the tile (one per thread), its
  //    unit vector for the rotated ball, the pixel's stamp; the rotated-ball
  //    bit goes back to the owning thread through s_rotb
  {
    const int n_q = s_ninp;
#pragma unroll 1
    for (int k = threadIdx.x; k < n_q; k += kThreads) {
      const unsigned e = s_inp[k];
      const int lx = e & 31, ly = (e >> 5) & 31;
      const bool active = (e & 0x8000u) != 0;
      const int gx = tx0 + lx, gyq = ty0 + ly;
      const int p = gyq * A.W + gx;
      double gxv = 0.0, gyv = 0.0;
      if (raster) {
        const bool exhaustive = s_ncand > kMaxCand;
        const int e0 = (exhaustive && A.frame_seg) ? A.frame_seg[f] : 0;
        const int n_eval = exhaustive ? (A.frame_seg ? A.frame_seg[f + 1] - e0 : A.n_seg) : s_ncand;
        double dmin = INFINITY;
        int nearest = 0x7fffffff;
        const double fx = (double)gx, fy = (double)gyq;
        // a segment whose bounding box lies farther than 3 eta cannot give
        // this pixel a non-zero g (d > cut for it), so its exact distance
        // is skipped; the bound is padded well past rounding, keeping every
        // segment with d <= cut -- the only ones that decide g
        const double cut2 = A.cut * A.cut * (1.0 + 1e-9) + 1e-9;
        for (int cc = 0; cc < n_eval; ++cc) {
          const int sidx = exhaustive ? e0 + cc : s_cand[cc];
          const double4 sg = A.seg[sidx];
          const double bx = fmax(fmax(fmin(sg.x, sg.z) - fx, fx - fmax(sg.x, sg.z)), 0.0);
          const double by = fmax(fmax(fmin(sg.y, sg.w) - fy, fy - fmax(sg.y, sg.w)), 0.0);
          if (bx * bx + by * by > cut2) continue;
          const double d = seg_dist(fx, fy, sg);
          const int sp = A.seg_spline[sidx];
          if (d < dmin || (d == dmin && sp < nearest)) {
            dmin = d;
            nearest = sp;
          }
        }
        if (dmin <= A.cut) {
          const double fall = exp_np((-(dmin * dmin)) / A.c2eta);
          const double2 dir = A.dirs[nearest];
          gxv = dir.x * fall;
          gyv = dir.y * fall;
        }
      } else if (A.g_mode == 2) {
        const double2 g = reinterpret_cast<const double2*>(A.gsrc)[(size_t)f * A.HW + p];
        gxv = g.x;
        gyv = g.y;
      } else if (A.g_mode == 1) {
        gxv = A.gfx;
        gyv = A.gfy;
      }
      const bool rot = (gxv != 0.0 || gyv != 0.0);
      if (rot) {
        atomicOr(&s_rotb[ly], 1u << lx);
        if (active) s_anyg = 1;
      }
      if (A.gbuf) {
        // the unit guide of the rotated ball (engine.py:155-158), once per pixel
        double ux = 0.0, uy = 1.0;
        if (rot) {
          const double nr = hypot_np(gxv, gyv);
          ux = gxv / nr;
          uy = gyv / nr;
        }
        A.gbuf[(size_t)f * A.HW + p] = make_double4(gxv, gyv, ux, uy);
      }
      const int st = (active ? kStampActive : kStampInactive) | (rot ? kRotBit : 0);
      work[p] = make_float4(0.f, 0.f, 0.f, __int_as_float(st));
    }
  }
  __syncthreads();
  const bool anyg = s_anyg != 0;
  uint32_t ent[4];
  {
    const unsigned rotb = s_rotb[ry];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int c = c0 + u;
      const bool rot = (rotb >> c) & 1u;
      // initial frontier entry of this pixel (published per block below)
      ent[u] = ((act4 >> u) & 1u) ? ((uint32_t)(gy * A.W + tx0 + c) | (rot ? kEntryRot : 0u)) : 0xffffffffu;
    }
  }
  // block-aggregated append of the initial frontier (lattice entries to the
  // front of the list, rotated-ball entries to the back when split), |D| and
  // the data-term flag: one barrier gathers the warps' counts, one atomic per
  // quantity per block, one barrier hands out the list bases
  {
    const unsigned lt = (1u << lane) - 1;
    int wL = 0, wR = 0;
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const bool act = ent[u] != 0xffffffffu;
      const bool back = act && (ent[u] & kEntryRot) && A.split;
      wL += __popc(__ballot_sync(0xffffffffu, act && !back));
      wR += __popc(__ballot_sync(0xffffffffu, back));
    }
    const int w_inp = __reduce_add_sync(0xffffffffu, (unsigned)n_inp);
    const bool w_ag = __any_sync(0xffffffffu, anyg);
    if (lane == 0) {
      s_wl[warp] = wL;
      s_wr[warp] = wR;
      s_cnt[warp] = w_inp | (w_ag ? (1 << 30) : 0);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      int tL = 0, tR = 0, tot = 0;
      bool ag = false;
      for (int w = 0; w < kThreads / 32; ++w) {
        const int a = s_wl[w], b = s_wr[w];
        s_wl[w] = tL;
        s_wr[w] = tR;
        tL += a;
        tR += b;
        tot += s_cnt[w] & ((1 << 30) - 1);
        ag |= (s_cnt[w] >> 30) != 0;
      }
      s_bL = tL > 0 ? atomicAdd(&A.cnt[f], tL) : 0;
      s_bR = tR > 0 ? atomicAdd(&A.cntR[f], tR) : 0;
      if (tot) {
        atomicAdd(&A.remaining[f], tot);
        atomicAdd(&A.inpaint[f], tot);
      }
      if (ag) A.anyg[f] = 1;
    }
    __syncthreads();
    int bL = s_bL + s_wl[warp], bR = s_bR + s_wr[warp];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const bool act = ent[u] != 0xffffffffu;
      const bool back = act && (ent[u] & kEntryRot) && A.split;
      const unsigned mL = __ballot_sync(0xffffffffu, act && !back);
      const unsigned mR = __ballot_sync(0xffffffffu, back);
      if (back) A.list0[(size_t)f * A.cap + A.cap - 1 - (bR + __popc(mR & lt))] = ent[u];
      else if (act) A.list0[(size_t)f * A.cap + bL + __popc(mL & lt)] = ent[u];
      bL += __popc(mL);
      bR += __popc(mR);
    }
  }
  timeline_mark(A, 0, false);
}

// ------------------------------------------------------------ TMA helpers
// (raw PTX: mbarrier transaction counts, 3-D bulk tensor copies)
__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return (unsigned)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned phase) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra.uni WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(phase)
      : "memory");
}
__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, int x, int y, int z,
                                            unsigned long long* bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(
          smem_u32(dst)),
      "l"(reinterpret_cast<unsigned long long>(map)), "r"(x), "r"(y), "r"(z), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void tma_store_3d(const CUtensorMap* map, int x, int y, int z, const void* src) {
  asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%1, %2, %3}], [%4];" ::"l"(
                   reinterpret_cast<unsigned long long>(map)),
               "r"(x), "r"(y), "r"(z), "r"(smem_u32(src))
               : "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read0() {
  asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
}

// Prep with TMA (frames whose rows are 16-byte multiples, not periodic): the
// same pass as k_prep, but the pixel tile and the label halo arrive by two
// bulk tensor loads into shared memory and the copy to the output is one
// bulk tensor store -- no per-thread global traffic on the streaming part.
template <typename T, int C>
__global__ void __launch_bounds__(kThreads, GF_PREP_MIN_BLOCKS)
    k_prep_tma(const __grid_constant__ PrepMaps M, const __grid_constant__ FillArgs A) {
  // (the maps come first: a CUtensorMap operand must be 64-byte aligned in
  // the parameter space)
  // grid (tile column, tile row, frame): no division for the tile index
  const int f = blockIdx.z;
  const int tiles_x = gridDim.x;
  const int tix = blockIdx.x, tiy = blockIdx.y;
  const int tile = tiy * tiles_x + tix;
  const int tx0 = tix * kTile;
  const int ty0 = tiy * kTile;
  timeline_mark(A, 0, true);
  PREP_PROF_T0;
  // every prep block is resident once all have passed here: the shell
  // kernel may start launching (it waits for this grid's completion)
  pdl_trigger();
  const int R = A.halo;
  const int ext = kTile + 2 * R;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  // the tile's pixels and its labels with the (r+1) halo, staged by TMA; the
  // pixel tile goes straight back out to the output by a TMA store (the copy
  // of engine.py:289 -- Readable pixels are final)
  __shared__ __align__(128) T s_img[kTile * kTile * C];
  __shared__ __align__(128) uint8_t s_lab[kTileExt * kLabBoxMax];
  __shared__ __align__(8) unsigned long long s_bar;
  __shared__ unsigned int s_hrow[kTileExt];
  __shared__ unsigned int s_vrow[kTile];
  __shared__ unsigned long long s_hrow64[kTileExt];
  __shared__ unsigned long long s_rrow64[kTileExt];
  __shared__ int s_cand[kMaxCand];
  __shared__ int s_ncand;
  __shared__ uint16_t s_inp[kTile * kTile];
  __shared__ unsigned int s_rotb[kTile];
  __shared__ int s_ninp, s_anyg;
  __shared__ int s_cnt[kThreads / 32];
  __shared__ int s_wl[kThreads / 32], s_wr[kThreads / 32];
  __shared__ int s_bL, s_bR;
  __shared__ unsigned long long s_red[4][kThreads / 32];
  if (threadIdx.x == 0) {
    mbar_init(&s_bar, 1);
    fence_mbar_init();
    s_ncand = 0;
    s_ninp = 0;
    s_anyg = 0;
  }
  if (threadIdx.x < kTile) s_rotb[threadIdx.x] = 0u;
  // the frame's hull as last seen (a filter for the hull atomics below: the
  // hull only grows, so a stale value skips no needed update), read while
  // the tile loads
  unsigned long long hull_seen = 0ULL;
  if (threadIdx.x < 4)
    hull_seen = *(volatile unsigned long long*)(threadIdx.x < 2 ? &A.hull[2 * f + threadIdx.x]
                                                                 : &A.bys_frame[2 * f + threadIdx.x - 2]);
  __syncthreads();
  if (threadIdx.x == 0) {
    mbar_expect_tx(&s_bar, (unsigned)(sizeof(T) * kTile * kTile * C + M.lab_bw * ext));
    tma_load_3d(s_img, &M.img, tx0 * C, ty0, f, &s_bar);
    tma_load_3d(s_lab, &M.lab, tx0 - 16, ty0 - R, f, &s_bar);
  }
  const bool raster = A.n_seg > 0;
  const int s0 = A.frame_seg ? A.frame_seg[f] : 0;
  const int s1 = A.frame_seg ? A.frame_seg[f + 1] : A.n_seg;
  // the segments whose cut box meets the tile (tiles that need the guide;
  // culling here, while the tile loads, measured slower)
  auto cull = [&]() {
    const double x0 = (double)tx0, x1 = (double)min(A.W - 1, tx0 + kTile - 1);
    const double y0 = (double)ty0, y1 = (double)min(A.H - 1, ty0 + kTile - 1);
    for (int i = s0 + threadIdx.x; i < s1; i += kThreads) {
      const double4 sg = A.seg[i];
      const double lo_x = fmin(sg.x, sg.z) - A.cut, hi_x = fmax(sg.x, sg.z) + A.cut;
      const double lo_y = fmin(sg.y, sg.w) - A.cut, hi_y = fmax(sg.y, sg.w) + A.cut;
      if (hi_x >= x0 && lo_x <= x1 && hi_y >= y0 && lo_y <= y1) {
        const int slot = atomicAdd(&s_ncand, 1);
        if (slot < kMaxCand) s_cand[slot] = i;
      }
    }
  };
  const uint8_t* lab = A.labels + (size_t)f * A.HW;
  const T* img = reinterpret_cast<const T*>(A.image) + (size_t)f * A.HW * C;
  float4* work = A.work + (size_t)f * A.HW;
  const int ry = threadIdx.x >> 3;
  const int c0 = (threadIdx.x & 7) * 4;
  const int gy = ty0 + ry;

  // 1. Inpaint / Readable bitmasks of the tile + halo rows (bit x <=> ext
  //    column x; out of lattice = neither -- TMA fills those cells with 0,
  //    so the lattice bounds mask them), four threads per ext row, 16 label
  //    bytes each, packed 4 at a time (one multiply per word)
  bool any_inp = false;
  const unsigned long long ext_mask = ext >= 64 ? ~0ULL : ((1ULL << ext) - 1);
  // ext columns inside the lattice
  unsigned long long col_ok = ext_mask;
  if (tx0 - R < 0) col_ok &= ~0ULL << (R - tx0);
  if (tx0 - R + ext > A.W) col_ok &= (A.W - (tx0 - R)) >= 64 ? ~0ULL : ((1ULL << (A.W - (tx0 - R))) - 1);
  mbar_wait(&s_bar, 0);
  PREP_STAGE(1);
  if (threadIdx.x == 0) {
    fence_proxy_async();
    tma_store_3d(&M.out, tx0 * C, ty0, f, s_img);
    bulk_commit();
  }
  {
    const int y = threadIdx.x >> 2, part = threadIdx.x & 3;
    const int gyy = ty0 - R + y;
    unsigned long long im = 0ULL, rm = 0ULL;
    if (y < ext && gyy >= 0 && gyy < A.H) {
      const uint4 q = *reinterpret_cast<const uint4*>(s_lab + y * M.lab_bw + 16 * part);
      const unsigned w[4] = {q.x, q.y, q.z, q.w};
      unsigned ib = 0, rb = 0;
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        ib |= nib4(w[i]) << (4 * i);
        rb |= nib4(~w[i] >> 7) << (4 * i);
      }
      im = (unsigned long long)ib << (16 * part);
      rm = (unsigned long long)rb << (16 * part);
    }
    im |= __shfl_xor_sync(0xffffffffu, im, 1);
    rm |= __shfl_xor_sync(0xffffffffu, rm, 1);
    im |= __shfl_xor_sync(0xffffffffu, im, 2);
    rm |= __shfl_xor_sync(0xffffffffu, rm, 2);
    if (part == 0 && y < ext) {
      // box column 16 - R is ext column 0
      im = (im >> (16 - R)) & col_ok;
      rm = (rm >> (16 - R)) & col_ok;
      s_hrow64[y] = im;
      s_rrow64[y] = rm;
      s_hrow[y] = hdilate(im, R);
      any_inp = im != 0ULL;
    }
  }
  // labels of the thread's own 4 pixels (byte u = column c0 + u)
  uint32_t own4 = 0x80808080u;
  if (gy < A.H) {
    const uint8_t* lr = s_lab + (ry + R) * M.lab_bw + 16 + c0;
#pragma unroll
    for (int u = 0; u < 4; ++u)
      if (tx0 + c0 + u < A.W) own4 = (own4 & ~(0xffu << (8 * u))) | ((uint32_t)lr[u] << (8 * u));
  }
  // the thread's 4 pixels, from the staged tile
  const int gx0 = tx0 + c0;
  constexpr int nv = (4 * C * (int)sizeof(T)) / 16;
  constexpr bool vec_ok = (4 * C * (int)sizeof(T)) % 16 == 0;
  const bool row_in = gy < A.H;
  union {
    T t[4 * C];
    uint4 q[nv > 0 ? nv : 1];
  } px;
  {
    const T* src = s_img + (size_t)ry * kTile * C + c0 * C;
    if constexpr (vec_ok) {
#pragma unroll
      for (int i = 0; i < nv; ++i) px.q[i] = reinterpret_cast<const uint4*>(src)[i];
    } else {
#pragma unroll
      for (int i = 0; i < 4 * C; ++i) px.t[i] = src[i];
    }
  }
  // label validation (grid.py:36-46) rides on the own-pixel load: any byte
  // outside {0, 128, 255} flags the frame
  {
    const unsigned bad = ~(__vcmpeq4(own4, 0u) | __vcmpeq4(own4, 0x80808080u) |
                           __vcmpeq4(own4, 0xffffffffu));
    if (bad && gy < A.H) {
      unsigned valid = 0;  // bytes of in-lattice columns
#pragma unroll
      for (int u = 0; u < 4; ++u)
        if (tx0 + c0 + u < A.W) valid |= 0xffu << (8 * u);
      if (bad & valid) A.badlab[f] = 1;
    }
  }
  const bool tile_d = __syncthreads_or(any_inp);
  PREP_STAGE(2);
  // value hull of the Readable pixels (the copy is the TMA store above)
  {
    // [0] value hull of the Readable pixels, [1] range of the Bystanders
    // per pixel: channel min / max, then merged into its class (branch-free)
    T vlo[2] = {T(INFINITY), T(INFINITY)}, vhi[2] = {T(-INFINITY), T(-INFINITY)};
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const uint8_t l = (uint8_t)(own4 >> (8 * u));
      T mn = px.t[u * C], mx = px.t[u * C];
#pragma unroll
      for (int ch = 1; ch < C; ++ch) {
        mn = fmin(mn, px.t[u * C + ch]);
        mx = fmax(mx, px.t[u * C + ch]);
      }
      const bool in = row_in && gx0 + u < A.W;
      const bool rd = in && l == 0, by = in && l == 128;
      vlo[0] = rd ? fmin(vlo[0], mn) : vlo[0];
      vhi[0] = rd ? fmax(vhi[0], mx) : vhi[0];
      vlo[1] = by ? fmin(vlo[1], mn) : vlo[1];
      vhi[1] = by ? fmax(vhi[1], mx) : vhi[1];
    }
    unsigned long long ered[4];  // max(~enc) <=> min(enc)
    if constexpr (sizeof(T) == 4) {
      // fp32 values: order-preserving 32-bit codes, one redux per quantity
      unsigned m[4];
#pragma unroll
      for (int b = 0; b < 2; ++b) {
        const bool any = vlo[b] <= vhi[b];
        m[2 * b] = __reduce_max_sync(0xffffffffu, any ? ~enc32((float)vlo[b]) : 0u);
        m[2 * b + 1] = __reduce_max_sync(0xffffffffu, any ? enc32((float)vhi[b]) : 0u);
      }
      // the block reduces the 32-bit codes; the fp64 codes are made once
      // per block below
#pragma unroll
      for (int i = 0; i < 4; ++i) ered[i] = m[i];
    } else {
#pragma unroll
      for (int b = 0; b < 2; ++b) {
        ered[2 * b] = vlo[b] <= vhi[b] ? ~enc_ordered((double)vlo[b]) : 0ULL;
        ered[2 * b + 1] = vlo[b] <= vhi[b] ? enc_ordered((double)vhi[b]) : 0ULL;
      }
#pragma unroll
      for (int i = 0; i < 4; ++i)
        for (int o = 16; o > 0; o >>= 1) {
          const unsigned long long a = __shfl_xor_sync(0xffffffffu, ered[i], o);
          ered[i] = a > ered[i] ? a : ered[i];
        }
    }
#pragma unroll
    for (int i = 0; i < 4; ++i)
      if (lane == 0) s_red[i][warp] = ered[i];
    if (A.fillshell && row_in) {
      int* fsh = A.fillshell + (size_t)f * A.HW + (size_t)gy * A.W + gx0;
#pragma unroll
      for (int u = 0; u < 4; ++u)
        if (gx0 + u < A.W) fsh[u] = -1;
    }
    __syncthreads();
    if (threadIdx.x < 4) {
      const int i = threadIdx.x;
      unsigned long long e = 0ULL;
      for (int w = 0; w < kThreads / 32; ++w) e = s_red[i][w] > e ? s_red[i][w] : e;
      if constexpr (sizeof(T) == 4) {
        // 32-bit order codes of fp32 values -> the fp64 codes of the hull
        const unsigned m = (unsigned)e;
        e = (i & 1) ? (m ? enc_ordered((double)dec32(m)) : 0ULL)
                    : (m ? ~enc_ordered((double)dec32(~m)) : 0ULL);
      }
      // i < 2: the frame's hull (most tiles cannot move it any more: skip
      // their atomics); i >= 2: the tile's Bystander range, read by the
      // shell loop's clip, and the frame's
      unsigned long long* fr = i < 2 ? &A.hull[2 * f + i] : &A.bys_frame[2 * f + i - 2];
      if (e != 0ULL && e > hull_seen) atomicMax(fr, e);
      if (i >= 2) A.bys[((size_t)f * A.ntiles + tile) * 2 + i - 2] = e;
    }
  }
  PREP_STAGE(3);
  if (!tile_d) {
    // no Inpaint pixel within reach: nothing of this tile is ever sampled
    if (A.enter && row_in) {
      int* en = A.enter + (size_t)f * A.HW + (size_t)gy * A.W + gx0;
#pragma unroll
      for (int u = 0; u < 4; ++u)
        if (gx0 + u < A.W) en[u] = -1;
    }
    timeline_mark(A, 0, false);
    if (threadIdx.x == 0) bulk_wait_read0();
    PREP_PROF(0);
    return;
  }
  if (raster) cull();
  // 2. dilation of the Inpaint indicator (the rows were dilated horizontally
  //    when they were built; visible since the label barrier)
  // ... and vertical: bit c of s_vrow[y] <=> an Inpaint pixel within
  // Chebyshev distance R of tile pixel (c, y)
  if (threadIdx.x < kTile) {
    unsigned int v = 0;
    for (int dy = 0; dy <= 2 * R; ++dy) v |= s_hrow[threadIdx.x + dy];
    s_vrow[threadIdx.x] = v;
  }
  __syncthreads();

  PREP_STAGE(4);
  // 3. four consecutive pixels per thread: row ry, columns c0 .. c0+3.
  //    The cheap per-pixel work (stamps, enter map, activity) runs here; the
  //    Inpaint pixels are queued in shared memory for step 4, so the guide
  //    evaluation (raster, exp, hypot in fp64) runs one pixel per thread over
  //    a dense list instead of four serial, divergent pixels per thread.
  const unsigned int vmask = s_vrow[ry];
  int n_inp = 0;
  unsigned act4 = 0;  // bit u: own pixel u is an active Inpaint pixel
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    const int c = c0 + u;
    const int gx = tx0 + c;
    const bool in = gy < A.H && gx < A.W;
    const int p = gy * A.W + gx;
    const uint8_t l = (uint8_t)(own4 >> (8 * u));
    const bool near = (vmask >> c) & 1u;
    bool active = false;
    const bool inp = in && l == 255;
    if (in) {
      if (l == 0) {
        if (near) {
          float cv[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
          for (int ch = 0; ch < C; ++ch) cv[ch] = (float)px.t[u * C + ch];
          work[p] = make_float4(cv[0], cv[1], cv[2], __int_as_float(kStampReadable));
          if (C > 3) A.c3[(size_t)f * A.HW + p] = cv[3];
        }
      } else if (inp) {
        ++n_inp;
        // a Readable 8-neighbour (the pixel itself is not Readable): the
        // three ext columns c+R-1 .. c+R+1 of the rows above, at and below
        const unsigned long long nb = s_rrow64[ry + R - 1] | s_rrow64[ry + R] | s_rrow64[ry + R + 1];
        active = ((nb >> (c + R - 1)) & 7ull) != 0;
      } else if (near) {
        work[p] = make_float4(0.f, 0.f, 0.f, __int_as_float(kStampBystander));
      }
      if (A.enter) A.enter[(size_t)f * A.HW + p] = active ? 0 : -1;
    }
    act4 |= active ? 1u << u : 0u;
    // queue the Inpaint pixel (warp-aggregated slot)
    const unsigned m = __ballot_sync(0xffffffffu, inp);
    if (m) {
      int base = 0;
      if (lane == __ffs(m) - 1) base = atomicAdd(&s_ninp, __popc(m));
      base = __shfl_sync(0xffffffffu, base, __ffs(m) - 1);
      if (inp) s_inp[base + __popc(m & ((1u << lane) - 1))] = (uint16_t)((ry << 5) | c | (active ? 0x8000 : 0));
    }
  }
  __syncthreads();
  PREP_STAGE(5);
  // 4. the guide at every Inpaint pixel of the tile (one per thread), its
  //    unit vector for the rotated ball, the pixel's stamp; the rotated-ball
  //    bit goes back to the owning thread through s_rotb
  {
    const int n_q = s_ninp;
#pragma unroll 1
    for (int k = threadIdx.x; k < n_q; k += kThreads) {
      const unsigned e = s_inp[k];
      const int lx = e & 31, ly = (e >> 5) & 31;
      const bool active = (e & 0x8000u) != 0;
      const int gx = tx0 + lx, gyq = ty0 + ly;
      const int p = gyq * A.W + gx;
      double gxv = 0.0, gyv = 0.0;
      if (raster) {
        const bool exhaustive = s_ncand > kMaxCand;
        const int e0 = (exhaustive && A.frame_seg) ? A.frame_seg[f] : 0;
        const int n_eval = exhaustive ? (A.frame_seg ? A.frame_seg[f + 1] - e0 : A.n_seg) : s_ncand;
        double dmin = INFINITY;
        int nearest = 0x7fffffff;
        const double fx = (double)gx, fy = (double)gyq;
        // a segment whose bounding box lies farther than 3 eta cannot give
        // this pixel a non-zero g (d > cut for it), so its exact distance
        // is skipped; the bound is padded well past rounding, keeping every
        // segment with d <= cut -- the only ones that decide g
        const double cut2 = A.cut * A.cut * (1.0 + 1e-9) + 1e-9;
        for (int cc = 0; cc < n_eval; ++cc) {
          const int sidx = exhaustive ? e0 + cc : s_cand[cc];
          const double4 sg = A.seg[sidx];
          const double bx = fmax(fmax(fmin(sg.x, sg.z) - fx, fx - fmax(sg.x, sg.z)), 0.0);
          const double by = fmax(fmax(fmin(sg.y, sg.w) - fy, fy - fmax(sg.y, sg.w)), 0.0);
          if (bx * bx + by * by > cut2) continue;
          const double d = seg_dist(fx, fy, sg);
          const int sp = A.seg_spline[sidx];
          if (d < dmin || (d == dmin && sp < nearest)) {
            dmin = d;
            nearest = sp;
          }
        }
        if (dmin <= A.cut) {
          const double fall = exp_np((-(dmin * dmin)) / A.c2eta);
          const double2 dir = A.dirs[nearest];
          gxv = dir.x * fall;
          gyv = dir.y * fall;
        }
      } else if (A.g_mode == 2) {
        const double2 g = reinterpret_cast<const double2*>(A.gsrc)[(size_t)f * A.HW + p];
        gxv = g.x;
        gyv = g.y;
      } else if (A.g_mode == 1) {
        gxv = A.gfx;
        gyv = A.gfy;
      }
      const bool rot = (gxv != 0.0 || gyv != 0.0);
      if (rot) {
        atomicOr(&s_rotb[ly], 1u << lx);
        if (active) s_anyg = 1;
      }
      if (A.gbuf) {
        // the unit guide of the rotated ball (engine.py:155-158), once per pixel
        double ux = 0.0, uy = 1.0;
        if (rot) {
          const double nr = hypot_np(gxv, gyv);
          ux = gxv / nr;
          uy = gyv / nr;
        }
        A.gbuf[(size_t)f * A.HW + p] = make_double4(gxv, gyv, ux, uy);
      }
      const int st = (active ? kStampActive : kStampInactive) | (rot ? kRotBit : 0);
      work[p] = make_float4(0.f, 0.f, 0.f, __int_as_float(st));
    }
  }
  __syncthreads();
  PREP_STAGE(6);
  const bool anyg = s_anyg != 0;
  uint32_t ent[4];
  {
    const unsigned rotb = s_rotb[ry];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int c = c0 + u;
      const bool rot = (rotb >> c) & 1u;
      // initial frontier entry of this pixel (published per block below)
      ent[u] = ((act4 >> u) & 1u) ? ((uint32_t)(gy * A.W + tx0 + c) | (rot ? kEntryRot : 0u)) : 0xffffffffu;
    }
  }
  // block-aggregated append of the initial frontier (lattice entries to the
  // front of the list, rotated-ball entries to the back when split), |D| and
  // the data-term flag: one barrier gathers the warps' counts, one atomic per
  // quantity per block, one barrier hands out the list bases
  {
    const unsigned lt = (1u << lane) - 1;
    int wL = 0, wR = 0;
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const bool act = ent[u] != 0xffffffffu;
      const bool back = act && (ent[u] & kEntryRot) && A.split;
      wL += __popc(__ballot_sync(0xffffffffu, act && !back));
      wR += __popc(__ballot_sync(0xffffffffu, back));
    }
    const int w_inp = __reduce_add_sync(0xffffffffu, (unsigned)n_inp);
    const bool w_ag = __any_sync(0xffffffffu, anyg);
    if (lane == 0) {
      s_wl[warp] = wL;
      s_wr[warp] = wR;
      s_cnt[warp] = w_inp | (w_ag ? (1 << 30) : 0);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      int tL = 0, tR = 0, tot = 0;
      bool ag = false;
      for (int w = 0; w < kThreads / 32; ++w) {
        const int a = s_wl[w], b = s_wr[w];
        s_wl[w] = tL;
        s_wr[w] = tR;
        tL += a;
        tR += b;
        tot += s_cnt[w] & ((1 << 30) - 1);
        ag |= (s_cnt[w] >> 30) != 0;
      }
      s_bL = tL > 0 ? atomicAdd(&A.cnt[f], tL) : 0;
      s_bR = tR > 0 ? atomicAdd(&A.cntR[f], tR) : 0;
      if (tot) {
        atomicAdd(&A.remaining[f], tot);
        atomicAdd(&A.inpaint[f], tot);
      }
      if (ag) A.anyg[f] = 1;
    }
    PREP_STAGE(7);
    __syncthreads();
    PREP_STAGE(8);
    int bL = s_bL + s_wl[warp], bR = s_bR + s_wr[warp];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const bool act = ent[u] != 0xffffffffu;
      const bool back = act && (ent[u] & kEntryRot) && A.split;
      const unsigned mL = __ballot_sync(0xffffffffu, act && !back);
      const unsigned mR = __ballot_sync(0xffffffffu, back);
      if (back) A.list0[(size_t)f * A.cap + A.cap - 1 - (bR + __popc(mR & lt))] = ent[u];
      else if (act) A.list0[(size_t)f * A.cap + bL + __popc(mL & lt)] = ent[u];
      bL += __popc(mL);
      bR += __popc(mR);
    }
  }
  timeline_mark(A, 0, false);
  if (threadIdx.x == 0) bulk_wait_read0();
  PREP_PROF(1u | ((unsigned)s_ncand << 1));
}


// ------------------------------------------------------- shell loop
//
// Frontier lists.  Each frame owns a list buffer of `cap` entries used from
// both ends: lattice entries (g = 0, 8-lane sampler) grow from the front,
// rotated-ball entries (g != 0, warp-per-item sampler) grow from the back,
// with separate counters cnt / cntR.  An entry is pixel | kEntryRot.  The
// per-frame item index j runs over [0, nL) for the front part and
// [nL, nL + nR) for the back part (conf[] and the guard use it).

struct GridTables {
  int pref[kMaxFramesPerLaunch + 1];   // all items
  int prefL[kMaxFramesPerLaunch + 1];  // lattice part
  int prefR[kMaxFramesPerLaunch + 1];  // rotated part
  int nLf[kMaxFramesPerLaunch];  // frame's lattice / rotated items (0 if inactive)
  int nRf[kMaxFramesPerLaunch];
  uint32_t app[kAppendCap];
};

struct Smem {
  BallTables tab;
  struct {
    GridTables g;
  } u;
  int g_one, g_f;  // guard of a single small stalled frame by block 0
  unsigned char act[kMaxFramesPerLaunch];
  unsigned char dl[kMaxFramesPerLaunch];
  int red[kShellThreads / 32];
  unsigned long long redk[kShellThreads / 32];
  int any_dl, any_clip;
  int total, totalL, totalR;
  // block-level flush of the warps' staged appends
  int bf_frame[kShellThreads / 32], bf_nL[kShellThreads / 32], bf_nR[kShellThreads / 32];
  int bf_fill[kShellThreads / 32], bf_anyg[kShellThreads / 32], bf_bL[kShellThreads / 32], bf_bR[kShellThreads / 32];
};

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// per-shell phase timestamps (profiling only, A.trace may be null)
constexpr int kTraceSlots = 8;
__device__ __forceinline__ void trace_max_val(const FillArgs& A, int k, int slot,
                                              unsigned long long v) {
  if (A.trace && k < A.trace_cap) atomicMax(&A.trace[k * kTraceSlots + slot], v);
}
__device__ __forceinline__ void trace_set(const FillArgs& A, int k, int slot, unsigned long long v) {
  if (A.trace && k < A.trace_cap && blockIdx.x == 0 && threadIdx.x == 0)
    A.trace[k * kTraceSlots + slot] = v;
}
__device__ __forceinline__ void trace_max(const FillArgs& A, int k, int slot) {
  if (A.trace && k < A.trace_cap && threadIdx.x == 0)
    atomicMax(&A.trace[k * kTraceSlots + slot], gtimer());
}

// Fine phase trace (experiment builds only, -DGF_FINE_TRACE): per-shell
// maxima of the phases of one work unit in trace row 128 + k; slots 0-3
// lattice units (entry load, eval, decide, activate), 4-7 rotated units.
#ifdef GF_FINE_TRACE
__device__ __forceinline__ unsigned long long fine_after(unsigned v) {
  if (v == 0xfffffffeu) asm volatile("trap;");
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ void fine_put(const FillArgs& A, int k, int slot, unsigned long long d) {
  if (A.trace && 128 + k < A.trace_cap - 1) atomicMax(&A.trace[(128 + k) * kTraceSlots + slot], d);
}
__device__ __forceinline__ void fine_add(const FillArgs& A, int k, int slot, unsigned long long d) {
  if (A.trace && 128 + k < A.trace_cap - 1) atomicAdd(&A.trace[(128 + k) * kTraceSlots + slot], d);
}
#define GF_FINE(x) x
#else
#define GF_FINE(x)
#endif

// largest f with pref[f] <= t
__device__ __forceinline__ int find_frame(const int* pref, int nF, int t) {
  int lo = 0, hi = nF - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (pref[mid] <= t) lo = mid; else hi = mid - 1;
  }
  return lo;
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
  for (int w = 0; w < kShellThreads / 32; ++w) t = S.redk[w] > t ? S.redk[w] : t;
  return t;
}

__device__ __forceinline__ unsigned long long conf_key(double c) {
  // numpy argmax: NaN is maximal; confidences are >= +0 otherwise
  return (c != c) ? ~0ULL : (unsigned long long)__double_as_longlong(c);
}

__device__ __forceinline__ void frame_guide(const FillArgs& A, int f, int p, double& gx,
                                            double& gy) {
  if (A.gbuf) {
    const double4 g = A.gbuf[(size_t)f * A.HW + p];
    gx = g.x;
    gy = g.y;
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

// Data-term latch (engine.py:327-329) as of shell k: released once some
// earlier frontier held no g != 0 pixel.  dt_dead covers the shells block 0
// has booked (it may lag one shell behind), the previous frontier's own flag
// the rest, so every block sees the same answer.
__device__ __forceinline__ bool frontier_has_g(const FillArgs& A, int which, int f);
__device__ __forceinline__ bool dt_dead_at(const FillArgs& A, int f, int k, int prv) {
  return A.dt_dead[f] != 0 || (k > 0 && !frontier_has_g(A, prv, f));
}

__device__ __forceinline__ int frontier_size(const FillArgs& A, int which, int f) {
  return A.cnt[which * A.nF + f] + A.cntR[which * A.nF + f];
}

// entry j of frame f's list (front part first, then the back part)
__device__ __forceinline__ uint32_t entry_at(const uint32_t* list, const FillArgs& A, int f, int j,
                                             int nL) {
  const uint32_t* l = list + (size_t)f * A.cap;
  return j < nL ? l[j] : l[A.cap - 1 - (j - nL)];
}

__device__ __forceinline__ bool entry_back(const FillArgs& A, uint32_t e) {
  return A.split && (e & kEntryRot) != 0;
}

// one entry straight into the global list (rare paths)
__device__ __forceinline__ void append_direct(const FillArgs& A, uint32_t* list, int nxt, int f,
                                              uint32_t e) {
  if (entry_back(A, e)) {
    const int r = atomicAdd(&A.cntR[nxt * A.nF + f], 1);
    list[(size_t)f * A.cap + A.cap - 1 - r] = e;
  } else {
    list[(size_t)f * A.cap + atomicAdd(&A.cnt[nxt * A.nF + f], 1)] = e;
  }
  if (A.order == 2 && A.g_mode == 2 && (e & kEntryRot)) A.anyg[nxt * A.nF + f] = 1;
}

// Warp-private append staging: each warp owns a slice of S.u.g.app and a
// warp-uniform count; a slice is published with one atomic per list part.
constexpr int kWarpAppCap = kAppendCap / (kShellThreads / 32);

__device__ __forceinline__ void warp_push(uint32_t* reg, int& n, bool want, uint32_t e) {
  const unsigned m = __ballot_sync(0xffffffffu, want);
  const int lane = threadIdx.x & 31;
  if (want) reg[n + __popc(m & ((1u << lane) - 1))] = e;
  n += __popc(m);
}

// staged entries of one warp: how many go to the back part, any g != 0
__device__ __forceinline__ void warp_count(const FillArgs& A, const uint32_t* reg, int n, int& nR,
                                           bool& anyg) {
  const int lane = threadIdx.x & 31;
  nR = 0;
  anyg = false;
  for (int c0 = 0; c0 < n; c0 += 32) {
    const bool in = c0 + lane < n;
    const uint32_t e = in ? reg[c0 + lane] : 0u;
    nR += __popc(__ballot_sync(0xffffffffu, in && entry_back(A, e)));
    anyg |= in && (e & kEntryRot) != 0;
  }
  anyg = __any_sync(0xffffffffu, anyg);
}

// copy staged entries to frame f's next list at reserved bases bL / bR
__device__ __forceinline__ void warp_copy(const FillArgs& A, const uint32_t* reg, int n, int f,
                                          uint32_t* nxt_list, int bL, int bR) {
  const int lane = threadIdx.x & 31;
  const unsigned lt = (1u << lane) - 1;
  uint32_t* l = nxt_list + (size_t)f * A.cap;
  for (int c0 = 0; c0 < n; c0 += 32) {
    const bool in = c0 + lane < n;
    const uint32_t e = in ? reg[c0 + lane] : 0u;
    const bool back = in && entry_back(A, e);
    const unsigned mR = __ballot_sync(0xffffffffu, back);
    const unsigned mL = __ballot_sync(0xffffffffu, in && !back);
    if (back) l[A.cap - 1 - (bR + __popc(mR & lt))] = e;
    else if (in) l[bL + __popc(mL & lt)] = e;
    bR += __popc(mR);
    bL += __popc(mL);
  }
}

// warp-level publish (frame switches, full staging slices -- rare)
__device__ __forceinline__ void warp_flush(const FillArgs& A, uint32_t* reg, int& n, int f,
                                           uint32_t* nxt_list, int nxt) {
  if (n == 0) return;
  __syncwarp();
  const int lane = threadIdx.x & 31;
  int nR;
  bool anyg;
  warp_count(A, reg, n, nR, anyg);
  int bL = 0, bR = 0;
  if (lane == 0) {
    if (n - nR > 0) bL = atomicAdd(&A.cnt[nxt * A.nF + f], n - nR);
    if (nR > 0) bR = atomicAdd(&A.cntR[nxt * A.nF + f], nR);
    if (A.order == 2 && A.g_mode == 2 && anyg) A.anyg[nxt * A.nF + f] = 1;
  }
  bL = __shfl_sync(0xffffffffu, bL, 0);
  bR = __shfl_sync(0xffffffffu, bR, 0);
  warp_copy(A, reg, n, f, nxt_list, bL, bR);
  __syncwarp();
  n = 0;
}

// Output of a filled pixel: its fp32 fill value clipped to the frame's value
// hull of the initially Readable values (engine.py:372-375), stored in the
// caller's dtype.
__device__ __forceinline__ void write_out(const FillArgs& A, int f, uint32_t p, const float* v,
                                          unsigned long long hl, unsigned long long hh) {
  const unsigned long long elo = ~hl, ehi = hh;
  const bool has_hull = ehi != 0ULL;
  const double lo = has_hull ? dec_ordered(elo) : 0.0;
  const double hi = has_hull ? dec_ordered(ehi) : 0.0;
  const size_t o = ((size_t)f * A.HW + p) * A.C;
#pragma unroll
  for (int c = 0; c < 4; ++c) {  // compile-time indices: v stays in registers
    if (c >= A.C) break;
    double x = (double)v[c];
    if (has_hull) x = (x < lo) ? lo : ((x > hi) ? hi : x);
    if (A.dtype == GF_F64) reinterpret_cast<double*>(A.out)[o + c] = x;
    else reinterpret_cast<float*>(A.out)[o + c] = (float)x;
  }
}

// Bystander clip (engine.py:372-375), one 32x32 tile per warp.  k_prep
// recorded each tile's Bystander value range: a tile whose range lies in
// the frame's hull is already final (the clip is the identity), so only
// tiles holding out-of-hull Bystanders are touched.  Tiles are handed out by
// an atomic counter to every warp after the last shell (doing them in a
// shell's idle warps could stretch that shell: a tile is several memory
// round trips).
__device__ __forceinline__ bool range_inside(const FillArgs& A, int f, const unsigned long long* r) {
  const unsigned long long hl = A.hull[2 * f], hh = A.hull[2 * f + 1];
  if (hh == 0ULL || r[1] == 0ULL) return true;  // no hull (no clip) or no Bystander
  return r[0] <= hl && r[1] <= hh;              // ~enc(min) <= ~enc(lo), enc(max) <= enc(hi)
}

template <typename T>
__device__ __forceinline__ void clip_tile_rows(const FillArgs& A, int f, int tx0, int ty0, double lo,
                                               double hi) {
  // lane = column; the tile's 32 label bytes of this column are loaded at
  // once, then the Bystanders' values in two batches of 16 rows, so a tile
  // costs a few memory round trips, not one per row
  const int lane = threadIdx.x & 31;
  const int x = tx0 + lane;
  if (x >= A.W) return;
  const uint8_t* lab = A.labels + (size_t)f * A.HW;
  const T* in = reinterpret_cast<const T*>(A.image) + (size_t)f * A.HW * A.C;
  T* out = reinterpret_cast<T*>(A.out) + (size_t)f * A.HW * A.C;
  const int rows = min(kTile, A.H - ty0);
  unsigned bys = 0;  // bit y: row ty0 + y of this column is a Bystander
#pragma unroll
  for (int y = 0; y < kTile; ++y)
    if (y < rows && lab[(size_t)(ty0 + y) * A.W + x] == 128) bys |= 1u << y;
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    T v[16][4];
#pragma unroll
    for (int y = 0; y < 16; ++y)
      if ((bys >> (16 * h + y)) & 1u) {
        const size_t g = ((size_t)(ty0 + 16 * h + y) * A.W + x) * A.C;
#pragma unroll
        for (int c = 0; c < 4; ++c)
          if (c < A.C) v[y][c] = in[g + c];
      }
#pragma unroll
    for (int y = 0; y < 16; ++y)
      if ((bys >> (16 * h + y)) & 1u) {
        const size_t g = ((size_t)(ty0 + 16 * h + y) * A.W + x) * A.C;
#pragma unroll
        for (int c = 0; c < 4; ++c)
          if (c < A.C) {
            double val = (double)v[y][c];
            val = (val < lo) ? lo : ((val > hi) ? hi : val);
            out[g + c] = (T)val;
          }
      }
  }
}

__device__ __noinline__ void clip_tile(const FillArgs& A, int chunk) {
  const int f = chunk / A.ntiles, t = chunk - f * A.ntiles;
  const unsigned long long* r = A.bys + ((size_t)f * A.ntiles + t) * 2;
  if (range_inside(A, f, r)) return;
  const double lo = dec_ordered(~A.hull[2 * f]), hi = dec_ordered(A.hull[2 * f + 1]);
  const int tiles_x = (A.W + kTile - 1) / kTile;
  const int tx0 = (t % tiles_x) * kTile, ty0 = (t / tiles_x) * kTile;
  if (A.dtype == GF_F64) clip_tile_rows<double>(A, f, tx0, ty0, lo, hi);
  else clip_tile_rows<float>(A, f, tx0, ty0, lo, hi);
}

// one tile for the calling warp; false once every tile is taken
__device__ __forceinline__ bool clip_claim(const FillArgs& A) {
  int c = A.clip_total;
  if ((threadIdx.x & 31) == 0 && *(volatile int*)A.clip_next < A.clip_total) c = atomicAdd(A.clip_next, 1);
  c = __shfl_sync(0xffffffffu, c, 0);
  if (c >= A.clip_total) return false;
  clip_tile(A, c);
  return true;
}

// ready / fill decision of one item (engine.py:317-333) and the in-place
// write of its colour with the shell stamp (snapshot-safe: stamp k+1 is
// unreadable for every other item of shell k).
// hl / hh: the frame's encoded hull, loaded by the caller when the unit
// starts so the output store never waits on it (in-order issue would stall
// the group's shuffle behind that load).
__device__ __forceinline__ bool decide_and_write(const FillArgs& A, int f, int j, uint32_t p, int k,
                                                 bool dt_eff, double gx, double gy,
                                                 const SampleResult& r, unsigned long long hl,
                                                 unsigned long long hh) {
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
  // the guard only reads confidences of frames where no item filled, and
  // fills its pick with the value sampled here (no second evaluation)
  if (!fill) {
    A.conf[(size_t)f * A.cap + j] = conf;
    if (r.rw > 0.0)
      A.gval[(size_t)f * A.HW + p] =
          make_float4((float)r.v[0], (float)r.v[1], (float)r.v[2], (float)r.v[3]);
  }
  if (fill) {
    float4 o;
    o.x = (float)r.v[0];
    o.y = (float)r.v[1];
    o.z = (float)r.v[2];
    o.w = __int_as_float(k + 1);
    A.work[(size_t)f * A.HW + p] = o;
    const float v[4] = {o.x, o.y, o.z, (float)r.v[3]};
    if (A.c3) A.c3[(size_t)f * A.HW + p] = v[3];
    write_out(A, f, p, v, hl, hh);
    if (A.fillshell) A.fillshell[(size_t)f * A.HW + p] = k;
  }
  return fill;
}

// 8-neighbour o (grid.py:29-33 order) of pixel (pi, pj)
__device__ __forceinline__ int neighbor_at(const FillArgs& A, int pi, int pj, int o, bool& in) {
  // NEIGHBOR_OFFSETS (grid.py:29-33) packed as 2-bit (d + 1) fields: no branches
  const int di = (int)((0x9224u >> (2 * o)) & 3u) - 1;
  const int dj = (int)((0xA940u >> (2 * o)) & 3u) - 1;
  int ii = pi + di;
  const int jj = pj + dj;
  if (A.periodic) ii = ii < 0 ? ii + A.W : (ii >= A.W ? ii - A.W : ii);
  in = ii >= 0 && ii < A.W && jj >= 0 && jj < A.H;
  return in ? jj * A.W + ii : 0;
}

__device__ __forceinline__ int neighbor_of(const FillArgs& A, uint32_t p, int o, bool& in) {
  int i, j;
  col_row(A, (int)p, i, j);
  return neighbor_at(A, i, j, o, in);
}

// Claim Inpaint neighbour q for the next frontier: INACTIVE -> ACTIVE (the
// dedup of tracker.py:78).  One CAS in the common case, a second only when q
// is an inactive rotated-ball pixel.  Returns the list entry or ~0u.
__device__ __forceinline__ uint32_t claim(float4* fw, int q) {
  int* sp = stamp_ptr(fw, q);
  const int old = atomicCAS(sp, kStampInactive, kStampActive);
  if (old == kStampInactive) return (uint32_t)q;
  if (old == (kStampInactive | kRotBit) &&
      atomicCAS(sp, kStampInactive | kRotBit, kStampActive | kRotBit) == (kStampInactive | kRotBit))
    return (uint32_t)q | kEntryRot;
  return 0xffffffffu;
}

// Tracked frontier maintenance fused into the fill (tracker.py:42-79): an
// unfilled item re-enters the next list (entry e, flag kept), a filled
// item's Inpaint 8-neighbours join it.  Lane gl (0..LG-1, -1 = idle) of the
// item's group handles neighbours gl, gl + LG, ...  `staged`: warp-uniform;
// false -> direct global appends (the items of this warp-round belong to
// different frames).  Every lane calls.
template <int LG>
__device__ __forceinline__ void activate(const FillArgs& A, uint32_t* reg, int& n, bool staged,
                                         uint32_t* nxt_list, int nxt, float4* fw, int f, int k,
                                         int gl, bool filled, uint32_t e, unsigned cand, int pi,
                                         int pj) {
  constexpr int NPL = 8 / LG;  // neighbours per lane
  const bool survive = gl == 0 && !filled;
  uint32_t qe[NPL];
#pragma unroll
  for (int r = 0; r < NPL; ++r) {
    qe[r] = 0xffffffffu;
    // cand: the neighbours that can still be claimed (the others are
    // Readable, Bystander, filled or already in a frontier: no CAS needed)
    if (gl >= 0 && filled && ((cand >> (gl + LG * r)) & 1u)) {
      bool in;
      const int q = neighbor_at(A, pi, pj, gl + LG * r, in);
      if (in) {
        qe[r] = claim(fw, q);
        if (qe[r] != 0xffffffffu && A.enter) A.enter[(size_t)f * A.HW + q] = k + 1;
      }
    }
  }
  if (staged) {
    warp_push(reg, n, survive, e);
#pragma unroll
    for (int r = 0; r < NPL; ++r) warp_push(reg, n, qe[r] != 0xffffffffu, qe[r]);
  } else {
    if (survive) append_direct(A, nxt_list, nxt, f, e);
#pragma unroll
    for (int r = 0; r < NPL; ++r)
      if (qe[r] != 0xffffffffu) append_direct(A, nxt_list, nxt, f, qe[r]);
  }
}

// End of the fill phase: every warp's pending appends and fill count are
// published with one atomic per list part and per frame for the whole block
// (same-address atomics from every warp of the grid would serialise in L2).
// All threads of the block call.
__device__ void block_flush(const FillArgs& A, Smem& S, const uint32_t* reg, int wn, int wf,
                            int wfills, uint32_t* nxt_list, int nxt, int cur, bool tracked) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int nR = 0;
  bool anyg = false;
  if (tracked) warp_count(A, reg, wn, nR, anyg);
  if (lane == 0) {
    S.bf_frame[warp] = wf;
    S.bf_nL[warp] = tracked ? wn - nR : 0;
    S.bf_nR[warp] = nR;
    S.bf_fill[warp] = wfills;
    S.bf_anyg[warp] = anyg ? 1 : 0;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    constexpr int NW = kShellThreads / 32;
    bool done[NW];
    for (int w = 0; w < NW; ++w) done[w] = S.bf_frame[w] < 0;
    for (int w = 0; w < NW; ++w) {
      if (done[w]) continue;
      const int f = S.bf_frame[w];
      int nL = 0, nRt = 0, fl = 0, ag = 0;
      for (int v = w; v < NW; ++v)
        if (!done[v] && S.bf_frame[v] == f) {
          nL += S.bf_nL[v];
          nRt += S.bf_nR[v];
          fl += S.bf_fill[v];
          ag |= S.bf_anyg[v];
        }
      int bL = nL > 0 ? atomicAdd(&A.cnt[nxt * A.nF + f], nL) : 0;
      int bR = nRt > 0 ? atomicAdd(&A.cntR[nxt * A.nF + f], nRt) : 0;
      if (fl > 0) atomicAdd(&A.fills[cur * A.nF + f], fl);
      if (ag && A.order == 2 && A.g_mode == 2) A.anyg[nxt * A.nF + f] = 1;
      for (int v = w; v < NW; ++v)
        if (!done[v] && S.bf_frame[v] == f) {
          S.bf_bL[v] = bL;
          S.bf_bR[v] = bR;
          bL += S.bf_nL[v];
          bR += S.bf_nR[v];
          done[v] = true;
        }
    }
  }
  __syncthreads();
  if (tracked && wf >= 0 && wn > 0) warp_copy(A, reg, wn, wf, nxt_list, S.bf_bL[warp], S.bf_bR[warp]);
}

// Bookkeeping of shell k-1 (block 0 only): report row, remaining, latch.
__device__ void bookkeep(const FillArgs& A, int k) {
  const int prev = (k + 3) % 4;  // counter slot of shell k-1
  for (int f = threadIdx.x; f < A.nF; f += blockDim.x) {
    const int F = frontier_size(A, prev, f);
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

// Shell prologue (every block): the frame table of the frontier in slot
// `slot` -- which frames are active and the prefix sums that deal their
// items over the grid.
__device__ __forceinline__ void build_prefix(const FillArgs& A, Smem& S) {
  if (threadIdx.x == 0) {
    int run = 0, runL = 0, runR = 0;
    for (int f = 0; f < A.nF; ++f) {
      S.u.g.pref[f] = run;
      S.u.g.prefL[f] = runL;
      S.u.g.prefR[f] = runR;
      run += S.u.g.nLf[f] + S.u.g.nRf[f];
      runL += S.u.g.nLf[f];
      runR += S.u.g.nRf[f];
    }
    S.u.g.pref[A.nF] = run;
    S.u.g.prefL[A.nF] = runL;
    S.u.g.prefR[A.nF] = runR;
    S.total = run;
    S.totalL = runL;
    S.totalR = runR;
  }
  __syncthreads();
}

__device__ __forceinline__ void stage_frame(Smem& S, int f, int nL, int nR, int done) {
  const bool act = nL + nR > 0 && done == 0;
  S.act[f] = act ? 1 : 0;
  S.u.g.nLf[f] = act ? nL : 0;
  S.u.g.nRf[f] = act ? nR : 0;
}

__device__ void load_p0(const FillArgs& A, Smem& S, int slot) {
  for (int f = threadIdx.x; f < A.nF; f += blockDim.x)
    stage_frame(S, f, A.cnt[slot * A.nF + f], A.cntR[slot * A.nF + f], A.done[f]);
  __syncthreads();
  build_prefix(A, S);
}

// Book-keeping done by one block while the others fill shell k: the report
// row of shell k-1, the unfillable mark of shell k's frames, and the
// clearing of the counter slot shell k+1 will append to (no block touches
// it in shell k).  Ordered before the shell-end barrier.
__device__ void book_shell(const FillArgs& A, int k, int cur, int clr) {
  if (k > 0) bookkeep(A, k);
  for (int f = threadIdx.x; f < A.nF; f += blockDim.x) {
    if (A.done[f] == 0 && frontier_size(A, cur, f) == 0 && A.remaining[f] > 0) A.done[f] = 2;
    A.cnt[clr * A.nF + f] = 0;
    A.cntR[clr * A.nF + f] = 0;
    A.anyg[clr * A.nF + f] = 0;
    A.fills[clr * A.nF + f] = 0;
    A.best_key[f] = 0ULL;
    A.best_p[f] = 0x7fffffff;
  }
}

#ifndef GF_SHELL_MIN_BLOCKS
#define GF_SHELL_MIN_BLOCKS 2
#endif

// R in 1..6: radius-specialised evaluators (K <= 128, one pairwise leaf);
// R == 0: the generic multi-leaf evaluator for larger balls.
// The guarded fill of one stalled frame (engine.py:334-348), by one warp:
// the argmax pixel best_p[f] is evaluated at the shell's snapshot (its rw,
// else the mean of its readable 8-neighbours, engine.py:252-267, else the
// frame is unfillable), written, and -- tracked -- dropped from the next
// frontier, its Inpaint neighbours claimed.  fvalid false: the warp idles.
template <int R, bool kTracked>
__device__ __forceinline__ void guard_fill_frame(const FillArgs& A, const BallParams& P, Smem& S,
                                                 int f_in, bool fvalid, int k, int cur, int nxt,
                                                 uint32_t* nxt_list) {
  const int lane = threadIdx.x & 31;
        const int f = f_in;
        const int p = fvalid ? A.best_p[f] : 0;
        const int fs = fvalid ? f : 0;
        float4* fw = A.work + (size_t)fs * A.HW;
        WorkSource src{fw, A.c3 ? A.c3 + (size_t)fs * A.HW : nullptr, A.H, A.W, A.C, k};
        // rw > 0 <=> the best confidence rw / tw is > 0 (NaN: tw = rw = 0);
        // then the value this shell's fill phase sampled for p
        const unsigned long long bk = fvalid ? A.best_key[f] : 0ULL;
        bool ok = bk != ~0ULL && bk != 0ULL;
        double v[4] = {0.0, 0.0, 0.0, 0.0};
        if (ok) {
          const float4 gv = A.gval[(size_t)fs * A.HW + p];
          v[0] = gv.x;
          v[1] = gv.y;
          v[2] = gv.z;
          v[3] = gv.w;
        }
        if (fvalid && lane == 0 && !ok) {
          // mean of readable 8-neighbours, engine.py:252-267
          double acc[4] = {0.0, 0.0, 0.0, 0.0};
          int n = 0;
          for (int o = 0; o < 8; ++o) {
            bool in;
            const int q = neighbor_of(A, (uint32_t)p, o, in);
            double cv[4];
            if (in && src.load(q, cv)) {
              for (int c = 0; c < 4; ++c) acc[c] += cv[c];
              ++n;
            }
          }
          if (n > 0) {
            for (int c = 0; c < 4; ++c) v[c] = acc[c] / n;
            ok = true;
          }
        }
        ok = __shfl_sync(0xffffffffu, ok, 0);
        if (fvalid && !ok && lane == 0) {
          A.done[f] = 2;  // unfillable: engine.py:342-345
          A.last_f[f] = frontier_size(A, cur, f);
        }
        if (fvalid && ok) {
          if (kTracked) {
            // every item re-entered the next list as a survivor: drop p, add
            // its Inpaint neighbours, refresh the data-term flag
            uint32_t* lst = nxt_list + (size_t)f * A.cap;
            const int nL = A.cnt[nxt * A.nF + f], nR = A.cntR[nxt * A.nF + f];
            int pos = -1;
            for (int i = lane; i < nL + nR; i += 32) {
              const int at = i < nL ? i : A.cap - 1 - (i - nL);
              if ((lst[at] & kEntryPix) == (uint32_t)p) pos = i;
            }
            for (int o = 16; o > 0; o >>= 1) pos = max(pos, __shfl_xor_sync(0xffffffffu, pos, o));
            __syncwarp();
            if (lane == 0 && pos >= 0) {
              if (pos < nL) {
                lst[pos] = lst[nL - 1];
                A.cnt[nxt * A.nF + f] = nL - 1;
              } else {
                const int rr = pos - nL;
                lst[A.cap - 1 - rr] = lst[A.cap - 1 - (nR - 1)];
                A.cntR[nxt * A.nF + f] = nR - 1;
              }
            }
            __syncwarp();
            if (lane < 8) {
              bool in;
              const int q = neighbor_of(A, (uint32_t)p, lane, in);
              const uint32_t qe = in ? claim(fw, q) : 0xffffffffu;
              if (qe != 0xffffffffu) {
                append_direct(A, nxt_list, nxt, f, qe);
                if (A.enter) A.enter[(size_t)f * A.HW + q] = k + 1;
              }
            }
            __syncwarp();
            if (A.order == 2 && A.g_mode == 2) {
              const int mL = A.cnt[nxt * A.nF + f], mR = A.cntR[nxt * A.nF + f];
              bool any = false;
              for (int i = lane; i < mL + mR; i += 32) {
                const int at = i < mL ? i : A.cap - 1 - (i - mL);
                any |= (lst[at] & kEntryRot) != 0;
              }
              any = __any_sync(0xffffffffu, any);
              if (lane == 0) A.anyg[nxt * A.nF + f] = any ? 1 : 0;
            }
          }
          if (lane == 0) {
            float4 o;
            o.x = (float)v[0];
            o.y = (float)v[1];
            o.z = (float)v[2];
            o.w = __int_as_float(k + 1);
            A.work[(size_t)f * A.HW + p] = o;
            const float fv[4] = {o.x, o.y, o.z, (float)v[3]};
            if (A.c3) A.c3[(size_t)f * A.HW + p] = fv[3];
            write_out(A, f, (uint32_t)p, fv, A.hull[2 * f], A.hull[2 * f + 1]);
            if (A.fillshell) A.fillshell[(size_t)f * A.HW + p] = k;
            A.fills[cur * A.nF + f] = 1;
            A.deadlocks[f] += 1;
          }
        }
}

// The deadlock guard of ONE stalled frame with a small frontier: block 0
// alone finds the argmax of the confidences the fill phase stored (NaN
// maximal, ties to the smallest pixel = numpy's first index of the sorted
// frontier, engine.py:336-337) by a block reduction, and its warp 0 does the
// guarded fill, while the other blocks wait at one grid barrier -- instead of
// the multi-frame guard's three barriers and grid-wide atomics (measured on
// the 256^2 half-planes: 24 -> ~19 us per guarded shell).
constexpr int kGuardBlockMax = 16384;

__device__ __forceinline__ void guard_argmax(const FillArgs& A, Smem& S, int f, int cur,
                                             const uint32_t* cur_list) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  constexpr int kWarps = kShellThreads / 32;
  const int T = S.u.g.pref[f + 1] - S.u.g.pref[f];
  const int nL = A.cnt[cur * A.nF + f];
  unsigned long long key = 0ULL;
  int pix = 0x7fffffff;
  for (int j = tid; j < T; j += kShellThreads) {
    const unsigned long long kk = conf_key(A.conf[(size_t)f * A.cap + j]);
    const int pp = (int)(entry_at(cur_list, A, f, j, nL) & kEntryPix);
    if (pix == 0x7fffffff || kk > key || (kk == key && pp < pix)) {
      key = kk;
      pix = pp;
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const unsigned long long k2 = __shfl_xor_sync(0xffffffffu, key, o);
    const int p2 = __shfl_xor_sync(0xffffffffu, pix, o);
    if (p2 != 0x7fffffff && (pix == 0x7fffffff || k2 > key || (k2 == key && p2 < pix))) {
      key = k2;
      pix = p2;
    }
  }
  if (lane == 0) {
    S.redk[warp] = key;
    S.red[warp] = pix;
  }
  __syncthreads();
  if (tid == 0) {
    for (int w = 0; w < kWarps; ++w) {
      const int p2 = S.red[w];
      const unsigned long long k2 = S.redk[w];
      if (p2 != 0x7fffffff && (pix == 0x7fffffff || k2 > key || (k2 == key && p2 < pix))) {
        key = k2;
        pix = p2;
      }
    }
    A.best_p[f] = pix;
    A.best_key[f] = key;
  }
}

template <int R, bool kTracked>
#ifdef GF_SHELL_MAXNREG
__global__ void __maxnreg__(GF_SHELL_MAXNREG)
#else
__global__ void __launch_bounds__(kShellThreads, GF_SHELL_MIN_BLOCKS)
#endif
    k_shells(const __grid_constant__ FillArgs A, const __grid_constant__ BallParams P,
             const __grid_constant__ BallTables tables) {
  cg::grid_group grid = cg::this_grid();
  extern __shared__ __align__(16) unsigned char smem_raw[];
  Smem& S = *reinterpret_cast<Smem*>(smem_raw);
#ifdef GF_PREP_PROF
  if (threadIdx.x == 0) atomicMin(&g_shell_prof[0], gtimer0());
#endif
  for (int i = threadIdx.x; i < P.K; i += blockDim.x) {
    S.tab.n[i] = tables.n[i];
    S.tab.m[i] = tables.m[i];
    S.tab.w0[i] = tables.w0[i];
    S.tab.w0f[i] = tables.w0f[i];
    S.tab.ni[i] = tables.ni[i];
    S.tab.mi[i] = tables.mi[i];
    S.tab.kn[i] = tables.kn[i];
    S.tab.off[i] = tables.ni[i] + tables.mi[i] * A.W;
  }
  pdl_wait();
#ifdef GF_PREP_PROF
  if (threadIdx.x == 0) {
    const unsigned long long t = gtimer0();
    atomicMin(&g_shell_prof[1], t);
    atomicMax(&g_shell_prof[2], t);
  }
#endif
  timeline_mark(A, 1, true);
  __syncthreads();

  // does any frame hold a Bystander outside its hull?  (else no clip work)
  if (threadIdx.x == 0) {
    int need = 0;
    for (int f = 0; f < A.nF && !need; ++f) need = !range_inside(A, f, A.bys_frame + 2 * f);
    S.any_clip = need;
  }
  __syncthreads();
  const bool clip_work = S.any_clip != 0;
  constexpr int kWarps = kShellThreads / 32;
  // rotated items take the warp-per-item path when the ball is one
  // pairwise leaf (K <= 128; then A.split == 1)
  constexpr int NL = R > 0 ? 1 : kMaxLeaves;
  constexpr bool kWarpRot = R > 0;
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  const int glane = lane & (kGroup - 1);
  // lattice items: LG lanes each (4 for the r <= 3 balls: K <= 28 samples,
  // 7 per lane), IPU = 32 / LG items per warp round
#ifndef GF_LATTICE_LANES
#define GF_LATTICE_LANES 4
#endif
#ifndef GF_LG4_MAX_R
#define GF_LG4_MAX_R 3
#endif
  constexpr int LG = (R > 0 && R <= GF_LG4_MAX_R) ? GF_LATTICE_LANES : 8;
  constexpr int IPU = 32 / LG;
  const int lglane = lane & (LG - 1);
  const int lsub = lane / LG;
  uint32_t* reg = S.u.g.app + warp * kWarpAppCap;
  const bool booker = blockIdx.x == gridDim.x - 1;  // last block: fewest fill units

  load_p0(A, S, 0);
  int k = 0;
  for (;; ++k) {
    // Frontier lists alternate between two buffers; their counters (cnt,
    // cntR, anyg) and the fill counts rotate through four slots: cur = this
    // shell's frontier, nxt = the one being built, prv = shell k-1's (its
    // report row is booked in this shell, its g flag read by the data-term
    // latch), clr = shell k-2's, cleared by the booking block for shell k+1
    // -- a slot no other block reads or writes in this shell.
    const int cur = k % 4, nxt = (k + 1) % 4, prv = (k + 3) % 4, clr = (k + 2) % 4;
    uint32_t* cur_list = (k & 1) ? A.list1 : A.list0;
    uint32_t* nxt_list = (k & 1) ? A.list0 : A.list1;
    const int T = S.total;
    if (T == 0) break;
    trace_set(A, k, 0, gtimer());
    trace_set(A, k, 5, (unsigned long long)T);

    // ---- A: fill (+ fused frontier update when tracked)
    // Work units, dealt over every warp of the grid: a rotated
    // item (whole warp) or a round of 4 consecutive lattice items (one per
    // 8-lane group).  No block barrier.
    {
      const int TR = S.totalR, TL = S.totalL;
      const int UL = (TL + IPU - 1) / IPU;
      const int U = TR + UL;
      const int NW = gridDim.x * kWarps;
      int wn = 0, wf = -1, wfills = 0;
      // units dealt block-contiguously: consecutive list entries are
      // neighbouring pixels, and a block's warps share its SM's L1 lines
      // (dealing across SMs first measured 5% slower)
      const int u0 = blockIdx.x * kWarps + warp;
      for (int u = u0; u < U; u += NW) {
        if (kWarpRot && u < TR) {
          // ---- rotated-ball item, one whole warp
          const int f = find_frame(S.u.g.prefR, A.nF, u);
          const int nL = S.u.g.prefL[f + 1] - S.u.g.prefL[f];
          const int rr = u - S.u.g.prefR[f];
          const int j = nL + rr;
          GF_FINE(const unsigned long long fr0 = fine_after(0u);)
          const uint32_t e = cur_list[(size_t)f * A.cap + A.cap - 1 - rr];
          const uint32_t p = e & kEntryPix;
          int pi_r, pj_r;
          col_row(A, (int)p, pi_r, pj_r);
          GF_FINE(const unsigned long long fr1 = fine_after(e);)
          if (f != wf) {
            if (kTracked && wf >= 0) warp_flush(A, reg, wn, wf, nxt_list, nxt);
            if (lane == 0 && wf >= 0 && wfills > 0) atomicAdd(&A.fills[cur * A.nF + wf], wfills);
            wfills = 0;
            wf = f;
          }
          const unsigned long long hl = A.hull[2 * f], hh = A.hull[2 * f + 1];
          const bool dt_eff = (A.order == 2) && !dt_dead_at(A, f, k, prv) && frontier_has_g(A, cur, f);
          const double4 g4 = A.gbuf[(size_t)f * A.HW + p];
          const double gx = g4.x, gy = g4.y;
          float4* fw = A.work + (size_t)f * A.HW;
          WorkSource src{fw, A.c3 ? A.c3 + (size_t)f * A.HW : nullptr, A.H, A.W, A.C, k};
          SampleResult res;
          GF_FINE(const unsigned long long tw0 = A.trace ? gtimer() : 0ULL;)
          if constexpr (R > 0)
            eval_rot_warp<R>(P, S.tab, src, lane, (double)pi_r, (double)pj_r, gx, gy, g4.z, g4.w,
                             res);
          GF_FINE(if (A.trace && lane == 0) trace_max_val(A, k, 7, gtimer() - tw0);)
          GF_FINE(const unsigned long long fr2 = fine_after((unsigned)(__double_as_longlong(res.rw) >> 32));)
          bool filled = false;
          if (lane == 0) filled = decide_and_write(A, f, j, p, k, dt_eff, gx, gy, res, hl, hh);
          filled = __shfl_sync(0xffffffffu, filled, 0);
          GF_FINE(const unsigned long long fr3 = fine_after(filled ? 1u : 0u);)
          if (lane == 0 && filled) ++wfills;
          if (kTracked)
            activate<8>(A, reg, wn, true, nxt_list, nxt, fw, f, k, lane < 8 ? lane : -1, filled, e,
                        0xffu, pi_r, pj_r);
          GF_FINE(if (lane == 0) fine_put(A, k, 7, fr2 - fr1); (void)fr0; (void)fr3;)
        } else {
          // ---- lattice round: items IPU q .. IPU q + IPU-1 of the concatenated
          // front parts, one per LG-lane group
          GF_FINE(const unsigned long long fl0 = fine_after(0u);)
          const int q = kWarpRot ? u - TR : u;
          const int t = q * IPU + lsub;
          const int TLx = kWarpRot ? TL : T;  // NL > 1: everything lives in the front part
          const bool valid = t < TLx;
          const int* pf = kWarpRot ? S.u.g.prefL : S.u.g.pref;
          const int f = valid ? find_frame(pf, A.nF, t) : -1;
          const int f0 = __shfl_sync(0xffffffffu, f, 0);
          const bool uniform = __all_sync(0xffffffffu, !valid || f == f0);
          if (!uniform || f0 != wf) {
            if (kTracked && wf >= 0) warp_flush(A, reg, wn, wf, nxt_list, nxt);
            if (lane == 0 && wf >= 0 && wfills > 0) atomicAdd(&A.fills[cur * A.nF + wf], wfills);
            wfills = 0;
            wf = uniform ? f0 : -1;
          }
          const int fs = valid ? f : 0;
          const unsigned long long hl = A.hull[2 * fs], hh = A.hull[2 * fs + 1];
          const int j = valid ? t - pf[fs] : 0;
          const uint32_t e = valid ? cur_list[(size_t)fs * A.cap + j] : 0u;
          const uint32_t p = e & kEntryPix;
          int pi, pj;
          col_row(A, (int)p, pi, pj);
          GF_FINE(const unsigned long long fl1 = fine_after(e);)
          float4* fw = A.work + (size_t)fs * A.HW;
          WorkSource src{fw, A.c3 ? A.c3 + (size_t)fs * A.HW : nullptr, A.H, A.W, A.C, k};
          const bool dt_eff =
              valid && (A.order == 2) && !dt_dead_at(A, fs, k, prv) && frontier_has_g(A, cur, fs);
          double gx = 0.0, gy = 0.0;
          SampleResult res;
          GF_FINE(const unsigned long long te0 = A.trace ? gtimer() : 0ULL;)
          if constexpr (R > 0) {
            eval_lattice<R, LG>(P, S.tab, src, lglane, lsub, valid, pi, pj, res);
          } else {
            if (valid && (e & kEntryRot)) frame_guide(A, fs, (int)p, gx, gy);
            eval_item<NL, 0>(P, S.tab, src, glane, valid, (double)pi, (double)pj, true, gx, gy,
                             res);
          }
          GF_FINE(if (A.trace && valid && lglane == 0) trace_max_val(A, k, 6, gtimer() - te0);)
          GF_FINE(const unsigned long long fl2 = fine_after((unsigned)(__double_as_longlong(res.rw) >> 32));)
          bool filled = false;
          if (valid && lglane == 0) filled = decide_and_write(A, fs, j, p, k, dt_eff, gx, gy, res, hl, hh);
          filled = __shfl_sync(0xffffffffu, filled, 0, LG);
          GF_FINE(const unsigned long long fl3 = fine_after(filled ? 1u : 0u);)
          if (kTracked)
            activate<LG>(A, reg, wn, uniform, nxt_list, nxt, fw, fs, k, valid ? lglane : -1, filled, e,
                         R > 0 ? res.nb : 0xffu, pi, pj);
          GF_FINE(const unsigned long long fl4 = fine_after((unsigned)wn);
                  if (valid && lglane == 0) {
                    fine_put(A, k, 0, fl1 - fl0); fine_put(A, k, 1, fl2 - fl1);
                    fine_add(A, k, 2, fl2 - fl1); fine_add(A, k, 3, 1);
                    fine_put(A, k, 4, fl4 - fl2); (void)fl3;
                  })
          const int nf = (valid && lglane == 0 && filled) ? 1 : 0;
          if (uniform) wfills += __reduce_add_sync(0xffffffffu, (unsigned)nf);
          else if (nf) atomicAdd(&A.fills[cur * A.nF + fs], 1);
        }
        if (kTracked && wn > kWarpAppCap - 80) warp_flush(A, reg, wn, wf, nxt_list, nxt);
      }
      GF_FINE(const unsigned long long ff0 = fine_after((unsigned)wn);)
      if (kTracked && wf >= 0) warp_flush(A, reg, wn, wf, nxt_list, nxt);
      if (lane == 0 && wf >= 0 && wfills > 0) atomicAdd(&A.fills[cur * A.nF + wf], wfills);
      GF_FINE(const unsigned long long ff1 = fine_after((unsigned)wn);
              if (lane == 0 && wf >= 0) fine_put(A, k, 5, ff1 - ff0);)
      if (A.trace && lane == 0 && k < A.trace_cap)
        atomicMax(&A.trace[k * kTraceSlots + 1], gtimer());
    }
    if (booker) book_shell(A, k, cur, clr);
    grid.sync();
    trace_set(A, k, 2, gtimer());

    // ---- G: deadlock guard (engine.py:334-348), only when some frame
    // stalled.  The stall test and the next shell's frame table come from
    // one round of loads (tracked: the next frontier is complete here).
    int any = 0;
    for (int f = threadIdx.x; f < A.nF; f += blockDim.x) {
      const int d = S.act[f] && A.fills[cur * A.nF + f] == 0;
      S.dl[f] = (unsigned char)d;
      any |= d;
      if (kTracked) stage_frame(S, f, A.cnt[nxt * A.nF + f], A.cntR[nxt * A.nF + f], A.done[f]);
    }
    any = __syncthreads_or(any);
    if (kTracked && !any) build_prefix(A, S);
    if (any) {
      if (threadIdx.x == 0) {
        int nst = 0, fst = 0;
        for (int f = 0; f < A.nF; ++f)
          if (S.dl[f]) {
            ++nst;
            fst = f;
          }
        S.g_f = fst;
        S.g_one = nst == 1 && S.u.g.pref[fst + 1] - S.u.g.pref[fst] <= kGuardBlockMax;
      }
      __syncthreads();
    }
    if (any && S.g_one) {
      if (blockIdx.x == 0) guard_argmax(A, S, S.g_f, cur, cur_list);
    } else if (any) {
      const int chunk = max(kShellThreads, (T + gridDim.x - 1) / gridDim.x);
      const int c_lo = min(T, blockIdx.x * chunk), c_hi = min(T, c_lo + chunk);
      // G1: max confidence key per stalled frame
      for (int s = c_lo; s < c_hi;) {
        const int f = find_frame(S.u.g.pref, A.nF, s);
        const int fe = min(c_hi, S.u.g.pref[f + 1]);
        unsigned long long key = 0ULL;
        if (S.dl[f]) {
          for (int t = s + threadIdx.x; t < fe; t += blockDim.x) {
            const unsigned long long kk = conf_key(A.conf[(size_t)f * A.cap + (t - S.u.g.pref[f])]);
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
        const int f = find_frame(S.u.g.pref, A.nF, s);
        const int fe = min(c_hi, S.u.g.pref[f + 1]);
        if (S.dl[f]) {
          const unsigned long long best = A.best_key[f];
          const int nL = A.cnt[cur * A.nF + f];
          for (int t = s + threadIdx.x; t < fe; t += blockDim.x) {
            const int j = t - S.u.g.pref[f];
            if (conf_key(A.conf[(size_t)f * A.cap + j]) == best)
              atomicMin(&A.best_p[f], (int)(entry_at(cur_list, A, f, j, nL) & kEntryPix));
          }
        }
        s = fe;
      }
      grid.sync();
    }
    if (any) {
      // G3: the guarded fill, one warp per stalled frame (single frame: warp
      // 0 of block 0, which found its argmax)
      __syncthreads();
      const bool one = S.g_one != 0;
      for (int fb = one ? 0 : blockIdx.x * kWarps; fb < A.nF; fb += gridDim.x * kWarps) {
        const int f = one ? S.g_f : fb + warp;
        const bool fv = one ? (blockIdx.x == 0 && warp == 0) : (f < A.nF && S.dl[f]);
        guard_fill_frame<R, kTracked>(A, P, S, f, fv, k, cur, nxt, nxt_list);
        if (one) break;
      }
      grid.sync();
      if (kTracked) {
        load_p0(A, S, nxt);
      }
    }

    // ---- B: untracked frontier = full-lattice rescan (engine.py:357-360)
    if (!kTracked) {
      int nA = 0;
      for (int f = 0; f < A.nF; ++f) nA += S.act[f] && A.done[f] == 0;
      const long long TP = (long long)nA * A.HW;
      const long long pchunk =
          ((TP + gridDim.x - 1) / gridDim.x + kShellThreads - 1) / kShellThreads * kShellThreads;
      const long long p_lo = min(TP, (long long)blockIdx.x * pchunk), p_hi = min(TP, p_lo + pchunk);
      int wn = 0;
      for (long long s = p_lo; s < p_hi;) {
        const int a = (int)(s / A.HW);
        int f = -1;
        for (int ff = 0, seen = 0; ff < A.nF; ++ff)
          if (S.act[ff] && A.done[ff] == 0) {
            if (seen == a) {
              f = ff;
              break;
            }
            ++seen;
          }
        const long long fe = min(p_hi, (long long)(a + 1) * A.HW);
        float4* fw = A.work + (size_t)f * A.HW;
        for (long long base = s; base < fe; base += kShellThreads) {
          const long long t = base + threadIdx.x;
          bool want = false;
          uint32_t e = 0;
          if (t < fe) {
            const int p = (int)(t - (long long)a * A.HW);
            // only Inpaint pixels have a working-buffer entry far from D
            const int st = A.labels[(size_t)f * A.HW + p] == 255 ? stamp_of(fw, p) : 0;
            if (stamp_unfilled(st)) {
              for (int o = 0; o < 8 && !want; ++o) {
                bool in;
                const int q = neighbor_of(A, (uint32_t)p, o, in);
                if (in && stamp_of(fw, q) <= k + 1) want = true;
              }
              if (want && (st & ~kRotBit) == kStampInactive) {
                *stamp_ptr(fw, p) = st | 2;  // INACTIVE -> ACTIVE, rot bit kept
                if (A.enter) A.enter[(size_t)f * A.HW + p] = k + 1;
              }
              e = (uint32_t)p | ((st & kRotBit) ? kEntryRot : 0u);
            }
          }
          warp_push(reg, wn, want, e);
          if (wn > kWarpAppCap - 32) warp_flush(A, reg, wn, f, nxt_list, nxt);
        }
        warp_flush(A, reg, wn, f, nxt_list, nxt);
        s = fe;
      }
      trace_max(A, k, 3);
      grid.sync();
      trace_set(A, k, 4, gtimer());
      load_p0(A, S, nxt);
    }
  }
  // Bystander clip of the tiles that need it
  while (clip_work && clip_claim(A)) {
  }
  timeline_mark(A, 1, false);
  // the last shell's row, then the stats
  if (booker) {
    if (k > 0) bookkeep(A, k);
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
      st[GF_STAT_BAD_LABELS] = A.badlab[f];
    }
  }
}

// ---------------------------------------------------------------- host

static void launch_prep(bool f64, int C, dim3 grid, cudaStream_t stream, const FillArgs& A) {
#define GF_PREP(T, CC)                                   \
  do {                                                   \
    k_prep<T, CC><<<grid, kThreads, 0, stream>>>(A);     \
  } while (0)
  if (f64) {
    switch (C) {
      case 1: GF_PREP(double, 1); break;
      case 2: GF_PREP(double, 2); break;
      case 3: GF_PREP(double, 3); break;
      default: GF_PREP(double, 4); break;
    }
  } else {
    switch (C) {
      case 1: GF_PREP(float, 1); break;
      case 2: GF_PREP(float, 2); break;
      case 3: GF_PREP(float, 3); break;
      default: GF_PREP(float, 4); break;
    }
  }
#undef GF_PREP
}

// cuTensorMapEncodeTiled through the runtime's driver entry point (no -lcuda)
static PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* ptr = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPointByVersion("cuTensorMapEncodeTiled", &ptr, 12000, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(ptr);
  });
  return fn;
}

// 3-D map (cols, rows, frames) with a (box_c, box_r, 1) box
static bool encode_map(CUtensorMap* m, CUtensorMapDataType dt, size_t elem, void* base, int cols,
                       int rows, int frames, int box_c, int box_r) {
  auto enc = tensor_map_encoder();
  if (!enc) return false;
  const cuuint64_t dims[3] = {(cuuint64_t)cols, (cuuint64_t)rows, (cuuint64_t)frames};
  const cuuint64_t strides[2] = {(cuuint64_t)cols * elem, (cuuint64_t)cols * rows * elem};
  const cuuint32_t box[3] = {(cuuint32_t)box_c, (cuuint32_t)box_r, 1};
  const cuuint32_t es[3] = {1, 1, 1};
  return enc(m, dt, 3, base, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
             CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// The TMA prep applies when every row is a multiple of 16 bytes (the maps'
// stride rule) and x is not periodic (a box does not wrap); GF_NO_TMA=1
// forces the plain kernel (A/B experiments).
static bool launch_prep_tma(bool f64, int C, dim3 grid, cudaStream_t stream, const FillArgs& A,
                            const void* image, void* out, const uint8_t* labels) {
  if (A.periodic || getenv("GF_NO_TMA")) return false;
  const size_t elem = f64 ? 8 : 4;
  if ((size_t)A.W * C * elem % 16 || A.W % 16) return false;
  const int ext = kTile + 2 * A.halo;
  PrepMaps M;
  memset(&M, 0, sizeof(M));
  M.lab_bw = kLabBoxMax;
  if (A.halo > 16) return false;
  const CUtensorMapDataType dt = f64 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT64 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32;
  if (!encode_map(&M.img, dt, elem, const_cast<void*>(image), A.W * C, A.H, A.nF, kTile * C, kTile) ||
      !encode_map(&M.out, dt, elem, out, A.W * C, A.H, A.nF, kTile * C, kTile) ||
      !encode_map(&M.lab, CU_TENSOR_MAP_DATA_TYPE_UINT8, 1, const_cast<uint8_t*>(labels), A.W, A.H,
                  A.nF, M.lab_bw, ext))
    return false;
#define GF_PREP_TMA(T, CC)                                       \
  do {                                                          \
    k_prep_tma<T, CC><<<grid, kThreads, 0, stream>>>(M, A);     \
  } while (0)
  if (f64) {
    switch (C) {
      case 1: GF_PREP_TMA(double, 1); break;
      case 2: GF_PREP_TMA(double, 2); break;
      case 3: GF_PREP_TMA(double, 3); break;
      default: GF_PREP_TMA(double, 4); break;
    }
  } else {
    switch (C) {
      case 1: GF_PREP_TMA(float, 1); break;
      case 2: GF_PREP_TMA(float, 2); break;
      case 3: GF_PREP_TMA(float, 3); break;
      default: GF_PREP_TMA(float, 4); break;
    }
  }
#undef GF_PREP_TMA
  return true;
}

static size_t align_up(size_t x) { return (x + 255) & ~size_t(255); }

// round-up multiplier for division by d of dividends below 2^31 (q =
// umulhi(n, mul) >> shr), the scheme of CUTLASS's FastDivmod
static void div_magic(int d, unsigned& mul, int& shr) {
  if (d <= 1) {
    mul = 0;
    shr = 0;
    return;
  }
  int l = 0;
  while ((1LL << l) < d) ++l;
  const int p = 31 + l;
  mul = (unsigned)(((1ULL << p) + (unsigned long long)d - 1) / (unsigned long long)d);
  shr = p - 32;
}

struct Layout {
  size_t work, c3, list0, list1, conf, gval, gbuf, bys, ints, u64, total;
};

static int tiles_of(int H, int W) {
  return ((W + kTile - 1) / kTile) * ((H + kTile - 1) / kTile);
}

static Layout layout_for(int nF, int H, int W, int C, bool need_g) {
  const int HW = H * W;
  Layout L;
  size_t off = 0;
  const size_t n = (size_t)nF * HW;
  L.work = off; off = align_up(off + n * sizeof(float4));
  L.gbuf = off; off = align_up(off + (need_g ? n * sizeof(double4) : 0));
  L.c3 = off; off = align_up(off + (C > 3 ? n * sizeof(float) : 0));
  L.list0 = off; off = align_up(off + n * sizeof(uint32_t));
  L.list1 = off; off = align_up(off + n * sizeof(uint32_t));
  L.conf = off; off = align_up(off + n * sizeof(double));
  L.gval = off; off = align_up(off + n * sizeof(float4));
  L.bys = off; off = align_up(off + (size_t)nF * tiles_of(H, W) * 2 * sizeof(unsigned long long));
  L.ints = off; off = align_up(off + (size_t)nF * kIntsPerFrame * sizeof(int));
  L.u64 = off; off = align_up(off + (size_t)nF * 6 * sizeof(unsigned long long));
  L.total = off;
  return L;
}

size_t fill_workspace_bytes(int nF, int H, int W, int C, bool need_g) {
  if (nF <= 0 || H <= 0 || W <= 0) return 0;
  return layout_for(nF, H, W, C, need_g).total;
}

// kernel specialised on the ball size: samples per lane = ceil(K / 8)
template <bool kTracked>
static const void* shell_kernel(const BallParams& P) {
  if (P.plan.n_leaves == 1) {
    switch (P.r) {
      case 1: return (const void*)k_shells<1, kTracked>;
      case 2: return (const void*)k_shells<2, kTracked>;
      case 3: return (const void*)k_shells<3, kTracked>;
      case 4: return (const void*)k_shells<4, kTracked>;
      case 5: return (const void*)k_shells<5, kTracked>;
      case 6: return (const void*)k_shells<6, kTracked>;
      default: break;
    }
  }
  return (const void*)k_shells<0, kTracked>;
}

// Cooperative grid size of a shell kernel on the current device, cached per
// (device, kernel): the attribute call and the occupancy query cost host
// microseconds on every fill otherwise.
static int coop_grid(const void* fn, size_t smem, int* out_grid) {
  struct Entry {
    int dev;
    const void* fn;
    size_t smem;
    int grid;
  };
  static std::mutex mu;
  static std::vector<Entry> cache;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return GF_E_CUDA;
  {
    std::lock_guard<std::mutex> lock(mu);
    for (const Entry& e : cache)
      if (e.dev == dev && e.fn == fn && e.smem == smem) {
        *out_grid = e.grid;
        return GF_OK;
      }
  }
  int sms = 0, coop = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, dev);
  if (!coop) return set_error(GF_E_UNSUPPORTED, "device lacks cooperative launch");
  if (cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
    return set_error(GF_E_CUDA, "cudaFuncSetAttribute failed");
  int per_sm = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, kShellThreads, smem) != cudaSuccess ||
      per_sm <= 0)
    return set_error(GF_E_CUDA, "occupancy query failed");
  // GF_SHELL_BPS caps the blocks per SM (experiments: room for a concurrent prep)
  if (const char* e = getenv("GF_SHELL_BPS")) per_sm = std::max(1, std::min(per_sm, atoi(e)));
  *out_grid = sms * per_sm;
  std::lock_guard<std::mutex> lock(mu);
  cache.push_back(Entry{dev, fn, smem, *out_grid});
  return GF_OK;
}

int fill_launch(const gf_frames* fr, const gf_fill_params* prm, const gf_fill_outputs* out,
                const gf_splines* spl, void* ws, size_t ws_bytes, cudaStream_t stream,
                const BallParams& P, const BallTables& host_tab) {
  const int nF = fr->n_frames, H = fr->height, W = fr->width, C = fr->channels;
  const int HW = H * W;
  const bool raster = spl && spl->n_seg > 0;
  const bool need_g = raster || prm->g_mode != GF_G_ZERO;
  const Layout L = layout_for(nF, H, W, C, need_g);
  if (ws_bytes < L.total) return set_error(GF_E_WORKSPACE, "workspace too small");
  unsigned char* base = static_cast<unsigned char*>(ws);

  FillArgs A;
  memset(&A, 0, sizeof(A));
  A.nF = nF; A.H = H; A.W = W; A.HW = HW; A.C = C; A.cap = HW;
  div_magic(W, A.w_mul, A.w_shr);
  A.image = fr->image;
  A.labels = fr->labels;
  A.gsrc = fr->guide;
  A.out = fr->out;
  if (raster) {
    A.n_seg = spl->n_seg;
    A.frame_seg = spl->frame_seg;
    A.seg = reinterpret_cast<const double4*>(spl->seg);
    A.seg_spline = spl->seg_spline;
    A.dirs = reinterpret_cast<const double2*>(spl->dirs);
    A.cut = 3.0 * spl->eta;
    A.c2eta = 2.0 * spl->eta * spl->eta;
  }
  A.gbuf = need_g ? reinterpret_cast<double4*>(base + L.gbuf) : nullptr;
  A.trace = reinterpret_cast<unsigned long long*>(out->shell_trace);
  A.trace_cap = out->shell_trace ? out->trace_cap : 0;
  A.work = reinterpret_cast<float4*>(base + L.work);
  A.c3 = C > 3 ? reinterpret_cast<float*>(base + L.c3) : nullptr;
  A.list0 = reinterpret_cast<uint32_t*>(base + L.list0);
  A.list1 = reinterpret_cast<uint32_t*>(base + L.list1);
  A.conf = reinterpret_cast<double*>(base + L.conf);
  A.gval = reinterpret_cast<float4*>(base + L.gval);
  int* ints = reinterpret_cast<int*>(base + L.ints);
  A.cnt = ints;              ints += 4 * nF;
  A.cntR = ints;             ints += 4 * nF;
  A.fills = ints;            ints += 4 * nF;
  A.anyg = ints;             ints += 4 * nF;
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
  A.badlab = ints;           ints += nF;
  A.clip_next = ints;         ints += 1;
  A.ntiles = tiles_of(H, W);
  A.clip_total = nF * A.ntiles;
  A.bys = reinterpret_cast<unsigned long long*>(base + L.bys);
  unsigned long long* u64 = reinterpret_cast<unsigned long long*>(base + L.u64);
  A.best_key = u64;
  A.hull = u64 + nF;
  A.bys_frame = u64 + 3 * nF;
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
  A.split = P.plan.n_leaves == 1 ? 1 : 0;
  A.halo = P.r + 1;
  A.dtype = fr->dtype;

  // per-frame counters start at zero (the hull minimum is stored inverted
  // and the data-term latch as a "dead" flag, so zero is the initial state)
  if (cudaMemsetAsync(base + L.ints, 0, L.u64 + (size_t)nF * 6 * sizeof(unsigned long long) - L.ints,
                      stream) != cudaSuccess)
    return set_error(GF_E_CUDA, "memset failed");
  {
    const dim3 pg((W + kTile - 1) / kTile, (H + kTile - 1) / kTile, nF);
    if (!launch_prep_tma(fr->dtype == GF_F64, C, pg, stream, A, fr->image, fr->out, fr->labels))
      launch_prep(fr->dtype == GF_F64, C, pg, stream, A);
  }
  count_launches(1);
  if (cudaPeekAtLastError() != cudaSuccess)
    return set_error(GF_E_CUDA, cudaGetErrorString(cudaGetLastError()));

  const size_t smem = sizeof(Smem);
  const void* fn = prm->tracked ? shell_kernel<true>(P) : shell_kernel<false>(P);
  int grid = 0;
  int rc = coop_grid(fn, smem, &grid);
  if (rc != GF_OK) return rc;
  void* args[] = {(void*)&A, (void*)&P, (void*)&host_tab};
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(kShellThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeCooperative;
  attr[0].val.cooperative = 1;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 2;
  cudaError_t e = cudaLaunchKernelExC(&cfg, fn, args);
#ifdef GF_PDL_STRICT
  if (e != cudaSuccess) return set_error(GF_E_CUDA, cudaGetErrorString(e));
#endif
  if (e != cudaSuccess) {
    // without programmatic serialisation: a plain cooperative launch
    (void)cudaGetLastError();
    e = cudaLaunchCooperativeKernel(fn, grid, kShellThreads, args, smem, stream);
  }
  if (e != cudaSuccess) return set_error(GF_E_CUDA, cudaGetErrorString(e));
  count_launches(1);

  e = cudaPeekAtLastError();
  if (e != cudaSuccess) return set_error(GF_E_CUDA, cudaGetErrorString(e));
  return GF_OK;
}

}  // namespace gf
