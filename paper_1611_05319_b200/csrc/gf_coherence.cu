// Coherence-transport guide directions on the device:
// g_source = "modified_structure_tensor", engine._resolve_g (engine.py:243-249)
// -> guide.coherence_directions (guide.py:330-355) -> guide._tensor_field
// (guide.py:91-120) and guide.eigen_2x2 (guide.py:123-136).
//
// The reference evaluates the masked structure tensor on the frontier's
// bounding box padded by cascade_radius + 2.  Every tap that reaches a queried
// pixel lies inside that crop (the pad exceeds the sigma window + 1 gradient
// step + the rho window), so evaluating the same separable passes over the
// whole frame gives the queried values operation for operation.  The passes:
//   seed     P = [ind, ind*u_0 .. ind*u_{C-1}]          ind = (label == Readable)
//   smooth   scipy.ndimage.gaussian_filter(truncate=2, mode='constant', cval=0):
//            axis 0 then axis 1, each a symmetric correlate1d summed from the
//            outermost tap pair inwards: t = x[0]*w0; t += (x[-k] + x[k]) * wk,
//            k = R..1 (bit-matches scipy, checked against it on the host)
//   tensor   v_c = S_c / (S_ind > 0 ? S_ind : 1); (gy, gx) = np.gradient(v_c)
//            (central /2.0 inside, one-sided at the frame edges);
//            J11 += gx*gx, J12 += gx*gy, J22 += gy*gy over channels; J *= ind
//   smooth   the four planes [J11, J12, J22, ind] with rho -- only at the
//            queried pixels (k_ct_query: column sums, then the row sum)
//   query    a = J11s / safe_r ...; eigen split; coh = tanh((hi - lo) / lam);
//            g = coh * (-sin phi, cos phi), g = 0 where mass_r <= 0.
// The weights follow scipy's _gaussian_kernel1d: exp(-0.5 / s^2 * x^2) / sum,
// with numpy's exp (exp_np) and pairwise sum (plan_sum) restated.
// arctan2 / tanh / sin / cos are numpy's own, restated bit for bit
// (gf_npmath.cuh): the smart-order deadlock argmax can hinge on a 1-ulp
// difference in g.
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include <stdio.h>
#include <stdlib.h>

#include <algorithm>
#include <mutex>
#include <vector>

#include <cooperative_groups.h>

#include "gf_internal.cuh"
#include "gf_math.cuh"
#include "gf_npmath.cuh"

namespace cg = cooperative_groups;

namespace gf {

namespace {

constexpr int kMaxTaps = 64;  // radius int(2 s + 0.5) <= 64

struct Taps {
  double w[kMaxTaps + 1];  // w[k] = weight at offset +-k
  int R;
};

int make_taps(double s, Taps& t) {
  if (!(s > 0.0) || !(2.0 * s + 0.5 < (double)kMaxTaps)) return GF_E_UNSUPPORTED;
  const int R = (int)(2.0 * s + 0.5);
  const int n = 2 * R + 1;
  double phi[2 * kMaxTaps + 1];
  const double scale = -0.5 / (s * s);
  for (int i = 0; i < n; ++i) {
    const double x = (double)(i - R);
    phi[i] = exp_np(scale * (x * x));
  }
  const double sum = plan_sum(make_plan(n), phi);
  t.R = R;
  for (int k = 0; k <= R; ++k) t.w[k] = phi[R + k] / sum;
  return GF_OK;
}

// Grids are 2-D: x over columns (128 per block), y over rows -- no 64-bit
// division per pixel.  Work is limited to the 128 x kTileRows tiles that a
// query can reach (k_ct_tiles): a query reads J within R_rho, J reads S
// within 1, S reads the axis-0 output within R_sigma columns -- every value
// outside the reach box R_rho + R_sigma + 1 is never read.
constexpr int kTileRows = 8;

__global__ void k_ct_tiles(int H, int W, int n, const int64_t* __restrict__ idx, int D,
                           int tiles_x, uint8_t* __restrict__ tiles, double* __restrict__ points) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= n) return;
  const int64_t p = idx[k];
  const int j = (int)(p / W), i = (int)(p % W);
  if (points) {  // (x, y) of the query for gf_sample_points
    points[2 * k] = (double)i;
    points[2 * k + 1] = (double)j;
  }
  const int ty0 = max(0, j - D) / kTileRows, ty1 = min(H - 1, j + D) / kTileRows;
  const int tx0 = max(0, i - D) / 128, tx1 = min(W - 1, i + D) / 128;
  for (int ty = ty0; ty <= ty1; ++ty)
    for (int tx = tx0; tx <= tx1; ++tx) tiles[ty * tiles_x + tx] = 1;
}

// axis-1 pass of one plane row (blockIdx.z = plane)
__global__ void k_ct_smooth1(int H, int W, const Taps t, const double* __restrict__ in,
                             double* __restrict__ out, const uint8_t* __restrict__ tiles,
                             int tiles_x) {
  if (!tiles[(blockIdx.y / kTileRows) * tiles_x + blockIdx.x]) return;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= W) return;
  const int64_t row = ((int64_t)blockIdx.z * H + blockIdx.y) * W;
  const double* x = in + row + i;
  double acc = x[0] * t.w[0];
  for (int k = t.R; k >= 1; --k) {
    const double a = i - k >= 0 ? x[-k] : 0.0;
    const double b = i + k < W ? x[k] : 0.0;
    acc += (a + b) * t.w[k];
  }
  out[row + i] = acc;
}

// seed fused into the sigma stage's axis-0 pass, all C + 1 planes per thread:
// plane 0 = ind, plane c+1 = ind*u_c
template <int C>
__global__ void k_ct_seed_smooth0(int H, int W, const Taps t, const double* __restrict__ u,
                                  const uint8_t* __restrict__ labels, double* __restrict__ out,
                                  const uint8_t* __restrict__ tiles, int tiles_x) {
  if (!tiles[(blockIdx.y / kTileRows) * tiles_x + blockIdx.x]) return;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= W) return;
  const int j = blockIdx.y;
  const int64_t HW = (int64_t)H * W;
  double acc[C + 1];
  auto tap = [&](int jj, double (&v)[C + 1]) {
    const int64_t pp = (int64_t)jj * W + i;
    const double ind = labels[pp] == 0 ? 1.0 : 0.0;
    v[0] = ind;
#pragma unroll
    for (int c = 0; c < C; ++c) v[c + 1] = ind * u[pp * C + c];
  };
  double v0[C + 1];
  tap(j, v0);
#pragma unroll
  for (int f = 0; f <= C; ++f) acc[f] = v0[f] * t.w[0];
  for (int k = t.R; k >= 1; --k) {
    double a[C + 1], b[C + 1];
    if (j - k >= 0) tap(j - k, a);
    else
#pragma unroll
      for (int f = 0; f <= C; ++f) a[f] = 0.0;
    if (j + k < H) tap(j + k, b);
    else
#pragma unroll
      for (int f = 0; f <= C; ++f) b[f] = 0.0;
#pragma unroll
    for (int f = 0; f <= C; ++f) acc[f] += (a[f] + b[f]) * t.w[k];
  }
  const int64_t p = (int64_t)j * W + i;
#pragma unroll
  for (int f = 0; f <= C; ++f) out[f * HW + p] = acc[f];
}

constexpr int kTensorRows = kTileRows;

// v_c = S_c / (S_ind > 0 ? S_ind : 1) once per pixel into a shared tile of
// (kTensorRows + 2) x (128 + 2) pixels, then np.gradient (central /2.0 inside,
// one-sided /1.0 at the frame edges) and J = sum_c (gx gx, gx gy, gy gy) * ind.
template <int C>
__global__ void k_ct_tensor(int H, int W, const double* __restrict__ S,
                            const uint8_t* __restrict__ labels, double* __restrict__ Q,
                            const uint8_t* __restrict__ tiles) {
  __shared__ double v[kTensorRows + 2][130][C];
  if (!tiles[blockIdx.y * gridDim.x + blockIdx.x]) return;
  const int64_t HW = (int64_t)H * W;
  const int i0 = blockIdx.x * 128, j0 = blockIdx.y * kTensorRows;
  for (int e = threadIdx.x; e < (kTensorRows + 2) * 130; e += blockDim.x) {
    const int r = e / 130, cc = e - r * 130;
    const int j = j0 + r - 1, i = i0 + cc - 1;
    if (j < 0 || j >= H || i < 0 || i >= W) continue;
    const int64_t p = (int64_t)j * W + i;
    const double m = S[p];
    const double safe = m > 0.0 ? m : 1.0;
#pragma unroll
    for (int c = 0; c < C; ++c) v[r][cc][c] = S[(int64_t)(c + 1) * HW + p] / safe;
  }
  __syncthreads();
  const int i = i0 + threadIdx.x;
  if (i >= W) return;
  const int cc = threadIdx.x + 1;
  for (int r = 1; r <= kTensorRows; ++r) {
    const int j = j0 + r - 1;
    if (j >= H) break;
    double J11 = 0.0, J12 = 0.0, J22 = 0.0;
#pragma unroll
    for (int c = 0; c < C; ++c) {
      double gy, gx;
      if (j == 0) gy = (v[r + 1][cc][c] - v[r][cc][c]) / 1.0;
      else if (j == H - 1) gy = (v[r][cc][c] - v[r - 1][cc][c]) / 1.0;
      else gy = (v[r + 1][cc][c] - v[r - 1][cc][c]) / 2.0;
      if (i == 0) gx = (v[r][cc + 1][c] - v[r][cc][c]) / 1.0;
      else if (i == W - 1) gx = (v[r][cc][c] - v[r][cc - 1][c]) / 1.0;
      else gx = (v[r][cc + 1][c] - v[r][cc - 1][c]) / 2.0;
      J11 += gx * gx;
      J12 += gx * gy;
      J22 += gy * gy;
    }
    const int64_t p = (int64_t)j * W + i;
    const double ind = labels[p] == 0 ? 1.0 : 0.0;
    Q[3 * HW + p] = ind;
    Q[p] = J11 * ind;
    Q[HW + p] = J12 * ind;
    Q[2 * HW + p] = J22 * ind;
  }
}

// The rho stage evaluated only at the queried pixels, in scipy's order: the
// axis-0 pass T(j, i') for the 2R+1 columns i' of the window (0 outside the
// frame: cval of the axis-1 pass), then the axis-1 pass over them.
__device__ __forceinline__ double ct_col(const double* P, int H, int W, int j, int i,
                                         const Taps& t) {
  if (i < 0 || i >= W) return 0.0;
  const double* x = P + (int64_t)j * W + i;
  double acc = x[0] * t.w[0];
  for (int k = t.R; k >= 1; --k) {
    const double a = j - k >= 0 ? x[-(int64_t)k * W] : 0.0;
    const double b = j + k < H ? x[(int64_t)k * W] : 0.0;
    acc += (a + b) * t.w[k];
  }
  return acc;
}

constexpr int kQueryWarps = 4;

// one warp per query: the 4 x (2R+1) column sums are spread over the lanes
// and parked in shared memory, lanes 0..3 then run the ordered row sums
__global__ void k_ct_query(int H, int W, int n, const int64_t* __restrict__ idx,
                           const double* __restrict__ Q, const Taps t, double lam,
                           double* __restrict__ g, double* __restrict__ eig) {
  __shared__ double cols[kQueryWarps][4][2 * kMaxTaps + 1];
  __shared__ double red[kQueryWarps][4];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int k = blockIdx.x * kQueryWarps + warp;
  if (k >= n) return;  // whole warp
  const int64_t HW = (int64_t)H * W;
  const int64_t p = idx[k];
  const int j = (int)(p / W), i = (int)(p % W);
  const int ncol = 2 * t.R + 1;
  for (int e = lane; e < 4 * ncol; e += 32) {
    const int plane = e / ncol, c = e - plane * ncol;
    cols[warp][plane][c] = ct_col(Q + plane * HW, H, W, j, i + c - t.R, t);
  }
  __syncwarp();
  if (lane < 4) {
    const double* T = cols[warp][lane] + t.R;
    double acc = T[0] * t.w[0];
    for (int d = t.R; d >= 1; --d) acc += (T[-d] + T[d]) * t.w[d];
    red[warp][lane] = acc;
  }
  __syncwarp();
  if (lane) return;
  const double J11 = red[warp][0], J12 = red[warp][1], J22 = red[warp][2], mass = red[warp][3];
  const double safe = mass > 0.0 ? mass : 1.0;
  const double a = J11 / safe, b = J12 / safe, c = J22 / safe;
  const double mean = (a + c) / 2.0;
  const double h = (a - c) / 2.0;
  const double disc = sqrt(h * h + b * b);
  const double phi = 0.5 * atan2_np(2.0 * b, a - c);
  const double lo = mean - disc, hi = mean + disc;
  const double coh = tanh_np((hi - lo) / lam);
  const double vx = -sin_np(phi), vy = cos_np(phi);
  if (eig) {  // guide.eigen_2x2's minor eigenvector and the coherence (make_spline),
              // the normalised tensor (structure_tensor) and the rho mass
    double* e = eig + 8 * k;
    e[0] = vx;
    e[1] = vy;
    e[2] = coh;
    e[3] = a;
    e[4] = b;
    e[5] = c;
    e[6] = mass;
    e[7] = 0.0;
  }
  if (!g) return;
  double gx = coh * vx, gy = coh * vy;
  if (mass <= 0.0) gx = gy = 0.0;
  g[2 * k] = gx;
  g[2 * k + 1] = gy;
}

__device__ __forceinline__ bool ct_active(const uint8_t* lab, int H, int W, int periodic, int j,
                                          int i) {
  if (lab[(int64_t)j * W + i] != 255) return false;
  for (int dj = -1; dj <= 1; ++dj)
    for (int di = -1; di <= 1; ++di) {
      if (!di && !dj) continue;
      int ii = i + di;
      const int jj = j + dj;
      if (periodic) ii = (ii % W + W) % W;
      if (ii >= 0 && ii < W && jj >= 0 && jj < H && lab[(int64_t)jj * W + ii] == 0) return true;
    }
  return false;
}

// tracker._update_arrays (tracker.py:59-79) as a byte map: survivors and the
// Inpaint 8-neighbours of filled pixels are candidates (mark >= 1); mark = 2
// when the candidate passes _active_filter (Inpaint with a Readable neighbour).
// Every writer of a pixel stores the same value.
__global__ void k_ct_mark(int H, int W, int periodic, const uint8_t* __restrict__ lab, int n,
                          const int64_t* __restrict__ frontier, const uint8_t* __restrict__ fill,
                          uint8_t* __restrict__ mark) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= n) return;
  const int64_t p = frontier[k];
  const int j = (int)(p / W), i = (int)(p % W);
  if (!fill[k]) {
    mark[p] = 1 + ct_active(lab, H, W, periodic, j, i);
    return;
  }
  for (int dj = -1; dj <= 1; ++dj)
    for (int di = -1; di <= 1; ++di) {
      if (!di && !dj) continue;
      int ii = i + di;
      const int jj = j + dj;
      if (periodic) ii = (ii % W + W) % W;
      if (ii < 0 || ii >= W || jj < 0 || jj >= H) continue;
      const int64_t q = (int64_t)jj * W + ii;
      if (lab[q] == 255) mark[q] = 1 + ct_active(lab, H, W, periodic, jj, ii);
    }
}


// engine.py:317-356 for one shell: ready predicate (onion / conf > c /
// (|g| > c2) & (conf > c)), fill = ready & (rw > 0), then the scatter and
// relabel of the filled pixels.
__global__ void k_ct_commit(int C, int n, const int64_t* __restrict__ frontier,
                            const double* __restrict__ rw, const double* __restrict__ tw,
                            const double* __restrict__ vals, const double* __restrict__ g,
                            int ready_mode, double c, double c2, int shell, double* __restrict__ u,
                            uint8_t* __restrict__ lab, int32_t* __restrict__ fillshell,
                            uint8_t* __restrict__ fill, int32_t* __restrict__ count) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  bool f = false;
  if (k < n) {
    const double conf = rw[k] / tw[k];
    bool ready = true;
    if (ready_mode == 1) ready = conf > c;
    else if (ready_mode == 2) ready = hypot_np(g[2 * k], g[2 * k + 1]) > c2 && conf > c;
    f = ready && rw[k] > 0.0;
    fill[k] = f ? 1 : 0;
    if (f) {
      const int64_t p = frontier[k];
      for (int ch = 0; ch < C; ++ch) u[p * C + ch] = vals[(int64_t)k * C + ch];
      lab[p] = 0;
      fillshell[p] = shell;
    }
  }
  const unsigned b = __ballot_sync(0xffffffffu, f);
  if ((threadIdx.x & 31) == 0 && b) atomicAdd(count, __popc(b));
}

}  // namespace

}  // namespace gf

using namespace gf;

extern "C" size_t gf_coherence_workspace_bytes(int32_t height, int32_t width, int32_t channels) {
  if (height <= 0 || width <= 0 || channels < 1) return 0;
  const size_t planes = (size_t)(channels + 1 > 4 ? channels + 1 : 4);
  const size_t tiles = (size_t)((width + 127) / 128) * ((height + kTileRows - 1) / kTileRows);
  return 2 * planes * (size_t)height * width * sizeof(double) + tiles;
}

static int coherence_run(int32_t height, int32_t width, int32_t channels, const double* image,
                         const uint8_t* labels, int32_t n, const int64_t* idx, double sigma,
                         double rho, double lam, double* g, double* eig, double* points,
                         void* workspace, size_t workspace_bytes, void* stream);

extern "C" int gf_coherence_directions(int32_t height, int32_t width, int32_t channels,
                                       const double* image, const uint8_t* labels, int32_t n,
                                       const int64_t* idx, double sigma, double rho, double lam,
                                       double* g, double* points, void* workspace,
                                       size_t workspace_bytes, void* stream) {
  if (n > 0 && !g) return set_error(GF_E_INVALID, "NULL buffer");
  return coherence_run(height, width, channels, image, labels, n, idx, sigma, rho, lam, g, nullptr,
                       points, workspace, workspace_bytes, stream);
}

extern "C" int gf_structure_eigen(int32_t height, int32_t width, int32_t channels,
                                  const double* image, const uint8_t* labels, int32_t n,
                                  const int64_t* idx, double sigma, double rho, double lam,
                                  double* eig, void* workspace, size_t workspace_bytes,
                                  void* stream) {
  if (n > 0 && !eig) return set_error(GF_E_INVALID, "NULL buffer");
  return coherence_run(height, width, channels, image, labels, n, idx, sigma, rho, lam, nullptr,
                       eig, nullptr, workspace, workspace_bytes, stream);
}

static int coherence_run(int32_t height, int32_t width, int32_t channels, const double* image,
                         const uint8_t* labels, int32_t n, const int64_t* idx, double sigma,
                         double rho, double lam, double* g, double* eig, double* points,
                         void* workspace, size_t workspace_bytes, void* stream) {
  if (height < 2 || width < 2 || height > 65535 || channels < 1 || channels > 4 || n < 0)
    return set_error(GF_E_INVALID, "bad geometry");
  if (!image || !labels || (n > 0 && !idx) || !workspace)
    return set_error(GF_E_INVALID, "NULL buffer");
  if (workspace_bytes < gf_coherence_workspace_bytes(height, width, channels))
    return set_error(GF_E_WORKSPACE, "workspace too small");
  Taps ts, tr;
  if (make_taps(sigma, ts) != GF_OK || make_taps(rho, tr) != GF_OK)
    return set_error(GF_E_UNSUPPORTED, "sigma / rho window outside 1..64 taps");
  if (n == 0) return GF_OK;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const int64_t HW = (int64_t)height * width;
  const int planes = channels + 1 > 4 ? channels + 1 : 4;
  double* A = static_cast<double*>(workspace);
  double* B = A + (size_t)planes * HW;
  const int tiles_x = (width + 127) / 128, tiles_y = (height + kTileRows - 1) / kTileRows;
  uint8_t* tmask = reinterpret_cast<uint8_t*>(B + (size_t)planes * HW);
  cudaMemsetAsync(tmask, 0, (size_t)tiles_x * tiles_y, s);
  k_ct_tiles<<<(n + 127) / 128, 128, 0, s>>>(height, width, n, idx, tr.R + ts.R + 1, tiles_x,
                                            tmask, points);
  // sigma stage (seed fused into axis 0): B = axis 0, A = axis 1 (S)
  const dim3 blk(128);
  const dim3 rows((width + 127) / 128, height, 1);
  switch (channels) {
    case 1: k_ct_seed_smooth0<1><<<rows, blk, 0, s>>>(height, width, ts, image, labels, B, tmask, tiles_x); break;
    case 2: k_ct_seed_smooth0<2><<<rows, blk, 0, s>>>(height, width, ts, image, labels, B, tmask, tiles_x); break;
    case 3: k_ct_seed_smooth0<3><<<rows, blk, 0, s>>>(height, width, ts, image, labels, B, tmask, tiles_x); break;
    default: k_ct_seed_smooth0<4><<<rows, blk, 0, s>>>(height, width, ts, image, labels, B, tmask, tiles_x); break;
  }
  k_ct_smooth1<<<dim3(rows.x, height, channels + 1), blk, 0, s>>>(height, width, ts, B, A, tmask,
                                                                 tiles_x);
  // tensor: B = [J11, J12, J22, ind] (J * ind)
  const dim3 tiles(tiles_x, tiles_y, 1);
  switch (channels) {
    case 1: k_ct_tensor<1><<<tiles, blk, 0, s>>>(height, width, A, labels, B, tmask); break;
    case 2: k_ct_tensor<2><<<tiles, blk, 0, s>>>(height, width, A, labels, B, tmask); break;
    case 3: k_ct_tensor<3><<<tiles, blk, 0, s>>>(height, width, A, labels, B, tmask); break;
    default: k_ct_tensor<4><<<tiles, blk, 0, s>>>(height, width, A, labels, B, tmask); break;
  }
  // rho stage at the queries only
  k_ct_query<<<(n + kQueryWarps - 1) / kQueryWarps, 32 * kQueryWarps, 0, s>>>(height, width, n,
                                                                            idx, B, tr, lam, g, eig);
  count_launches(5);
  cudaError_t e = cudaPeekAtLastError();
  if (e != cudaSuccess) return set_error(GF_E_CUDA, cudaGetErrorString(e));
  return GF_OK;
}

extern "C" int gf_frontier_candidates(int32_t height, int32_t width, const uint8_t* labels,
                                      int32_t periodic_x, int32_t n, const int64_t* frontier,
                                      const uint8_t* fill, uint8_t* mark, void* stream) {
  if (height <= 0 || width <= 0 || n < 0) return set_error(GF_E_INVALID, "bad geometry");
  if (n == 0) return GF_OK;
  if (!labels || !frontier || !fill || !mark) return set_error(GF_E_INVALID, "NULL buffer");
  k_ct_mark<<<(n + 127) / 128, 128, 0, static_cast<cudaStream_t>(stream)>>>(
      height, width, periodic_x, labels, n, frontier, fill, mark);
  count_launches(1);
  cudaError_t e = cudaPeekAtLastError();
  if (e != cudaSuccess) return set_error(GF_E_CUDA, cudaGetErrorString(e));
  return GF_OK;
}

extern "C" int gf_commit_shell(int32_t channels, int32_t n, const int64_t* frontier,
                               const double* rw, const double* tw, const double* vals,
                               const double* g, int32_t ready_mode, double c, double c2,
                               int32_t shell, double* image, uint8_t* labels, int32_t* fillshell,
                               uint8_t* fill, int32_t* count, void* stream) {
  if (channels < 1 || channels > 4 || n < 0 || ready_mode < 0 || ready_mode > 2)
    return set_error(GF_E_INVALID, "bad arguments");
  if (n == 0) return GF_OK;
  if (!frontier || !rw || !tw || !vals || !image || !labels || !fillshell || !fill || !count ||
      (ready_mode == 2 && !g))
    return set_error(GF_E_INVALID, "NULL buffer");
  k_ct_commit<<<(n + 127) / 128, 128, 0, static_cast<cudaStream_t>(stream)>>>(
      channels, n, frontier, rw, tw, vals, g, ready_mode, c, c2, shell, image, labels, fillshell,
      fill, count);
  count_launches(1);
  cudaError_t e = cudaPeekAtLastError();
  if (e != cudaSuccess) return set_error(GF_E_CUDA, cudaGetErrorString(e));
  return GF_OK;
}

namespace gf {
// The coherence transcendentals on the device, element-wise (test hook for
// gf_npmath.cuh against numpy; the query kernel inlines the same functions).
__global__ void k_npmath(int op, int64_t n, const double* __restrict__ a,
                         const double* __restrict__ b, double* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const double x = a[i];
    out[i] = op == 0 ? atan2_np(x, b[i]) : op == 1 ? tanh_np(x) : op == 2 ? sin_np(x) : cos_np(x);
  }
}
}  // namespace gf

extern "C" int gf_npmath_eval(int32_t op, int64_t n, const double* a, const double* b,
                              double* out, void* stream) {
  if (op < 0 || op > 3 || n < 0) return set_error(GF_E_INVALID, "bad op / n");
  if (n == 0) return GF_OK;
  if (!a || !out || (op == 0 && !b)) return set_error(GF_E_INVALID, "NULL buffer");
  const int64_t blocks = std::min<int64_t>((n + 255) / 256, 148 * 16);
  k_npmath<<<(int)blocks, 256, 0, static_cast<cudaStream_t>(stream)>>>(op, n, a, b, out);
  count_launches(1);
  cudaError_t e = cudaPeekAtLastError();
  if (e != cudaSuccess) return set_error(GF_E_CUDA, cudaGetErrorString(e));
  return GF_OK;
}

// ---------------------------------------------------------------------------
// The whole coherence-transport fill as ONE persistent cooperative kernel
// (engine._fill_loop, engine.py:286-376, with g from guide.coherence_directions,
// guide.py:330-355).  Per shell s, separated by grid-wide barriers:
//   B  one warp per query: the rho stage at the query (scipy order) -> g,
//      then 4 queries per warp through the ball sampler (eval_item, exact
//      einsum-order values) -> rw, tw, vals of the frontier entry
//   C  ready predicate (onion / conf > c / |g| > c2 & conf > c) -> fill flags
//   D  (only when nothing is ready) the deadlock pick: first maximal
//      confidence (NaN first, ties to the lowest pixel index = numpy's
//      argmax over the sorted frontier), its average or the 8-neighbour mean
//   E  commit: scatter the values, relabel, fillshell; every 32 x 8 tile
//      within sigma_R + 1 of a filled pixel is queued as dirty
//   A+F  the dirty tiles' tensor field is recomputed from u / labels (seed,
//      both sigma passes and the gradient tensor fused in shared memory: the
//      field elsewhere is unchanged, so the planes stay exact), and the
//      frontier is updated (tracker._update_arrays: survivors and Inpaint
//      8-neighbours of filled pixels, deduplicated by a per-pixel shell stamp,
//      active filter; or the full active rescan when untracked)
// The frontier is kept unsorted: only the deadlock argmax depends on its
// order, and that is resolved by pixel index.  Per-shell counters live in
// two parity banks so one bank can be reset while the other is in use.
// ---------------------------------------------------------------------------
namespace gf {
namespace {

constexpr int kLoopThreads = 256;
#ifndef GF_CT_MIN_BLOCKS
#define GF_CT_MIN_BLOCKS 2  // 2 x 256 threads per SM (3 spills and runs slower)
#endif
constexpr int kLTW = 16, kLTH = 16;  // tensor tile: 16 x 16 pixels
constexpr int kLoopRsMax = 6;       // sigma window radius the fused tile supports
static_assert(kLTW * kLTH == kLoopThreads, "one J output per thread");

enum CtCounter {
  kCtNF = 0,      // [2] next-frontier appends
  kCtFill = 2,    // [2] fills
  kCtCand = 4,    // [2] tracker candidates
  kCtAnyG = 6,    // [2] any |g| > 0 (data term)
  kCtTiles = 8,   // [2] dirty tiles queued (tile list length)
  kCtDone = 10,   // 2: unfillable, 3: rows capacity exceeded
  kCtIters = 11,
  kCtDeadlocks = 12,
  kCtFilled = 13,
  kCtInpaint = 14,  // Inpaint pixels at the start
  kCtGrab = 16,     // [2] next tile-list entry to take
  kCtCount = 20     // then two u64 hull keys (min, max) at ctr + kCtCount
};

struct CtLoopArgs {
  int H, W, C, periodic, tracked, order;
  double c, c2;
  double lam;
  int tiles_x, tiles_y;
  int rows_cap;
  long long capacity;      // frontier entry capacity (>= Inpaint pixels)
  double* u;
  uint8_t* lab;
  double* Q;              // [J11, J12, J22] * ind, ind
  int* fr[2];             // frontier lists (pixel indices), shell s in fr[s & 1]
  double* eg;             // per frontier entry: g (2), rw, tw, vals (C), fill flag
  double* erw;
  double* etw;
  double* evals;
  uint8_t* efill;
  int* stamp;             // tracker dedup: last shell + 1 that claimed the pixel
  unsigned* tflag;        // tile queued for recomputation (cleared when recomputed)
  int* tlist;             // queued tiles, taken in order by whichever block is free
  int* fillshell;
  int* enter;             // or nullptr
  long long* rows;        // [rows_cap][5]
  int* ctr;
  double* slot_c;         // deadlock argmax partials, one per block
  int* slot_k;
  unsigned long long* trace;  // GF_CT_TRACE: %globaltimer at the phase barriers, or nullptr
  Taps ts, tr;
};

__device__ __forceinline__ unsigned long long ct_now() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
// phase stamp (block 0, thread 0): slot 0 = init done, then 12 per shell
// (0..5 barriers, 6 tiles, 7 F, 8 / 9 block 0's own B / E work done,
// 10 / 11 the last block's B / E work done)
__device__ __forceinline__ void ct_trace_work(const CtLoopArgs& A, int s, int own, int last) {
  if (!A.trace || s >= 4096) return;
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned long long t = ct_now();
    if (blockIdx.x == 0) A.trace[1 + 16 * s + own] = t;
    atomicMax(&A.trace[1 + 16 * s + last], t);
  }
}
__device__ __forceinline__ void ct_trace(const CtLoopArgs& A, int s, int ph) {
  if (A.trace && blockIdx.x == 0 && threadIdx.x == 0 && s < 4096) A.trace[1 + 16 * s + ph] = ct_now();
}

__device__ __forceinline__ int ld_cg(const int* p) { return *(const volatile int*)p; }

// order-preserving u64 key of a double (atomicMin / atomicMax of the hull)
__device__ __forceinline__ unsigned long long ct_key(double x) {
  const unsigned long long u = (unsigned long long)__double_as_longlong(x);
  return (u >> 63) ? ~u : (u | 0x8000000000000000ULL);
}
__device__ __forceinline__ double ct_unkey(unsigned long long k) {
  return __longlong_as_double((long long)((k >> 63) ? (k & 0x7fffffffffffffffULL) : ~k));
}

// warp-aggregated append: every lane of the warp calls it (full mask); lanes
// with pred get consecutive slots of list from one atomicAdd on *count
__device__ __forceinline__ void warp_append(bool pred, int value, int* count, int* list) {
  const int lane = threadIdx.x & 31;
  const unsigned m = __ballot_sync(0xffffffffu, pred);
  int base = 0;
  if (lane == 0 && m) base = atomicAdd(count, __popc(m));
  base = __shfl_sync(0xffffffffu, base, 0);
  if (pred) list[base + __popc(m & ((1u << lane) - 1u))] = value;
}

// a grid-wide counter read once per block and broadcast through shared
// memory (75k threads polling one L2 line serialise for microseconds);
// block-uniform call sites only
__device__ __forceinline__ int block_ld(const int* p) {
  __shared__ int v;
  __syncthreads();
  if (threadIdx.x == 0) v = ld_cg(p);
  __syncthreads();
  return v;
}

// NEIGHBOR_OFFSETS (grid.py:29-33) as (di, dj) packed in 2-bit fields
__device__ __forceinline__ int ct_nb_di(int o) { return (int)((0x9224u >> (2 * o)) & 3u) - 1; }
__device__ __forceinline__ int ct_nb_dj(int o) { return (int)((0xA940u >> (2 * o)) & 3u) - 1; }

// numpy argmax order on (conf, pixel): NaN first, then larger, ties to the
// lower pixel index (the reference's frontier is sorted)
__device__ __forceinline__ bool ct_better(double a, int pa, double b, int pb) {
  const bool na = a != a, nb = b != b;
  if (na != nb) return na;
  if (!na && a != b) return a > b;
  return pa < pb;
}

// The tensor field of one 32 x 8 tile from u / labels (the sigma radius R a
// compile-time constant so every tap is unrolled): seed (ind, ind * u_c, 0
// outside the frame), scipy's axis-0 then axis-1 pass, v = S_c / safe(S_ind),
// np.gradient and J * ind -- written as one 32-byte record per pixel
// Q[p] = (J11 ind, J12 ind, J22 ind, ind).
template <int C, int R>
__device__ void ct_loop_tile_r(const CtLoopArgs& A, int t, double* sm) {
  const int H = A.H, W = A.W;
  const int tx = t % A.tiles_x, ty = t / A.tiles_x;
  const int i0 = tx * kLTW, j0 = ty * kLTH;
  constexpr int SR = kLTH + 2 + 2 * R, SC = kLTW + 2 + 2 * R, BR = kLTH + 2, VC = kLTW + 2;
  double* seed = sm;                       // [C + 1][SR][SC]
  double* Bv = seed + (C + 1) * SR * SC;   // [C + 1][BR][SC]: sigma axis-0 pass
  double* V = Bv + (C + 1) * BR * SC;      // [C][BR][VC]: S_c / safe(S_ind)
  double w[R + 1];
#pragma unroll
  for (int k = 0; k <= R; ++k) w[k] = A.ts.w[k];
  constexpr int kSeedIt = (SR * SC + kLoopThreads - 1) / kLoopThreads;
#pragma unroll
  for (int it = 0; it < kSeedIt; ++it) {
    const int e = threadIdx.x + it * kLoopThreads;
    if (e >= SR * SC) break;
    const int r = e / SC, cc = e - r * SC;
    const int j = j0 - 1 - R + r, i = i0 - 1 - R + cc;
    double ind = 0.0, uc[C];
#pragma unroll
    for (int f = 0; f < C; ++f) uc[f] = 0.0;
    if (j >= 0 && j < H && i >= 0 && i < W) {
      const int64_t p = (int64_t)j * W + i;
      double uv[C];
#pragma unroll
      for (int f = 0; f < C; ++f) uv[f] = A.u[p * C + f];
      ind = A.lab[p] == 0 ? 1.0 : 0.0;
#pragma unroll
      for (int f = 0; f < C; ++f) uc[f] = ind * uv[f];
    }
    seed[e] = ind;
#pragma unroll
    for (int f = 0; f < C; ++f) seed[(f + 1) * SR * SC + e] = uc[f];
  }
  __syncthreads();
  for (int e = threadIdx.x; e < BR * SC; e += blockDim.x) {
    const int r = e / SC, cc = e - r * SC;
#pragma unroll
    for (int f = 0; f <= C; ++f) {
      const double* sp = seed + f * SR * SC + (r + R) * SC + cc;
      double acc = sp[0] * w[0];
#pragma unroll
      for (int k = R; k >= 1; --k) acc += (sp[-k * SC] + sp[k * SC]) * w[k];
      Bv[f * BR * SC + e] = acc;
    }
  }
  __syncthreads();
  for (int e = threadIdx.x; e < BR * VC; e += blockDim.x) {
    const int r = e / VC, cc = e - r * VC;
    const int i = i0 - 1 + cc;
    double S[C + 1];
#pragma unroll
    for (int f = 0; f <= C; ++f) {
      const double* b = Bv + f * BR * SC + r * SC + cc + R;
      double acc = b[0] * w[0];
#pragma unroll
      for (int k = R; k >= 1; --k) {
        const double a = i - k >= 0 ? b[-k] : 0.0;
        const double bb = i + k < W ? b[k] : 0.0;
        acc += (a + bb) * w[k];
      }
      S[f] = acc;
    }
    const double safe = S[0] > 0.0 ? S[0] : 1.0;
#pragma unroll
    for (int f = 0; f < C; ++f) V[f * BR * VC + e] = S[f + 1] / safe;
  }
  __syncthreads();
  {
    const int e = threadIdx.x;  // kLTH * kLTW == kLoopThreads
    const int r = e / kLTW, cc = e - r * kLTW;
    const int j = j0 + r, i = i0 + cc;
    if (j < H && i < W) {
      const int vr = r + 1, vc = cc + 1;
      double J11 = 0.0, J12 = 0.0, J22 = 0.0;
#pragma unroll
      for (int f = 0; f < C; ++f) {
        const double* v = V + f * BR * VC;
        double gy, gx;
        if (j == 0) gy = (v[(vr + 1) * VC + vc] - v[vr * VC + vc]) / 1.0;
        else if (j == H - 1) gy = (v[vr * VC + vc] - v[(vr - 1) * VC + vc]) / 1.0;
        else gy = (v[(vr + 1) * VC + vc] - v[(vr - 1) * VC + vc]) / 2.0;
        if (i == 0) gx = (v[vr * VC + vc + 1] - v[vr * VC + vc]) / 1.0;
        else if (i == W - 1) gx = (v[vr * VC + vc] - v[vr * VC + vc - 1]) / 1.0;
        else gx = (v[vr * VC + vc + 1] - v[vr * VC + vc - 1]) / 2.0;
        J11 += gx * gx;
        J12 += gx * gy;
        J22 += gy * gy;
      }
      const int64_t p = (int64_t)j * W + i;
      const double ind = A.lab[p] == 0 ? 1.0 : 0.0;
      double2* q = reinterpret_cast<double2*>(A.Q + 4 * p);
      q[0] = make_double2(J11 * ind, J12 * ind);
      q[1] = make_double2(J22 * ind, ind);
    }
  }
  __syncthreads();
}

template <int C>
__device__ __forceinline__ void ct_loop_tile(const CtLoopArgs& A, int t, double* sm) {
  switch (A.ts.R) {
    case 1: ct_loop_tile_r<C, 1>(A, t, sm); break;
    case 2: ct_loop_tile_r<C, 2>(A, t, sm); break;
    case 3: ct_loop_tile_r<C, 3>(A, t, sm); break;
    case 4: ct_loop_tile_r<C, 4>(A, t, sm); break;
    case 5: ct_loop_tile_r<C, 5>(A, t, sm); break;
    default: ct_loop_tile_r<C, kLoopRsMax>(A, t, sm); break;
  }
}

// flag every tile within d of pixel (j, i) (idempotent plain stores; the
// initial scan only -- compacted into the list by ct_list_flags)
__device__ __forceinline__ void ct_mark_tiles(const CtLoopArgs& A, int j, int i, int d) {
  const int ty0 = max(0, j - d) / kLTH, ty1 = min(A.H - 1, j + d) / kLTH;
  const int tx0 = max(0, i - d) / kLTW, tx1 = min(A.W - 1, i + d) / kLTW;
  for (int ty = ty0; ty <= ty1; ++ty)
    for (int tx = tx0; tx <= tx1; ++tx) A.tflag[ty * A.tiles_x + tx] = 1u;
}

// every flagged tile into the list (block b scans tiles b, b + grid, ...)
__device__ __forceinline__ void ct_list_flags(const CtLoopArgs& A, int bank) {
  const int ntiles = A.tiles_x * A.tiles_y;
  const int per = (ntiles + gridDim.x - 1) / gridDim.x;
  for (int m0 = 0; m0 < per; m0 += blockDim.x) {
    const int t = blockIdx.x + (m0 + threadIdx.x) * gridDim.x;
    const bool q = m0 + (int)threadIdx.x < per && t < ntiles && A.tflag[t] != 0u;
    warp_append(q, t, &A.ctr[kCtTiles + bank], A.tlist);
  }
}

// queue the tiles within d of a filled pixel (warp-uniform: every lane calls,
// f = this lane filled a pixel at (j, i)); a tile is listed once
constexpr int kQueueRows = (2 * (kLoopRsMax + 1)) / kLTH + 2;
constexpr int kQueueCols = (2 * (kLoopRsMax + 1)) / kLTW + 2;
__device__ __forceinline__ void ct_queue_tiles(const CtLoopArgs& A, int bank, bool f, int j, int i,
                                               int d) {
  const int ty0 = max(0, j - d) / kLTH, ty1 = min(A.H - 1, j + d) / kLTH;
  const int tx0 = max(0, i - d) / kLTW, tx1 = min(A.W - 1, i + d) / kLTW;
  bool fresh[kQueueRows * kQueueCols];
  int tt[kQueueRows * kQueueCols];
#pragma unroll
  for (int a = 0; a < kQueueRows; ++a)
#pragma unroll
    for (int c = 0; c < kQueueCols; ++c) {
      const int ty = ty0 + a, tx = tx0 + c;
      const int t = ty * A.tiles_x + tx;
      tt[a * kQueueCols + c] = t;
      fresh[a * kQueueCols + c] = f && ty <= ty1 && tx <= tx1 && atomicExch(&A.tflag[t], 1u) == 0u;
    }
  // one atomicAdd per warp for all of its lanes' fresh tiles
  const int lane = threadIdx.x & 31;
  int mine = 0;
#pragma unroll
  for (int e = 0; e < kQueueRows * kQueueCols; ++e) mine += fresh[e] ? 1 : 0;
  int incl = mine;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int v = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += v;
  }
  const int total = __shfl_sync(0xffffffffu, incl, 31);
  int base = 0;
  if (lane == 0 && total) base = atomicAdd(&A.ctr[kCtTiles + bank], total);
  base = __shfl_sync(0xffffffffu, base, 0) + incl - mine;
#pragma unroll
  for (int e = 0; e < kQueueRows * kQueueCols; ++e)
    if (fresh[e]) A.tlist[base++] = tt[e];
}

// ct_queue_tiles for one thread (the guarded pixel)
__device__ __forceinline__ void ct_queue_tiles_one(const CtLoopArgs& A, int bank, int j, int i,
                                                   int d) {
  const int ty0 = max(0, j - d) / kLTH, ty1 = min(A.H - 1, j + d) / kLTH;
  const int tx0 = max(0, i - d) / kLTW, tx1 = min(A.W - 1, i + d) / kLTW;
  for (int ty = ty0; ty <= ty1; ++ty)
    for (int tx = tx0; tx <= tx1; ++tx) {
      const int t = ty * A.tiles_x + tx;
      if (atomicExch(&A.tflag[t], 1u) == 0u) A.tlist[atomicAdd(&A.ctr[kCtTiles + bank], 1)] = t;
    }
}

// recompute the listed tiles; blocks take the next entry as they free up
template <int C>
__device__ __forceinline__ void ct_run_tiles(const CtLoopArgs& A, int bank, double* sm) {
  __shared__ int s_idx;
  const int n = block_ld(&A.ctr[kCtTiles + bank]);
  for (;;) {
    __syncthreads();
    if (threadIdx.x == 0) s_idx = atomicAdd(&A.ctr[kCtGrab + bank], 1);
    __syncthreads();
    const int idx = s_idx;
    if (idx >= n) break;
    const int t = A.tlist[idx];
    if (threadIdx.x == 0) A.tflag[t] = 0u;
    ct_loop_tile<C>(A, t, sm);
  }
}

// rho stage axis-0 sums at column i, row j, for two planes of the AoS field
// (pl = 0: J11, J12; pl = 1: J22, ind), every tap load issued up front
constexpr int kColUnroll = 8;
__device__ __forceinline__ double2 ct_col2(const double* Q, int H, int W, int j, int i, int pl,
                                           const Taps& t) {
  if (i < 0 || i >= W) return make_double2(0.0, 0.0);
  const int R = t.R;
  const double2* x = reinterpret_cast<const double2*>(Q + 4 * ((int64_t)j * W + i)) + pl;
  const int64_t st = 2 * (int64_t)W;  // one row in double2
  if (R > kColUnroll) {
    double2 acc = x[0];
    acc.x *= t.w[0];
    acc.y *= t.w[0];
    for (int k = R; k >= 1; --k) {
      const double2 a = j - k >= 0 ? x[-k * st] : make_double2(0.0, 0.0);
      const double2 b = j + k < H ? x[k * st] : make_double2(0.0, 0.0);
      acc.x += (a.x + b.x) * t.w[k];
      acc.y += (a.y + b.y) * t.w[k];
    }
    return acc;
  }
  double2 a[kColUnroll + 1], b[kColUnroll + 1];
#pragma unroll
  for (int k = 1; k <= kColUnroll; ++k) {
    a[k] = (k <= R && j - k >= 0) ? x[-k * st] : make_double2(0.0, 0.0);
    b[k] = (k <= R && j + k < H) ? x[k * st] : make_double2(0.0, 0.0);
  }
  const double2 c0 = x[0];
  double2 acc = make_double2(c0.x * t.w[0], c0.y * t.w[0]);
#pragma unroll
  for (int k = kColUnroll; k >= 1; --k)
    if (k <= R) {
      acc.x += (a[k].x + b[k].x) * t.w[k];
      acc.y += (a[k].y + b[k].y) * t.w[k];
    }
  return acc;
}

// g for up to 4 queries at once (guide.coherence_directions): the 4 x 4
// planes x (2R+1) column sums are spread over the warp, 16 lanes run the
// ordered row sums, and lane group q (lanes 8q .. 8q+7) gets query q's g
__device__ __forceinline__ void ct_loop_g4(const CtLoopArgs& A, const int* pix, int nq,
                                           double* cols, double& gx, double& gy) {
  const int lane = threadIdx.x & 31;
  const int H = A.H, W = A.W;
  const int R = A.tr.R, ncol = 2 * R + 1;
  const int total = nq * 2 * ncol;  // (query, plane pair, column)
  for (int e = lane; e < total; e += 32) {
    const int q = e / (2 * ncol), rem = e - q * 2 * ncol;
    const int pl = rem / ncol, c = rem - pl * ncol;
    const int p = pix[q];
    const int j = p / W, i = p - j * W;
    const double2 v = ct_col2(A.Q, H, W, j, i + c - R, pl, A.tr);
    cols[(q * 4 + 2 * pl) * ncol + c] = v.x;
    cols[(q * 4 + 2 * pl + 1) * ncol + c] = v.y;
  }
  __syncwarp();
  double red = 0.0;
  if (lane < 4 * nq) {
    const double* T = cols + lane * ncol + R;
    double acc = T[0] * A.tr.w[0];
    for (int d = R; d >= 1; --d) acc += (T[-d] + T[d]) * A.tr.w[d];
    red = acc;
  }
  const int g0 = (lane >> 3) * 4;
  const double J11 = __shfl_sync(0xffffffffu, red, g0), J12 = __shfl_sync(0xffffffffu, red, g0 + 1);
  const double J22 = __shfl_sync(0xffffffffu, red, g0 + 2);
  const double mass = __shfl_sync(0xffffffffu, red, g0 + 3);
  __syncwarp();
  const double safe = mass > 0.0 ? mass : 1.0;
  const double a = J11 / safe, b = J12 / safe, c = J22 / safe;
  const double mean = (a + c) / 2.0;
  const double h = (a - c) / 2.0;
  const double disc = sqrt(h * h + b * b);
  const double phi = 0.5 * atan2_np(2.0 * b, a - c);
  const double lo = mean - disc, hi = mean + disc;
  const double coh = tanh_np((hi - lo) / A.lam);
  const double vx = -sin_np(phi), vy = cos_np(phi);
  gx = coh * vx;
  gy = coh * vy;
  if (mass <= 0.0) gx = gy = 0.0;
}

__device__ __forceinline__ bool ct_loop_active(const CtLoopArgs& A, int p) {
  const int j = p / A.W, i = p - j * A.W;
  return ct_active(A.lab, A.H, A.W, A.periodic, j, i);
}

template <int C, int NL>
__global__ void __launch_bounds__(kLoopThreads, GF_CT_MIN_BLOCKS)
    k_ct_loop(const __grid_constant__ CtLoopArgs A, const __grid_constant__ BallParams P,
              const __grid_constant__ BallTables tab) {
  extern __shared__ __align__(16) unsigned char smraw[];
  BallTables& T = *reinterpret_cast<BallTables*>(smraw);
  double* tdist = reinterpret_cast<double*>(smraw + ((sizeof(BallTables) + 15) & ~size_t(15)));
  double* sm = tdist + kMaxK;
  for (int k = threadIdx.x; k < P.K; k += blockDim.x) {
    T.n[k] = tab.n[k];
    T.m[k] = tab.m[k];
    T.w0[k] = tab.w0[k];
    T.ni[k] = tab.ni[k];
    T.mi[k] = tab.mi[k];
    tdist[k] = hypot_np(tab.n[k], tab.m[k]);  // the axis ball's sample distances
  }
  __syncthreads();
  if (A.trace && blockIdx.x == 0 && threadIdx.x == 0) A.trace[4095 * 16 + 2] = ct_now();
  cg::grid_group grid = cg::this_grid();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int wpb = blockDim.x >> 5;
  const int gwarp = blockIdx.x * wpb + warp, nwarps = gridDim.x * wpb;
  const int gtid = blockIdx.x * blockDim.x + threadIdx.x, nthreads = gridDim.x * blockDim.x;
  const int H = A.H, W = A.W;
  const int HW = H * W;
  int* ctr = A.ctr;
  const RawSource src{A.u, A.lab, H, W, C};
  const int dq = A.tr.R;          // a query reads the field within rho_R
  const int dd = A.ts.R + 1;      // a filled pixel changes the field within sigma_R + 1

  // initial frontier (engine.py:298: active boundary, fr[0], counted in bank 1)
  // and the field around every Inpaint pixel (all a query can ever read)
  // and the Inpaint count and the readable hull (engine.py:289-296)
  unsigned long long* hull = reinterpret_cast<unsigned long long*>(ctr + kCtCount);
  {
    int n_inp = 0;
    double lo = INFINITY, hi = -INFINITY;
    // 4 x 32 consecutive pixels per warp step: the labels and the colours of
    // all four rounds are loaded before any is used
    constexpr int kScan = 4;
    for (int p0 = gwarp * 32 * kScan; p0 < HW; p0 += nwarps * 32 * kScan) {
      uint8_t l[kScan];
      double v[kScan][C];
#pragma unroll
      for (int q = 0; q < kScan; ++q) {
        const int p = p0 + 32 * q + lane;
        l[q] = p < HW ? A.lab[p] : 128;
#pragma unroll
        for (int c = 0; c < C; ++c) v[q][c] = p < HW ? A.u[(int64_t)p * C + c] : 0.0;
      }
#pragma unroll
      for (int q = 0; q < kScan; ++q) {
        const int p = p0 + 32 * q + lane;
        bool act = false;
        if (p < HW) {
          A.fillshell[p] = -1;
          if (l[q] == 255) {
            ++n_inp;
            const int j = p / W, i = p - j * W;
            ct_mark_tiles(A, j, i, dq);
            act = ct_active(A.lab, H, W, A.periodic, j, i);
          } else if (l[q] == 0) {
#pragma unroll
            for (int c = 0; c < C; ++c) {
              lo = fmin(lo, v[q][c]);
              hi = fmax(hi, v[q][c]);
            }
          }
          if (A.enter) A.enter[p] = act ? 0 : -1;
        }
        warp_append(act, p, &ctr[kCtNF + 1], A.fr[0]);
      }
    }
    __shared__ int s_n;
    __shared__ unsigned long long s_lo, s_hi;
    if (threadIdx.x == 0) {
      s_n = 0;
      s_lo = ~0ULL;
      s_hi = 0ULL;
    }
    __syncthreads();
    atomicAdd(&s_n, n_inp);
    if (lo <= hi) {
      atomicMin(&s_lo, ct_key(lo));
      atomicMax(&s_hi, ct_key(hi));
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      if (s_n) atomicAdd(&ctr[kCtInpaint], s_n);
      if (s_lo <= s_hi) {
        atomicMin(&hull[0], s_lo);
        atomicMax(&hull[1], s_hi);
      }
    }
  }
  grid.sync();
  if (block_ld(&ctr[kCtInpaint]) > A.capacity) {  // cannot happen with capacity = H * W
    if (gtid == 0) ctr[kCtDone] = 3;
    return;
  }
  ct_list_flags(A, 1);
  grid.sync();
  if (A.trace && gtid == 0) A.trace[4095 * 16 + 1] = ct_now();
  ct_run_tiles<C>(A, 1, sm);
  grid.sync();
  if (A.trace && gtid == 0) A.trace[0] = ct_now();

  const long long remaining0 = block_ld(&ctr[kCtInpaint]);
  long long rem = remaining0;
  bool data_live = A.order == 2;
  int s = 0;
  for (;; ++s) {
    const int F = block_ld(&ctr[kCtNF + ((s + 1) & 1)]);
    if (s > 0 && gtid == 0)  // candidates of shell s - 1 (complete after its last barrier)
      A.rows[5 * (int64_t)(s - 1) + 2] =
          A.tracked ? (long long)ld_cg(&ctr[kCtCand + ((s - 1) & 1)]) : (long long)HW;
    if (rem <= 0) break;
    if (F == 0) {
      if (gtid == 0) ctr[kCtDone] = 2;
      break;
    }
    if (s >= A.rows_cap) {
      if (gtid == 0) ctr[kCtDone] = 3;
      break;
    }
    const int* fr = A.fr[s & 1];
    int* frn = A.fr[(s + 1) & 1];
    const int b = s & 1;

    // ---- B: g and the ball sample at every frontier pixel
    {
      double* cols = sm + warp * 16 * (2 * A.tr.R + 1);
      for (int base = gwarp * 4; base < F; base += nwarps * 4) {
        const int nq = min(4, F - base);
        double mgx, mgy;
        ct_loop_g4(A, fr + base, nq, cols, mgx, mgy);
        if (A.trace && gtid == 0 && base == 0 && s < 4096) A.trace[1 + 16 * s + 12] = ct_now();
        const int k = base + (lane >> 3);
        const bool valid = k < F;
        const int p = valid ? fr[k] : 0;
        const int pj = p / W, pi = p - pj * W;
        SampleResult r;
        eval_item<NL, 0, true>(P, T, src, lane & 7, valid, (double)pi, (double)pj, true, mgx, mgy,
                               r, tdist);
        if (A.trace && gtid == 0 && base == 0 && s < 4096) A.trace[1 + 16 * s + 13] = ct_now();
        if (valid && (lane & 7) == 0) {
          A.eg[2 * k] = mgx;
          A.eg[2 * k + 1] = mgy;
          A.erw[k] = r.rw;
          A.etw[k] = r.tw;
#pragma unroll
          for (int c = 0; c < C; ++c) A.evals[(int64_t)k * C + c] = r.v[c];
        }
        const unsigned nz = __ballot_sync(0xffffffffu, valid && (mgx != 0.0 || mgy != 0.0));
        if (lane == 0 && nz) atomicOr(&ctr[kCtAnyG + b], 1);
      }
    }
    ct_trace_work(A, s, 8, 10);
    grid.sync();
    ct_trace(A, s, 0);
    if (gtid == 0) {  // the other bank: every block has read F and the last row
      const int o = (s + 1) & 1;
      ctr[kCtNF + o] = 0;
      ctr[kCtFill + o] = 0;
      ctr[kCtCand + o] = 0;
      ctr[kCtAnyG + o] = 0;
      ctr[kCtTiles + o] = 0;
      ctr[kCtGrab + o] = 0;
    }

    // ---- C: ready predicate (engine.py:317-330), fill = ready & rw > 0, and
    // the commit of the filled pixels (engine.py:350-356) with their dirty
    // tiles queued: no phase of this shell reads u or labels any more, and a
    // shell with nothing ready has written nothing (the guard below commits)
    if (data_live && block_ld(&ctr[kCtAnyG + b]) == 0) data_live = false;
    {
      const int mode = A.order == 0 ? 0 : (data_live ? 2 : 1);
      for (int k0 = gwarp * 32; k0 < F; k0 += nwarps * 32) {
        const int k = k0 + lane;
        bool f = false;
        int j = 0, i = 0;
        if (k < F) {
          const double rw = A.erw[k];
          const double conf = rw / A.etw[k];
          bool ready = true;
          if (mode == 1) ready = conf > A.c;
          else if (mode == 2) ready = hypot_np(A.eg[2 * k], A.eg[2 * k + 1]) > A.c2 && conf > A.c;
          f = ready && rw > 0.0;
          A.efill[k] = f ? 1 : 0;
          if (f) {
            const int p = fr[k];
#pragma unroll
            for (int c = 0; c < C; ++c) A.u[(int64_t)p * C + c] = A.evals[(int64_t)k * C + c];
            A.lab[p] = 0;
            A.fillshell[p] = s;
            j = p / W;
            i = p - j * W;
          }
        }
        ct_queue_tiles(A, b, f, j, i, dd);
        const unsigned bal = __ballot_sync(0xffffffffu, f);
        if (lane == 0 && bal) atomicAdd(&ctr[kCtFill + b], __popc(bal));
      }
    }
    ct_trace_work(A, s, 9, 11);
    grid.sync();
    ct_trace(A, s, 1);
    int n = block_ld(&ctr[kCtFill + b]);

    // ---- D: deadlock guard (engine.py:334-348)
    if (n == 0) {
      double bc = 0.0;
      int bk = -1, bp = 0x7fffffff;
      for (int k = gtid; k < F; k += nthreads) {
        const double cf = A.erw[k] / A.etw[k];
        const int p = fr[k];
        if (bk < 0 || ct_better(cf, p, bc, bp)) {
          bc = cf;
          bk = k;
          bp = p;
        }
      }
      double* rc = sm;
      int* rk = reinterpret_cast<int*>(sm + blockDim.x);
      rc[threadIdx.x] = bc;
      rk[threadIdx.x] = bk;
      __syncthreads();
      if (threadIdx.x == 0) {
        double c0 = 0.0;
        int k0 = -1;
        for (int t = 0; t < (int)blockDim.x; ++t) {
          const int kk = rk[t];
          if (kk < 0) continue;
          if (k0 < 0 || ct_better(rc[t], fr[kk], c0, fr[k0])) {
            c0 = rc[t];
            k0 = kk;
          }
        }
        A.slot_c[blockIdx.x] = c0;
        A.slot_k[blockIdx.x] = k0;
      }
      __syncthreads();
      grid.sync();
      if (gtid == 0) {
        double c0 = 0.0;
        int k0 = -1;
        for (int t = 0; t < (int)gridDim.x; ++t) {
          const int kk = A.slot_k[t];
          if (kk < 0) continue;
          if (k0 < 0 || ct_better(A.slot_c[t], fr[kk], c0, fr[k0])) {
            c0 = A.slot_c[t];
            k0 = kk;
          }
        }
        bool ok = true;
        if (!(A.erw[k0] > 0.0)) {
          // engine._neighbor_mean (engine.py:252-267): readable 8-neighbours
          const int p = fr[k0];
          const int j = p / W, i = p - j * W;
          double acc[C];
#pragma unroll
          for (int c = 0; c < C; ++c) acc[c] = 0.0;
          int cnt = 0;
          for (int o = 0; o < 8; ++o) {
            int ii = i + ct_nb_di(o);
            const int jj = j + ct_nb_dj(o);
            if (A.periodic) ii = (ii % W + W) % W;
            if (ii < 0 || ii >= W || jj < 0 || jj >= H) continue;
            const int64_t q = (int64_t)jj * W + ii;
            if (A.lab[q] != 0) continue;
#pragma unroll
            for (int c = 0; c < C; ++c) acc[c] += A.u[q * C + c];
            ++cnt;
          }
          if (cnt == 0) {
            ok = false;
            ctr[kCtDone] = 2;
          } else {
#pragma unroll
            for (int c = 0; c < C; ++c) A.evals[(int64_t)k0 * C + c] = acc[c] / cnt;
          }
        }
        if (ok) {
          // the guarded pixel's commit
          const int p = fr[k0];
#pragma unroll
          for (int c = 0; c < C; ++c) A.u[(int64_t)p * C + c] = A.evals[(int64_t)k0 * C + c];
          A.lab[p] = 0;
          A.fillshell[p] = s;
          A.efill[k0] = 1;
          ctr[kCtDeadlocks] += 1;
          ct_queue_tiles_one(A, b, p / W, p % W, dd);
        }
      }
      grid.sync();
      ct_trace(A, s, 2);
      if (block_ld(&ctr[kCtDone]) == 2) break;
      n = 1;
    }
    ct_trace(A, s, 3);
    rem -= n;

    // ---- A + F: the field on the dirty tiles; the next frontier
    if (A.trace && gtid == 0 && s < 4096) {
      A.trace[1 + 16 * s + 7] = (unsigned long long)F;
    }
    if (A.tracked) {
      // tracker._update_arrays (tracker.py:59-79): o < 8 the Inpaint
      // 8-neighbours of a filled entry, o == 8 the entry itself as survivor
      for (int k0 = gwarp * 32; k0 < F; k0 += nwarps * 32) {
        const int k = k0 + lane;
        const bool valid = k < F;
        const int p = valid ? fr[k] : 0;
        const bool filled = valid && A.efill[k];
        const int j = p / W, i = p - j * W;
        for (int o = 0; o < 9; ++o) {
          int q = -1, qj = 0, qi = 0;
          if (valid) {
            if (o == 8) {
              if (!filled) {
                q = p;
                qj = j;
                qi = i;
              }
            } else if (filled) {
              qi = i + ct_nb_di(o);
              qj = j + ct_nb_dj(o);
              if (A.periodic) qi = (qi % W + W) % W;
              if (qi >= 0 && qi < W && qj >= 0 && qj < H && A.lab[qj * W + qi] == 255)
                q = qj * W + qi;
            }
          }
          const bool claimed = q >= 0 && atomicMax(&A.stamp[q], s + 1) < s + 1;
          const bool act = claimed && ct_active(A.lab, H, W, A.periodic, qj, qi);
          const unsigned mc = __ballot_sync(0xffffffffu, claimed);
          if (lane == 0 && mc) atomicAdd(&ctr[kCtCand + b], __popc(mc));
          if (act && A.enter && A.enter[q] < 0) A.enter[q] = s + 1;
          warp_append(act, q, &ctr[kCtNF + b], frn);
        }
      }
    } else {
      for (int p0 = gwarp * 32; p0 < HW; p0 += nwarps * 32) {
        const int p = p0 + lane;
        bool act = false;
        if (p < HW && A.lab[p] == 255) {
          const int j = p / W, i = p - j * W;
          act = ct_active(A.lab, H, W, A.periodic, j, i);
          if (act && A.enter && A.enter[p] < 0) A.enter[p] = s + 1;
        }
        warp_append(act, p, &ctr[kCtNF + b], frn);
      }
    }
    ct_run_tiles<C>(A, b, sm);
    ct_trace(A, s, 4);  // block 0 out of tiles
    if (gtid == 0) {
      long long* row = A.rows + 5 * (int64_t)s;
      row[0] = s;
      row[1] = F;
      row[3] = A.tracked ? (long long)F : (long long)HW;
      row[4] = n;
    }
    grid.sync();
    ct_trace(A, s, 5);
    if (A.trace && gtid == 0 && s < 4096)
      A.trace[1 + 16 * s + 6] = (unsigned long long)ld_cg(&ctr[kCtTiles + b]);
  }
  if (gtid == 0) {
    ctr[kCtIters] = s;
    ctr[kCtFilled] = (int)(remaining0 - rem);
  }
  // hull clip of the whole image (engine.py:375-376); the caller clips after
  // painting when the fill ended unfillable
  grid.sync();
  if (block_ld(&ctr[kCtDone]) == 0) {
    const unsigned long long klo = hull[0], khi = hull[1];
    if (klo <= khi) {
      const double lo = ct_unkey(klo), hi = ct_unkey(khi);
      const int64_t n = (int64_t)HW * C;
      for (int64_t e = gtid; e < n; e += nthreads) {
        const double v = A.u[e];
        A.u[e] = v < lo ? lo : (v > hi ? hi : v);
      }
    }
  }
}

}  // namespace

int coherence_fill_launch(const CoherenceFillArgs& a, const BallParams& P, const BallTables& tab,
                          cudaStream_t stream) {
  if (a.height < 2 || a.width < 2 || a.channels < 1 || a.channels > 4)
    return set_error(GF_E_INVALID, "bad geometry");
  if ((long long)a.height * a.width >= (1LL << 31)) return set_error(GF_E_UNSUPPORTED, "frame too large");
  Taps ts, tr;
  if (make_taps(a.sigma, ts) != GF_OK || make_taps(a.rho, tr) != GF_OK)
    return set_error(GF_E_UNSUPPORTED, "sigma / rho window outside 1..64 taps");
  if (ts.R > kLoopRsMax) return set_error(GF_E_UNSUPPORTED, "sigma window too wide for the fused tile");
  const int H = a.height, W = a.width, C = a.channels;
  const size_t HW = (size_t)H * W;
  const int tiles_x = (W + kLTW - 1) / kLTW, tiles_y = (H + kLTH - 1) / kLTH;
  const size_t ntiles = (size_t)tiles_x * tiles_y;
  const size_t cap = a.capacity > 0 ? (size_t)a.capacity : 1;
  if (a.workspace_bytes < coherence_fill_workspace(H, W, C, a.capacity))
    return set_error(GF_E_WORKSPACE, "workspace too small");
  // carve the workspace (8-byte aligned pieces first)
  char* w = static_cast<char*>(a.workspace);
  auto take = [&](size_t bytes) {
    char* p = w;
    w += (bytes + 255) & ~size_t(255);
    return p;
  };
  CtLoopArgs A{};
  A.H = H;
  A.W = W;
  A.C = C;
  A.periodic = P.periodic;
  A.tracked = a.tracked;
  A.order = a.order;
  A.c = a.c;
  A.c2 = a.c2;
  A.lam = a.lam;
  A.tiles_x = tiles_x;
  A.tiles_y = tiles_y;
  A.rows_cap = a.rows_cap;
  A.capacity = a.capacity;
  A.u = a.image;
  A.lab = a.labels;
  A.Q = reinterpret_cast<double*>(take(4 * HW * sizeof(double)));
  A.eg = reinterpret_cast<double*>(take(2 * cap * sizeof(double)));
  A.erw = reinterpret_cast<double*>(take(cap * sizeof(double)));
  A.etw = reinterpret_cast<double*>(take(cap * sizeof(double)));
  A.evals = reinterpret_cast<double*>(take(cap * C * sizeof(double)));
  A.slot_c = reinterpret_cast<double*>(take(4096 * sizeof(double)));
  A.fr[0] = reinterpret_cast<int*>(take(cap * sizeof(int)));
  A.fr[1] = reinterpret_cast<int*>(take(cap * sizeof(int)));
  A.stamp = reinterpret_cast<int*>(take(HW * sizeof(int)));
  A.tflag = reinterpret_cast<unsigned*>(take(ntiles * sizeof(unsigned)));
  A.tlist = reinterpret_cast<int*>(take(ntiles * sizeof(int)));
  A.slot_k = reinterpret_cast<int*>(take(4096 * sizeof(int)));
  A.ctr = reinterpret_cast<int*>(take(kCtCount * sizeof(int) + 2 * sizeof(unsigned long long)));
  A.efill = reinterpret_cast<uint8_t*>(take(cap));
  A.fillshell = a.fillshell;
  A.enter = a.enter;
  A.rows = a.rows;
  A.ts = ts;
  A.tr = tr;
  cudaStream_t s = stream;
  // stamps / tile flags / counters start at zero; the field needs no init
  cudaMemsetAsync(A.stamp, 0, HW * sizeof(int), s);
  cudaMemsetAsync(A.tflag, 0, ntiles * sizeof(unsigned), s);
  cudaMemsetAsync(A.ctr, 0, kCtCount * sizeof(int) + 2 * sizeof(unsigned long long), s);
  cudaMemsetAsync(A.ctr + kCtCount, 0xff, sizeof(unsigned long long), s);  // hull min key
  const void* fn = nullptr;
  const bool wide = P.plan.n_leaves > 1;
  switch (C) {
    case 1: fn = wide ? (const void*)k_ct_loop<1, kMaxLeaves> : (const void*)k_ct_loop<1, 1>; break;
    case 2: fn = wide ? (const void*)k_ct_loop<2, kMaxLeaves> : (const void*)k_ct_loop<2, 1>; break;
    case 3: fn = wide ? (const void*)k_ct_loop<3, kMaxLeaves> : (const void*)k_ct_loop<3, 1>; break;
    default: fn = wide ? (const void*)k_ct_loop<4, kMaxLeaves> : (const void*)k_ct_loop<4, 1>; break;
  }
  const int R = ts.R;
  const size_t tile_dbl = (size_t)(C + 1) * (kLTH + 2 + 2 * R) * (kLTW + 2 + 2 * R) +
                          (size_t)(C + 1) * (kLTH + 2) * (kLTW + 2 + 2 * R) +
                          (size_t)C * (kLTH + 2) * (kLTW + 2);
  const size_t query_dbl = (size_t)(kLoopThreads / 32) * 16 * (2 * tr.R + 1);
  const size_t red_dbl = 2 * kLoopThreads;
  const size_t smem = ((sizeof(BallTables) + 15) & ~size_t(15)) + kMaxK * sizeof(double) +
                      std::max(tile_dbl, std::max(query_dbl, red_dbl)) * sizeof(double);
  if (smem > 200 * 1024) return set_error(GF_E_UNSUPPORTED, "rho window too wide for the fused loop");
  // grid size per (device, kernel, smem), cached: the occupancy query costs
  // host microseconds per call otherwise
  struct GridEntry {
    int dev;
    const void* fn;
    size_t smem;
    int grid;
  };
  static std::mutex mu;
  static std::vector<GridEntry> cache;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return set_error(GF_E_CUDA, "no device");
  int grid = 0;
  {
    std::lock_guard<std::mutex> lock(mu);
    for (const GridEntry& g : cache)
      if (g.dev == dev && g.fn == fn && g.smem == smem) grid = g.grid;
  }
  // the attribute is per function: set it for this launch's size every time
  if (cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
    return set_error(GF_E_CUDA, cudaGetErrorString(cudaGetLastError()));
  if (!grid) {
    int sms = 0, per_sm = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, kLoopThreads, smem) != cudaSuccess ||
        per_sm < 1)
      return set_error(GF_E_CUDA, "coherence loop does not fit on an SM");
    grid = std::min(sms * per_sm, 4096);
    std::lock_guard<std::mutex> lock(mu);
    cache.push_back({dev, fn, smem, grid});
  }
  const bool trace = getenv("GF_CT_TRACE") != nullptr;
  if (trace) {
    cudaMalloc(&A.trace, 4097 * 16 * sizeof(unsigned long long));
    cudaMemsetAsync(A.trace, 0, 4097 * 16 * sizeof(unsigned long long), s);
  }
  void* args[] = {(void*)&A, (void*)&P, (void*)&tab};
  cudaError_t e = cudaLaunchCooperativeKernel(fn, grid, kLoopThreads, args, smem, s);
  if (e != cudaSuccess) return set_error(GF_E_CUDA, cudaGetErrorString(e));
  count_launches(1);
  if (trace) {  // diagnostics: per-shell phase times (us) on stderr
    std::vector<unsigned long long> h(4097 * 16);
    cudaMemcpyAsync(h.data(), A.trace, h.size() * 8, cudaMemcpyDeviceToHost, s);
    cudaStreamSynchronize(s);
    cudaFree(A.trace);
    fprintf(stderr, "GF_CT_TRACE grid=%d frontier_scan_us=%.1f init_fields_us=%.1f\n", grid,
            (h[4095 * 16 + 1] - h[4095 * 16 + 2]) * 1e-3, (h[0] - h[4095 * 16 + 1]) * 1e-3);
    unsigned long long prev = h[0];
    for (int sh = 0; sh < 4095 && h[1 + 16 * sh + 5]; ++sh) {
      const unsigned long long* t = &h[1 + 16 * sh];
      const unsigned long long c_end = t[2] ? t[2] : t[1];
      fprintf(stderr,
              "shell %d (F %llu, tiles %llu): B %.1f (blk0 %.1f last %.1f) C %.1f D %.1f E %.1f "
              "(blk0 %.1f last %.1f) A(blk0) %.1f AF %.1f total %.1f | chunk0 g %.1f eval %.1f\n",
              sh, t[7], t[6], (t[0] - prev) * 1e-3, (t[8] - prev) * 1e-3, (t[10] - prev) * 1e-3,
              (t[1] - t[0]) * 1e-3, t[2] ? (t[2] - t[1]) * 1e-3 : 0.0, (t[3] - c_end) * 1e-3,
              (t[9] - c_end) * 1e-3, (t[11] - c_end) * 1e-3, (t[4] - t[3]) * 1e-3,
              (t[5] - t[3]) * 1e-3, (t[5] - prev) * 1e-3, (t[12] - prev) * 1e-3,
              (t[13] - t[12]) * 1e-3);
      prev = t[5];
    }
  }
  // report: [iterations, filled, deadlock_fills, done]
  if (a.report) {
    e = cudaMemcpyAsync(a.report, A.ctr + kCtDone, 4 * sizeof(int), cudaMemcpyDeviceToDevice, s);
    if (e != cudaSuccess) return set_error(GF_E_CUDA, cudaGetErrorString(e));
  }
  e = cudaPeekAtLastError();
  if (e != cudaSuccess) return set_error(GF_E_CUDA, cudaGetErrorString(e));
  return GF_OK;
}

size_t coherence_fill_workspace(int H, int W, int C, long long capacity) {
  const size_t HW = (size_t)H * W;
  const size_t ntiles = (size_t)((W + kLTW - 1) / kLTW) * ((H + kLTH - 1) / kLTH);
  const size_t cap = capacity > 0 ? (size_t)capacity : 1;
  auto r = [](size_t b) { return (b + 255) & ~size_t(255); };
  return r(4 * HW * 8) + r(2 * cap * 8) + 2 * r(cap * 8) + r(cap * C * 8) + r(4096 * 8) +
         2 * r(cap * 4) + r(HW * 4) + 2 * r(ntiles * 4) + r(4096 * 4) +
         r(kCtCount * 4 + 16) + r(cap);
}

}  // namespace gf
