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

#include <algorithm>

#include "gf_internal.cuh"
#include "gf_math.cuh"
#include "gf_npmath.cuh"

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
