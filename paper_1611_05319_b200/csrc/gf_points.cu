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
