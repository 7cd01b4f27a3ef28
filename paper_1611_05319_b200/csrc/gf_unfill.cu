// Unfillable fallback on the device (engine.py:270-283).
//
// When the frontier empties with Inpaint pixels left (cut off by a Bystander
// moat), the reference paints every stranded pixel with the colour of its
// nearest readable pixel, taken from scipy.ndimage.distance_transform_edt(
// ~readable, return_indices=True), or 0.5 when nothing is readable.  The
// nearest pixel -- ties included -- is whatever scipy's separable Voronoi
// feature transform returns, so this restates that transform
// (ni_morphology.c, _ComputeFT / _VoronoiFT; scipy's published algorithm):
//   pass 0 (axis 0, one thread per column): every pixel gets the nearest
//     feature row of its column; on a tie the upper one;
//   pass 1 (axis 1, one thread per row): the lower envelope of the column
//     candidates (stack test c*vR - b*uR - a*wR - a*b*c <= 0 keeps), then a
//     monotone sweep that advances only to a strictly closer candidate.
// All quantities are small integers held in doubles, so every product and
// comparison is exact and the ties resolve as in scipy.
#include <cuda_runtime.h>
#include <stdint.h>

#include "gf_internal.cuh"

namespace gf {

namespace {

__device__ __forceinline__ bool ft_feature(const uint8_t* labels, const int32_t* fillshell,
                                           int64_t p) {
  const uint8_t l = labels[p];
  return l == 0 || (l == 255 && fillshell[p] >= 0);  // Readable, or Inpaint already filled
}

// pass 0: nearest feature row per pixel along its column (-1: none)
__global__ void k_ft_cols(int H, int W, const uint8_t* __restrict__ labels,
                          const int32_t* __restrict__ fillshell, int32_t* __restrict__ row1) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= W) return;
  int up = -1;
  for (int i = 0; i < H; ++i) {
    const int64_t p = (int64_t)i * W + j;
    if (ft_feature(labels, fillshell, p)) up = i;
    row1[p] = up;
  }
  int dn = -1;
  for (int i = H - 1; i >= 0; --i) {
    const int64_t p = (int64_t)i * W + j;
    const int u = row1[p];
    if (u == i) dn = i;  // a feature pixel is its own nearest
    int best = u;
    if (u < 0) best = dn;
    else if (dn >= 0 && (i - u) > (dn - i)) best = dn;  // tie: the upper row (lower index)
    row1[p] = best;
  }
}

// pass 1 along each row, then paint the row's stranded pixels
template <typename T>
__global__ void k_ft_rows_paint(int H, int W, int C, const uint8_t* __restrict__ labels,
                                const int32_t* __restrict__ fillshell,
                                const int32_t* __restrict__ row1, int32_t* __restrict__ stack_ws,
                                T* out, int* n_painted) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= H) return;
  const int32_t* r1 = row1 + (int64_t)i * W;
  int32_t* g = stack_ws + (int64_t)i * W;  // candidate columns of the lower envelope
  const double ci = (double)i;
  int l = -1;
  for (int jj = 0; jj < W; ++jj) {
    if (r1[jj] < 0) continue;
    const double fd = (double)jj;
    const double tw = (double)r1[jj] - ci;
    const double wR = tw * tw;
    while (l >= 1) {
      const int i1 = g[l], i2 = g[l - 1];
      const double f1 = (double)i1;
      const double a = f1 - (double)i2;
      const double b = fd - f1;
      const double tu = (double)r1[i2] - ci, tv = (double)r1[i1] - ci;
      const double uR = tu * tu, vR = tv * tv;
      const double c = a + b;
      if (c * vR - b * uR - a * wR - a * b * c <= 0.0) break;
      --l;
    }
    g[++l] = jj;
  }
  const int maxl = l;
  int painted = 0;
  l = 0;
  for (int jj = 0; jj < W; ++jj) {
    const int64_t p = (int64_t)i * W + jj;
    int src_r = -1, src_c = -1;
    if (maxl >= 0) {
      double t0 = (double)r1[g[l]] - ci, t1 = (double)g[l] - (double)jj;
      double d1 = t0 * t0 + t1 * t1;
      while (l < maxl) {
        const double u0 = (double)r1[g[l + 1]] - ci, u1 = (double)g[l + 1] - (double)jj;
        const double d2 = u0 * u0 + u1 * u1;
        if (d1 <= d2) break;
        d1 = d2;
        ++l;
      }
      src_r = r1[g[l]];
      src_c = g[l];
    }
    if (labels[p] == 255 && fillshell[p] < 0) {
      ++painted;
      T* dst = out + p * C;
      if (src_r < 0) {
        for (int c = 0; c < C; ++c) dst[c] = (T)0.5;
      } else {
        const T* s = out + ((int64_t)src_r * W + src_c) * C;
        for (int c = 0; c < C; ++c) dst[c] = s[c];
      }
    }
  }
  if (painted && n_painted) atomicAdd(n_painted, painted);
}

}  // namespace

}  // namespace gf

using namespace gf;

extern "C" size_t gf_paint_unfillable_workspace_bytes(int32_t height, int32_t width) {
  if (height <= 0 || width <= 0) return 0;
  return (size_t)height * width * 2 * sizeof(int32_t);
}

extern "C" int gf_paint_unfillable(int32_t height, int32_t width, int32_t channels, int32_t dtype,
                                   const uint8_t* labels, const int32_t* fillshell, void* out,
                                   void* workspace, size_t workspace_bytes, int32_t* n_painted,
                                   void* stream) {
  if (height <= 0 || width <= 0 || channels < 1 || channels > 4 ||
      (dtype != GF_F32 && dtype != GF_F64))
    return set_error(GF_E_INVALID, "bad geometry or dtype");
  if (!labels || !fillshell || !out || !workspace) return set_error(GF_E_INVALID, "NULL buffer");
  if (workspace_bytes < gf_paint_unfillable_workspace_bytes(height, width))
    return set_error(GF_E_WORKSPACE, "workspace too small");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  int32_t* row1 = static_cast<int32_t*>(workspace);
  int32_t* stk = row1 + (size_t)height * width;
  k_ft_cols<<<(width + 127) / 128, 128, 0, s>>>(height, width, labels, fillshell, row1);
  if (dtype == GF_F64)
    k_ft_rows_paint<double><<<(height + 63) / 64, 64, 0, s>>>(
        height, width, channels, labels, fillshell, row1, stk, static_cast<double*>(out),
        n_painted);
  else
    k_ft_rows_paint<float><<<(height + 63) / 64, 64, 0, s>>>(
        height, width, channels, labels, fillshell, row1, stk, static_cast<float*>(out),
        n_painted);
  count_launches(2);
  cudaError_t e = cudaPeekAtLastError();
  if (e != cudaSuccess) return set_error(GF_E_CUDA, cudaGetErrorString(e));
  return GF_OK;
}
