// Automatic spline detection on the device:
// guide.detect_edge_seeds / make_spline (guide.py:65-88, 177-267).
//
//   ring     Readable pixels at chessboard distance ring_distance from
//            D u B (distance_transform_cdt, guide.py:65-88); the annulus
//            |d - ring| <= ceil(2 sigma) + 1 around it (guide.py:188-191)
//   canny    scikit-image's canny (skimage.feature._canny, >= 0.19), restated:
//            gray = mean over channels; Gaussian of the masked image divided
//            by the Gaussian of the mask (+ eps) ("bleed-over"), truncate 4,
//            zero padding; Sobel (scipy.ndimage.sobel, reflect); magnitude
//            sqrt(isobel^2 + jsobel^2); 3x3 erosion of the mask; bilinear
//            non-maximum suppression in four sectors; hysteresis = the
//            8-connected components of the low mask that hold a high pixel
//   hits     ring pixels on an edge, with strength hypot(np.gradient of the
//            guide's own Gaussian (truncate 2), guide.py:193-194)
//   rays     make_spline's entry search and extension (guide.py:231-259)
//            for each kept seed along the tensor's minor eigenvector
//
// Every per-pixel step follows numpy / scipy's evaluation order (no FMA;
// scipy's correlate1d symmetric / antisymmetric tap-pair order), so the
// masks are exact functions of the inputs.  scikit-image is absent from the
// build container: the Canny restatement is pinned by the reference's own
// detection tests (test_guide.py:154-216), not by skimage outputs.
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include "gf_internal.cuh"
#include "gf_math.cuh"

namespace gf {

namespace {

constexpr int kCdtCap = 24;  // chessboard distances are capped above ring + half
constexpr int kMaxGauss = 32;

struct Gauss {
  double w[kMaxGauss + 1];  // w[k] = weight at offset +-k
  int R;
};

// scipy.ndimage._gaussian_kernel1d(sigma, 0, radius), radius =
// int(truncate * sigma + 0.5): exp(-0.5 / sigma^2 * x^2) / sum (numpy exp,
// numpy pairwise sum)
int make_gauss(double sigma, double truncate, Gauss& g) {
  const int R = (int)(truncate * sigma + 0.5);
  if (!(sigma > 0.0) || R > kMaxGauss) return GF_E_UNSUPPORTED;
  const int n = 2 * R + 1;
  double phi[2 * kMaxGauss + 1];
  const double scale = -0.5 / (sigma * sigma);
  for (int i = 0; i < n; ++i) {
    const double x = (double)(i - R);
    phi[i] = exp_np(scale * (x * x));
  }
  const double sum = plan_sum(make_plan(n), phi);
  g.R = R;
  for (int k = 0; k <= R; ++k) g.w[k] = phi[R + k] / sum;
  return GF_OK;
}

// gray = image.mean(axis=2): ((c0 + c1) + c2) / C
__global__ void k_gray(int HW, int C, const double* __restrict__ img, double* __restrict__ gray) {
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= HW) return;
  const double* q = img + (size_t)p * C;
  double s = q[0];
  for (int c = 1; c < C; ++c) s = s + q[c];
  gray[p] = s / (double)C;
}

// distance to the nearest obstacle (label != 0) in the pixel's column, capped
__global__ void k_cdt_cols(int H, int W, const uint8_t* __restrict__ lab, uint8_t* __restrict__ g) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x, j = blockIdx.y;
  if (i >= W) return;
  int d = kCdtCap + 1;
  for (int dj = 0; dj <= kCdtCap && d > kCdtCap; ++dj) {
    if ((j - dj >= 0 && lab[(size_t)(j - dj) * W + i] != 0) ||
        (j + dj < H && lab[(size_t)(j + dj) * W + i] != 0))
      d = dj;
  }
  g[(size_t)j * W + i] = (uint8_t)d;
}

// chessboard distance d = min over columns of max(|di|, column distance);
// ring: Readable and d == ring; annulus: Readable and |d - ring| <= half
__global__ void k_cdt_rows(int H, int W, const uint8_t* __restrict__ lab,
                           const uint8_t* __restrict__ g, int ring, int half,
                           uint8_t* __restrict__ ring_m, uint8_t* __restrict__ ann_m) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x, j = blockIdx.y;
  if (i >= W) return;
  const size_t p = (size_t)j * W + i;
  int d = kCdtCap + 1;
  for (int di = -kCdtCap; di <= kCdtCap; ++di) {
    const int ii = i + di;
    if (ii < 0 || ii >= W) continue;
    const int a = abs(di), b = g[(size_t)j * W + ii];
    const int m = a > b ? a : b;
    d = m < d ? m : d;
  }
  const bool rd = lab[p] == 0;
  ring_m[p] = (rd && d == ring) ? 1 : 0;
  ann_m[p] = (rd && d >= ring - half && d <= ring + half) ? 1 : 0;
}

// the masked image and the mask as doubles (canny's _preprocess)
__global__ void k_mask_prep(int HW, const double* __restrict__ gray, const uint8_t* __restrict__ m,
                            double* __restrict__ masked, double* __restrict__ maskf) {
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= HW) return;
  masked[p] = m[p] ? gray[p] : 0.0;
  maskf[p] = m[p] ? 1.0 : 0.0;
}

// one correlate1d pass of scipy's symmetric path, zero padding: out = x[0] w0
// + sum over d = R .. 1 of (x[-d] + x[d]) w[d] (outermost pair first)
__global__ void k_gauss_axis(int H, int W, int axis, const Gauss gs, const double* __restrict__ in,
                             double* __restrict__ out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x, j = blockIdx.y;
  if (i >= W) return;
  auto at = [&](int jj, int ii) -> double {
    return (jj >= 0 && jj < H && ii >= 0 && ii < W) ? in[(size_t)jj * W + ii] : 0.0;
  };
  double acc = at(j, i) * gs.w[0];
  for (int d = gs.R; d >= 1; --d) {
    const double a = axis == 0 ? at(j - d, i) : at(j, i - d);
    const double b = axis == 0 ? at(j + d, i) : at(j, i + d);
    acc += (a + b) * gs.w[d];
  }
  out[(size_t)j * W + i] = acc;
}

// smoothed = gauss(masked) / (gauss(mask) + eps)
__global__ void k_bleed(int HW, const double* __restrict__ gm, const double* __restrict__ gk,
                        double* __restrict__ sm) {
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= HW) return;
  sm[p] = gm[p] / (gk[p] + 2.220446049250313e-16);
}

// scipy 'reflect': (d c b a | a b c d | d c b a)
__device__ __forceinline__ int reflect(int x, int n) {
  if (n == 1) return 0;
  while (x < 0 || x >= n) x = x < 0 ? -x - 1 : 2 * n - x - 1;
  return x;
}

// ndi.sobel along both axes (reflect) and the magnitude
__global__ void k_sobel(int H, int W, const double* __restrict__ x, double* __restrict__ isob,
                        double* __restrict__ jsob, double* __restrict__ mag) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x, j = blockIdx.y;
  if (i >= W) return;
  auto X = [&](int jj, int ii) { return x[(size_t)reflect(jj, H) * W + reflect(ii, W)]; };
  // jsobel: [-1, 0, 1] along axis 1, then [1, 2, 1] along axis 0
  double t[3], u[3];
  for (int k = 0; k < 3; ++k) {
    const int jj = reflect(j + k - 1, H);
    t[k] = X(jj, i + 1) - X(jj, i - 1);
    const int ii = reflect(i + k - 1, W);
    u[k] = X(j + 1, ii) - X(j - 1, ii);
  }
  const double js = t[1] * 2.0 + (t[0] + t[2]);
  const double is = u[1] * 2.0 + (u[0] + u[2]);
  const size_t p = (size_t)j * W + i;
  isob[p] = is;
  jsob[p] = js;
  double m = is * is;
  m += js * js;
  mag[p] = sqrt(m);
}

// 3x3 erosion of the mask (border_value 0) + bilinear non-maximum
// suppression (skimage _nonmaximum_suppression_bilinear); flags: 1 = low
// (local maximum >= low), 3 = also >= high
__global__ void k_nms(int H, int W, const uint8_t* __restrict__ mask, const double* __restrict__ isob,
                      const double* __restrict__ jsob, const double* __restrict__ mag, double low,
                      double high, uint8_t* __restrict__ flags) {
  const int y = blockIdx.x * blockDim.x + threadIdx.x, x = blockIdx.y;  // x row, y column
  if (y >= W) return;
  const size_t p = (size_t)x * W + y;
  uint8_t out = 0;
  bool er = x >= 1 && x < H - 1 && y >= 1 && y < W - 1;
  for (int dx = -1; dx <= 1 && er; ++dx)
    for (int dy = -1; dy <= 1 && er; ++dy) er = mask[(size_t)(x + dx) * W + y + dy] != 0;
  const double m = mag[p];
  if (er && m >= low && m > 0.0) {
    auto M = [&](int xx, int yy) { return mag[(size_t)xx * W + yy]; };
    const double is = isob[p], js = jsob[p];
    const bool up = is >= 0.0, left = js >= 0.0;
    const bool c1 = (up && left) || (!up && !left);
    const bool c2 = fabs(is) >= fabs(js);
    double w, n11, n12, n21, n22;
    if (c1) {
      if (c2) {
        w = fabs(js) / fabs(is);
        n11 = M(x + 1, y); n12 = M(x + 1, y + 1); n21 = M(x - 1, y); n22 = M(x - 1, y - 1);
      } else {
        w = fabs(is) / fabs(js);
        n11 = M(x, y + 1); n12 = M(x + 1, y + 1); n21 = M(x, y - 1); n22 = M(x - 1, y - 1);
      }
    } else {
      if (c2) {
        w = fabs(js) / fabs(is);
        n11 = M(x + 1, y); n12 = M(x + 1, y - 1); n21 = M(x - 1, y); n22 = M(x - 1, y + 1);
      } else {
        w = fabs(is) / fabs(js);
        n11 = M(x, y - 1); n12 = M(x + 1, y - 1); n21 = M(x, y + 1); n22 = M(x - 1, y + 1);
      }
    }
    if (n12 * w + n11 * (1.0 - w) <= m && n22 * w + n21 * (1.0 - w) <= m) out = m >= high ? 3 : 1;
  }
  flags[p] = out;
}

// hysteresis: grow the kept set (bit 2 = kept) from the high pixels through
// 8-connected low pixels; *changed counts the pixels added in this pass
__global__ void k_hyst(int H, int W, uint8_t* __restrict__ flags, int* __restrict__ changed) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x, j = blockIdx.y;
  if (i >= W) return;
  const size_t p = (size_t)j * W + i;
  const uint8_t f = flags[p];
  if (!f || (f & 4)) return;
  bool keep = (f & 2) != 0;
  for (int dj = -1; dj <= 1 && !keep; ++dj)
    for (int di = -1; di <= 1 && !keep; ++di) {
      const int jj = j + dj, ii = i + di;
      if (jj >= 0 && jj < H && ii >= 0 && ii < W && (flags[(size_t)jj * W + ii] & 4)) keep = true;
    }
  if (keep) {
    flags[p] = f | 4;
    atomicAdd(changed, 1);
  }
}

// ring pixels on a kept edge: flat index and the strength hypot(gx, gy) of
// (gy, gx) = np.gradient(S) (central inside, one-sided on the border)
__global__ void k_hits(int H, int W, const uint8_t* __restrict__ ring_m,
                       const uint8_t* __restrict__ flags, const double* __restrict__ S, int cap,
                       int64_t* __restrict__ idx, double* __restrict__ strength,
                       int* __restrict__ count) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x, j = blockIdx.y;
  if (i >= W) return;
  const size_t p = (size_t)j * W + i;
  if (!ring_m[p] || !(flags[p] & 4)) return;
  auto at = [&](int jj, int ii) { return S[(size_t)jj * W + ii]; };
  double gy, gx;
  if (H == 1) gy = 0.0;
  else if (j == 0) gy = at(1, i) - at(0, i);
  else if (j == H - 1) gy = at(H - 1, i) - at(H - 2, i);
  else gy = (at(j + 1, i) - at(j - 1, i)) / 2.0;
  if (W == 1) gx = 0.0;
  else if (i == 0) gx = at(j, 1) - at(j, 0);
  else if (i == W - 1) gx = at(j, W - 1) - at(j, W - 2);
  else gx = (at(j, i + 1) - at(j, i - 1)) / 2.0;
  const int k = atomicAdd(count, 1);
  if (k < cap) {
    idx[k] = (int64_t)p;
    strength[k] = hypot_np(gx, gy);
  }
}

// make_spline's ray search (guide.py:231-259), one thread per seed: the first
// step t = 0.5, 1.0, ... <= budget whose rounded point (round half to even)
// is Inpaint, along +v and -v; the earlier wins (+v on ties); then the ray is
// extended while it stays inside the lattice and off Readable pixels.
// out[3k] = +1 / -1 (direction) or 0 (no entry), out[3k + 2] = t_end.
__global__ void k_rays(int H, int W, const uint8_t* __restrict__ lab, int n,
                       const double* __restrict__ seeds, const double* __restrict__ v, double budget,
                       double* __restrict__ out) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= n) return;
  const double sx = seeds[2 * k], sy = seeds[2 * k + 1];
  const double vx = v[2 * k], vy = v[2 * k + 1];
  const double step = 0.5;
  auto entry = [&](double dx, double dy) -> double {
    for (int s = 1;; ++s) {
      const double t = step * (double)s;  // np.arange(step, budget + step / 2, step)
      if (t >= budget + step / 2.0) return -1.0;
      const double px = sx + t * dx, py = sy + t * dy;
      const double rx = rint(px), ry = rint(py);
      if (!(rx >= 0.0 && rx < (double)W && ry >= 0.0 && ry < (double)H)) return -1.0;
      if (lab[(size_t)ry * W + (size_t)rx] == 255) return t;
    }
  };
  const double tp = entry(vx, vy), tm = entry(-vx, -vy);
  double sign = 0.0, t_entry = 0.0;
  if (tp >= 0.0 || tm >= 0.0) {
    if (tm < 0.0 || (tp >= 0.0 && tp <= tm)) {
      sign = 1.0;
      t_entry = tp;
    } else {
      sign = -1.0;
      t_entry = tm;
    }
  }
  double t_end = t_entry;
  if (sign != 0.0) {
    const double dx = sign > 0.0 ? vx : -vx, dy = sign > 0.0 ? vy : -vy;
    const double limit = 2.0 * (double)(H + W);
    double t = t_entry;
    while (t < limit) {
      t += step;
      const double px = sx + t * dx, py = sy + t * dy;
      const double rx = rint(px), ry = rint(py);
      if (!(rx >= 0.0 && rx < (double)W && ry >= 0.0 && ry < (double)H) ||
          lab[(size_t)ry * W + (size_t)rx] == 0)
        break;
      t_end = t;
    }
  }
  out[3 * k] = sign;
  out[3 * k + 1] = t_entry;
  out[3 * k + 2] = t_end;
}

}  // namespace

}  // namespace gf

using namespace gf;

extern "C" size_t gf_detect_workspace_bytes(int32_t height, int32_t width) {
  if (height <= 0 || width <= 0) return 0;
  const size_t HW = (size_t)height * width;
  return 6 * HW * sizeof(double) + 5 * HW + 256;
}

extern "C" int gf_detect_edges(int32_t height, int32_t width, int32_t channels, const double* image,
                               const uint8_t* labels, double sigma, double rho, double low,
                               double high, int32_t cap, int64_t* hit_idx, double* hit_strength,
                               int32_t* n_hits, uint8_t* ring_out, uint8_t* edges_out,
                               void* workspace, size_t workspace_bytes, void* stream) {
  if (height <= 0 || width <= 0 || channels < 1 || channels > 4 || cap < 0)
    return set_error(GF_E_INVALID, "bad geometry");
  if (!image || !labels || !n_hits || (cap > 0 && (!hit_idx || !hit_strength)) || !workspace)
    return set_error(GF_E_INVALID, "NULL buffer");
  if (workspace_bytes < gf_detect_workspace_bytes(height, width))
    return set_error(GF_E_WORKSPACE, "workspace too small");
  if (!(low <= high)) return set_error(GF_E_INVALID, "low threshold above high threshold");
  const int ring = (int)ceil(2.0 * sigma + 2.0 * rho) + 1;  // guide.ring_distance
  const int half = (int)ceil(2.0 * sigma) + 1;              // guide.py:187
  if (ring + half > kCdtCap) return set_error(GF_E_UNSUPPORTED, "ring beyond the distance cap");
  Gauss gc, gs;
  if (make_gauss(sigma, 4.0, gc) != GF_OK || make_gauss(sigma, 2.0, gs) != GF_OK)
    return set_error(GF_E_UNSUPPORTED, "Gaussian window too wide");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const int H = height, W = width;
  const size_t HW = (size_t)H * W;
  double* D0 = static_cast<double*>(workspace);
  double* gray = D0;
  double* t0 = D0 + HW;
  double* t1 = D0 + 2 * HW;
  double* t2 = D0 + 3 * HW;
  double* t3 = D0 + 4 * HW;
  double* t4 = D0 + 5 * HW;
  uint8_t* B0 = reinterpret_cast<uint8_t*>(D0 + 6 * HW);
  uint8_t* colg = B0;
  uint8_t* ring_m = B0 + HW;
  uint8_t* ann_m = B0 + 2 * HW;
  uint8_t* flags = B0 + 3 * HW;
  int* counters = reinterpret_cast<int*>(B0 + 5 * HW + 64 - ((uintptr_t)(B0 + 5 * HW) & 63));
  const int tb = 128;
  const dim3 rows((W + tb - 1) / tb, H);
  const int lin = (int)((HW + 255) / 256);
  cudaMemsetAsync(counters, 0, 2 * sizeof(int), s);
  k_gray<<<lin, 256, 0, s>>>((int)HW, channels, image, gray);
  k_cdt_cols<<<rows, tb, 0, s>>>(H, W, labels, colg);
  k_cdt_rows<<<rows, tb, 0, s>>>(H, W, labels, colg, ring, half, ring_m, ann_m);
  // canny (masked by the annulus)
  k_mask_prep<<<lin, 256, 0, s>>>((int)HW, gray, ann_m, t0, t1);
  k_gauss_axis<<<rows, tb, 0, s>>>(H, W, 0, gc, t0, t2);
  k_gauss_axis<<<rows, tb, 0, s>>>(H, W, 1, gc, t2, t0);  // gauss(masked)
  k_gauss_axis<<<rows, tb, 0, s>>>(H, W, 0, gc, t1, t2);
  k_gauss_axis<<<rows, tb, 0, s>>>(H, W, 1, gc, t2, t1);  // gauss(mask)
  k_bleed<<<lin, 256, 0, s>>>((int)HW, t0, t1, t2);       // smoothed
  k_sobel<<<rows, tb, 0, s>>>(H, W, t2, t0, t1, t3);      // isob, jsob, magnitude
  k_nms<<<rows, tb, 0, s>>>(H, W, ann_m, t0, t1, t3, low, high, flags);
  // hysteresis: passes until no pixel joins (checked every 16 passes)
  for (int round = 0; round < 4096; ++round) {
    cudaMemsetAsync(counters, 0, sizeof(int), s);
    for (int q = 0; q < 16; ++q) k_hyst<<<rows, tb, 0, s>>>(H, W, flags, counters);
    int changed = 0;
    cudaMemcpyAsync(&changed, counters, sizeof(int), cudaMemcpyDeviceToHost, s);
    if (cudaStreamSynchronize(s) != cudaSuccess) break;
    count_launches(16);
    if (changed == 0) break;
  }
  // seeds' strength: the guide's own Gaussian (truncate 2) of the gray image
  k_gauss_axis<<<rows, tb, 0, s>>>(H, W, 0, gs, gray, t4);
  k_gauss_axis<<<rows, tb, 0, s>>>(H, W, 1, gs, t4, t0);
  k_hits<<<rows, tb, 0, s>>>(H, W, ring_m, flags, t0, cap, hit_idx, hit_strength, counters + 1);
  count_launches(15);
  if (ring_out) cudaMemcpyAsync(ring_out, ring_m, HW, cudaMemcpyDeviceToDevice, s);
  if (edges_out) cudaMemcpyAsync(edges_out, flags, HW, cudaMemcpyDeviceToDevice, s);
  cudaMemcpyAsync(n_hits, counters + 1, sizeof(int), cudaMemcpyDeviceToHost, s);
  cudaError_t e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) return set_error(GF_E_CUDA, cudaGetErrorString(e));
  e = cudaPeekAtLastError();
  if (e != cudaSuccess) return set_error(GF_E_CUDA, cudaGetErrorString(e));
  return GF_OK;
}

extern "C" int gf_trace_rays(int32_t height, int32_t width, const uint8_t* labels, int32_t n,
                             const double* seeds, const double* v, double budget, double* out,
                             void* stream) {
  if (height <= 0 || width <= 0 || n < 0) return set_error(GF_E_INVALID, "bad geometry");
  if (n == 0) return GF_OK;
  if (!labels || !seeds || !v || !out) return set_error(GF_E_INVALID, "NULL buffer");
  k_rays<<<(n + 63) / 64, 64, 0, static_cast<cudaStream_t>(stream)>>>(height, width, labels, n,
                                                                      seeds, v, budget, out);
  count_launches(1);
  cudaError_t e = cudaPeekAtLastError();
  if (e != cudaSuccess) return set_error(GF_E_CUDA, cudaGetErrorString(e));
  return GF_OK;
}
