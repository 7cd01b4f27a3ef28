// Spline -> guide-field rasteriser (guide.py:286-327).
//
// One thread per pixel.  Inpaint pixels walk every polyline segment in
// spline order and keep, per spline, the minimum point-to-segment distance
// (np.minimum semantics), then take the first spline attaining the overall
// minimum (np.argmin).  All distance arithmetic follows the reference's
// numpy evaluation order and uses the glibc-exact hypot, and the falloff
// uses the SVML-exact exp, so the field is bit-identical to the reference.
// Segments are staged in shared memory (they are tiny: a few hundred).
#include <cuda_runtime.h>
#include <stdint.h>

#include "gf_internal.cuh"

namespace gf {

constexpr int kGfThreads = 256;
constexpr int kGfMaxSmemSeg = 1024;

struct GfArgs {
  int H, W;
  const uint8_t* labels;
  int n_seg;
  const double4* seg;
  const int32_t* seg_spline;
  int n_splines;
  const double2* dirs;
  double c2eta;   // (2.0 * eta) * eta, as numpy's scalar expression 2.0*eta*eta
  double cut;     // 3.0 * eta
  double2* out;
};

__device__ __forceinline__ double segment_distance(double px, double py, double4 s) {
  const double ax = s.x, ay = s.y, bx = s.z, by = s.w;
  const double abx = bx - ax, aby = by - ay;
  const double L2 = abx * abx + aby * aby;
  if (L2 == 0.0) return hypot_np(px - ax, py - ay);
  double t = ((px - ax) * abx + (py - ay) * aby) / L2;
  // np.clip(t, 0, 1) == minimum(maximum(t, 0), 1), NaN-propagating
  t = (t < 0.0) ? 0.0 : t;
  t = (t > 1.0) ? 1.0 : t;
  return hypot_np(px - (ax + t * abx), py - (ay + t * aby));
}

__global__ void __launch_bounds__(kGfThreads) k_guide(GfArgs a) {
  __shared__ double4 s_seg[kGfMaxSmemSeg];
  __shared__ int s_spl[kGfMaxSmemSeg];
  const bool staged = a.n_seg <= kGfMaxSmemSeg;
  if (staged) {
    for (int i = threadIdx.x; i < a.n_seg; i += blockDim.x) {
      s_seg[i] = a.seg[i];
      s_spl[i] = a.seg_spline[i];
    }
  }
  __syncthreads();
  const int total = a.H * a.W;
  for (int p = blockIdx.x * blockDim.x + threadIdx.x; p < total; p += gridDim.x * blockDim.x) {
    double2 g = make_double2(0.0, 0.0);
    if (a.n_splines > 0 && a.n_seg > 0 && a.labels[p] == 255) {
      const double px = (double)(p % a.W), py = (double)(p / a.W);
      double dmin = INFINITY, best = INFINITY;
      int near = -1, cur = staged ? s_spl[0] : a.seg_spline[0];
      for (int i = 0; i < a.n_seg; ++i) {
        const double4 s = staged ? s_seg[i] : a.seg[i];
        const int sp = staged ? s_spl[i] : a.seg_spline[i];
        if (sp != cur) {
          // np.argmin over splines keeps the first minimum
          if (near < 0 || best < dmin) {
            dmin = best;
            near = cur;
          }
          cur = sp;
          best = INFINITY;
        }
        const double d = segment_distance(px, py, s);
        best = d < best ? d : best;  // np.minimum (distances are finite)
      }
      if (near < 0 || best < dmin) {
        dmin = best;
        near = cur;
      }
      // splines without segments (a single point) never occur: the wire
      // format requires >= 2 points (splines.py:98-99)
      double fall = exp_np((-(dmin * dmin)) / a.c2eta);
      if (dmin > a.cut) fall = 0.0;
      const double2 dir = a.dirs[near];
      g.x = dir.x * fall;
      g.y = dir.y * fall;
    }
    a.out[p] = g;
  }
}

int guide_launch(int H, int W, const uint8_t* labels, int n_seg, const double* seg,
                 const int32_t* seg_spline, int n_splines, const double* dirs, double eta,
                 double* out, cudaStream_t stream) {
  const int total = H * W;
  if (total <= 0) return GF_OK;
  GfArgs a;
  a.H = H;
  a.W = W;
  a.labels = labels;
  a.n_seg = n_seg;
  a.seg = reinterpret_cast<const double4*>(seg);
  a.seg_spline = seg_spline;
  a.n_splines = n_splines;
  a.dirs = reinterpret_cast<const double2*>(dirs);
  a.c2eta = 2.0 * eta * eta;
  a.cut = 3.0 * eta;
  a.out = reinterpret_cast<double2*>(out);
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int grid = std::min((total + kGfThreads - 1) / kGfThreads, sms * 8);
  k_guide<<<grid, kGfThreads, 0, stream>>>(a);
  count_launches(1);
  cudaError_t e = cudaPeekAtLastError();
  if (e != cudaSuccess) return set_error(GF_E_CUDA, cudaGetErrorString(e));
  return GF_OK;
}

}  // namespace gf
