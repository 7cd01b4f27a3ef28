// extern "C" boundary of libgf_b200.so (declared in include/guidefill_b200.h).
//
// Validates arguments (mirroring the reference's ValueError checks,
// engine.py:50-60), derives the ball constants on the host -- disk offsets in
// the reference's scan order (grid.py:109-124), the g = 0 weights
// 1/hypot(n, m) and the numpy pairwise-summation plan for K samples -- and
// dispatches to the kernels.
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <string.h>

#include <algorithm>
#include <atomic>
#include <string>
#include <vector>

#include "gf_internal.cuh"
#include "gf_npmath.cuh"

namespace gf {

static thread_local std::string g_last_error;

int set_error(int code, const char* msg) {
  g_last_error = msg ? msg : "";
  return code;
}

static std::atomic<long long> g_launches{0};
void count_launches(int n) { g_launches.fetch_add(n, std::memory_order_relaxed); }

// Disk offsets (n, m), n^2 + m^2 <= r^2, meshgrid order (m outer, n inner),
// centre moved to the front and then dropped (engine.py:172).
static const int kNbDi[8] = {-1, 0, 1, -1, 1, -1, 0, 1};
static const int kNbDj[8] = {-1, -1, -1, 0, 0, 1, 1, 1};

static int build_ball(const gf_fill_params* p, BallParams& P, BallTables& T) {
  if (p->r < 1) return set_error(GF_E_INVALID, "r must be >= 1");
  if (p->r > GF_MAX_RADIUS) return set_error(GF_E_UNSUPPORTED, "r exceeds GF_MAX_RADIUS");
  if (!(p->mu >= 0.0)) return set_error(GF_E_INVALID, "mu must be >= 0 (inf allowed)");
  if (p->order < 0 || p->order > 2) return set_error(GF_E_INVALID, "bad order");
  if (p->neighborhood < 0 || p->neighborhood > 1) return set_error(GF_E_INVALID, "bad neighborhood");
  if (p->g_mode < 0 || p->g_mode > 2) return set_error(GF_E_INVALID, "bad g_mode");
  memset(&P, 0, sizeof(P));
  memset(&T, 0, sizeof(T));
  const int r = p->r;
  int K = 0;
  for (int m = -r; m <= r; ++m)
    for (int n = -r; n <= r; ++n) {
      if (n * n + m * m > r * r) continue;
      if (n == 0 && m == 0) continue;
      T.n[K] = (double)n;
      T.m[K] = (double)m;
      T.w0[K] = 1.0 / hypot_np((double)n, (double)m);
      T.w0f[K] = (float)T.w0[K];
      T.ni[K] = n;
      T.mi[K] = m;
      T.kn[K] = -1;
      for (int o = 0; o < 8; ++o)  // NEIGHBOR_OFFSETS (grid.py:29-33)
        if (n == kNbDi[o] && m == kNbDj[o]) T.kn[K] = (signed char)o;
      ++K;
    }
  P.r = r;
  P.K = K;
  P.nb_unknown = 0;
  for (int o = 0; o < 8; ++o)
    if (kNbDi[o] * kNbDi[o] + kNbDj[o] * kNbDj[o] > r * r) P.nb_unknown |= 1u << o;
  P.rotated = p->neighborhood == GF_BALL_ROTATED;
  P.periodic = p->periodic_x != 0;
  P.mu_inf = isinf(p->mu) ? 1 : 0;
  const double mu = p->mu;
  P.coef = (-(mu * mu)) / (2.0 * (double)(r * r));
  P.tol_inf = 1e-12 * std::max(1.0, (double)(r * r));
  P.plan = make_plan(K);
  if (P.plan.n_leaves > kMaxLeaves) return set_error(GF_E_UNSUPPORTED, "pairwise plan too deep");
  P.tw0 = plan_sum(P.plan, T.w0);  // tw of every g = 0 item (engine.py:193)
  return GF_OK;
}

static int check_frames(const gf_frames* f) {
  if (!f) return set_error(GF_E_INVALID, "frames is NULL");
  if (f->n_frames < 0 || f->height <= 0 || f->width <= 0)
    return set_error(GF_E_INVALID, "bad frame geometry");
  if (f->channels < 1 || f->channels > 4) return set_error(GF_E_INVALID, "channels must be 1..4");
  if (f->dtype != GF_F32 && f->dtype != GF_F64) return set_error(GF_E_INVALID, "bad dtype");
  if ((long long)f->height * f->width >= (1LL << 31)) return set_error(GF_E_UNSUPPORTED, "frame too large");
  return GF_OK;
}

// numpy's pairwise summation tree for any K (gf_math.cuh's make_plan without
// the leaf cap): leaves of <= 128 elements, split at n/2 rounded down to a
// multiple of 8, as a postfix program
static void plan_dyn(int lo, int n, std::vector<int>& leaf_lo, std::vector<int>& leaf_n,
                     std::vector<int>& prog) {
  if (n <= 128) {
    prog.push_back((int)leaf_lo.size());
    leaf_lo.push_back(lo);
    leaf_n.push_back(n);
    return;
  }
  int n2 = n / 2;
  n2 -= n2 % 8;
  plan_dyn(lo, n2, leaf_lo, leaf_n, prog);
  plan_dyn(lo + n2, n - n2, leaf_lo, leaf_n, prog);
  prog.push_back(-1);
}

// gf_sample_points for r > GF_MAX_RADIUS: the ball (grid.py:109-124 order,
// engine.py:131-147 constants) in a temporary device buffer
static int sample_points_big(int H, int W, int C, const double* image, const uint8_t* labels,
                             int n, const double* points, const double* g,
                             const gf_fill_params* p, double* rw, double* tw, double* vals,
                             cudaStream_t s) {
  if (!(p->mu >= 0.0)) return set_error(GF_E_INVALID, "mu must be >= 0 (inf allowed)");
  if (p->neighborhood < 0 || p->neighborhood > 1) return set_error(GF_E_INVALID, "bad neighborhood");
  if (n <= 0) return GF_OK;
  const int r = p->r;
  std::vector<double> dn, dm, w0;
  std::vector<int> ni, mi;
  for (int m = -r; m <= r; ++m)
    for (int q = -r; q <= r; ++q) {
      if (q * q + m * m > r * r || (q == 0 && m == 0)) continue;
      dn.push_back((double)q);
      dm.push_back((double)m);
      w0.push_back(1.0 / hypot_np((double)q, (double)m));
      ni.push_back(q);
      mi.push_back(m);
    }
  const int K = (int)dn.size();
  std::vector<int> leaf_lo, leaf_n, prog;
  plan_dyn(0, K, leaf_lo, leaf_n, prog);
  const size_t nd = 3 * (size_t)K, nint = 2 * (size_t)K + 2 * leaf_lo.size() + prog.size();
  std::vector<unsigned char> host(nd * 8 + nint * 4);
  double* hd = reinterpret_cast<double*>(host.data());
  int* hi = reinterpret_cast<int*>(host.data() + nd * 8);
  std::copy(dn.begin(), dn.end(), hd);
  std::copy(dm.begin(), dm.end(), hd + K);
  std::copy(w0.begin(), w0.end(), hd + 2 * K);
  int* o = hi;
  o = std::copy(ni.begin(), ni.end(), o);
  o = std::copy(mi.begin(), mi.end(), o);
  o = std::copy(leaf_lo.begin(), leaf_lo.end(), o);
  o = std::copy(leaf_n.begin(), leaf_n.end(), o);
  std::copy(prog.begin(), prog.end(), o);
  void* dev = nullptr;
  cudaError_t e = cudaMallocAsync(&dev, host.size(), s);
  if (e != cudaSuccess) return set_error(GF_E_CUDA, cudaGetErrorString(e));
  e = cudaMemcpyAsync(dev, host.data(), host.size(), cudaMemcpyHostToDevice, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);  // the host vector is freed on return
  if (e != cudaSuccess) {
    cudaFreeAsync(dev, s);
    return set_error(GF_E_CUDA, cudaGetErrorString(e));
  }
  const double* dd = static_cast<const double*>(dev);
  const int* di = reinterpret_cast<const int*>(static_cast<unsigned char*>(dev) + nd * 8);
  BigBall B{};
  B.K = K;
  B.n = dd;
  B.m = dd + K;
  B.w0 = dd + 2 * K;
  B.ni = di;
  B.mi = di + K;
  B.n_leaves = (int)leaf_lo.size();
  B.leaf_lo = di + 2 * K;
  B.leaf_n = B.leaf_lo + leaf_lo.size();
  B.n_prog = (int)prog.size();
  B.prog = B.leaf_n + leaf_n.size();
  B.rotated = p->neighborhood == GF_BALL_ROTATED;
  B.periodic = p->periodic_x != 0;
  B.mu_inf = isinf(p->mu) ? 1 : 0;
  B.coef = (-(p->mu * p->mu)) / (2.0 * (double)(r * r));
  B.tol_inf = 1e-12 * std::max(1.0, (double)(r * r));
  const int rc = sample_points_big_launch(H, W, C, image, labels, n, points, g, B, rw, tw, vals, s);
  cudaFreeAsync(dev, s);
  return rc;
}

}  // namespace gf

using namespace gf;

extern "C" {

const char* gf_last_error(void) { return g_last_error.c_str(); }

int gf_abi_version(void) { return GF_ABI_VERSION; }

int64_t gf_launch_count(void) { return (int64_t)g_launches.load(std::memory_order_relaxed); }

size_t gf_fill_splines_workspace_bytes(const gf_frames* frames, const gf_fill_params* params,
                                       const gf_splines* splines) {
  if (check_frames(frames) != GF_OK) return 0;
  const int nF = std::min(frames->n_frames, kMaxFramesPerLaunch);
  // the per-pixel guide buffer exists whenever a guide can be non-zero
  const bool need_g = (splines && splines->n_seg > 0) || !params || params->g_mode != GF_G_ZERO;
  return fill_workspace_bytes(nF, frames->height, frames->width, frames->channels, need_g);
}

size_t gf_fill_workspace_bytes(const gf_frames* frames, const gf_fill_params* params) {
  return gf_fill_splines_workspace_bytes(frames, params, nullptr);
}

static int fill_common(const gf_frames* frames, const gf_fill_params* params,
                       const gf_splines* splines, const gf_fill_outputs* outputs,
                       void* workspace, size_t workspace_bytes, void* stream) {
  int rc = check_frames(frames);
  if (rc != GF_OK) return rc;
  if (!params || !outputs) return set_error(GF_E_INVALID, "NULL params/outputs");
  if (frames->n_frames == 0) return GF_OK;
  const bool raster = splines && splines->n_seg > 0;
  if (splines && splines->n_seg > 0 &&
      (!splines->seg || !splines->seg_spline || !splines->dirs || splines->n_splines <= 0))
    return set_error(GF_E_INVALID, "incomplete spline arrays");
  if (!raster && params->g_mode == GF_G_FIELD && !frames->guide)
    return set_error(GF_E_INVALID, "g_mode field needs a guide pointer");
  if (!frames->image || !frames->labels || !frames->out || !outputs->frame_stats || !outputs->rows)
    return set_error(GF_E_INVALID, "NULL device pointer");
  if (outputs->rows_cap < 1) return set_error(GF_E_INVALID, "rows_cap must be >= 1");
  BallParams P;
  BallTables* T = new BallTables;
  rc = build_ball(params, P, *T);
  if (rc != GF_OK) {
    delete T;
    return rc;
  }
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  // batches larger than one launch are split into consecutive launches
  const int H = frames->height, W = frames->width, C = frames->channels;
  const size_t HW = (size_t)H * W;
  const size_t esz = frames->dtype == GF_F64 ? 8 : 4;
  for (int f0 = 0; f0 < frames->n_frames && rc == GF_OK; f0 += kMaxFramesPerLaunch) {
    const int nF = std::min(kMaxFramesPerLaunch, frames->n_frames - f0);
    gf_frames sub = *frames;
    sub.n_frames = nF;
    sub.image = static_cast<const char*>(frames->image) + f0 * HW * C * esz;
    sub.out = static_cast<char*>(frames->out) + f0 * HW * C * esz;
    sub.labels = frames->labels + f0 * HW;
    sub.guide = frames->guide ? frames->guide + f0 * HW * 2 : nullptr;
    gf_fill_outputs o = *outputs;
    o.frame_stats = outputs->frame_stats + (size_t)f0 * GF_STATS;
    o.rows = outputs->rows + (size_t)f0 * outputs->rows_cap * 2;
    o.enter = outputs->enter ? outputs->enter + f0 * HW : nullptr;
    o.fillshell = outputs->fillshell ? outputs->fillshell + f0 * HW : nullptr;
    if (f0 > 0) o.shell_trace = nullptr;
    gf_splines sp;
    if (raster) {
      sp = *splines;
      if (sp.frame_seg) sp.frame_seg += f0;
    }
    rc = fill_launch(&sub, params, &o, raster ? &sp : nullptr, workspace, workspace_bytes, s, P,
                     *T);
  }
  delete T;  // passed by value as a kernel parameter: safe to free now
  return rc;
}

int gf_fill(const gf_frames* frames, const gf_fill_params* params, const gf_fill_outputs* outputs,
            void* workspace, size_t workspace_bytes, void* stream) {
  return fill_common(frames, params, nullptr, outputs, workspace, workspace_bytes, stream);
}

int gf_fill_splines(const gf_frames* frames, const gf_fill_params* params,
                    const gf_splines* splines, const gf_fill_outputs* outputs, void* workspace,
                    size_t workspace_bytes, void* stream) {
  if (!splines) return set_error(GF_E_INVALID, "NULL splines");
  return fill_common(frames, params, splines, outputs, workspace, workspace_bytes, stream);
}

int gf_guide_field(int32_t height, int32_t width, const uint8_t* labels, int32_t n_seg,
                   const double* seg, const int32_t* seg_spline, int32_t n_splines,
                   const double* dirs, double eta, double* out_field, void* stream) {
  if (height <= 0 || width <= 0) return set_error(GF_E_INVALID, "bad geometry");
  if (!labels || !out_field) return set_error(GF_E_INVALID, "NULL device pointer");
  if (n_seg < 0 || n_splines < 0) return set_error(GF_E_INVALID, "negative counts");
  if (n_seg > 0 && (!seg || !seg_spline || !dirs)) return set_error(GF_E_INVALID, "NULL spline arrays");
  return guide_launch(height, width, labels, n_seg, seg, seg_spline, n_splines, dirs, eta,
                      out_field, static_cast<cudaStream_t>(stream));
}

int gf_sample_points(int32_t height, int32_t width, int32_t channels, const double* image,
                     const uint8_t* labels, int32_t n, const double* points, const double* g,
                     const gf_fill_params* params, double* rw, double* tw, double* vals,
                     void* stream) {
  if (height <= 0 || width <= 0 || channels < 1 || channels > 4)
    return set_error(GF_E_INVALID, "bad geometry");
  if (params && params->r > GF_MAX_RADIUS)
    return sample_points_big(height, width, channels, image, labels, n, points, g, params, rw, tw,
                             vals, static_cast<cudaStream_t>(stream));
  BallParams P;
  BallTables* T = new BallTables;
  int rc = build_ball(params, P, *T);
  if (rc == GF_OK)
    rc = sample_points_launch(height, width, channels, image, labels, n, points, g, P, *T, rw, tw,
                              vals, static_cast<cudaStream_t>(stream));
  delete T;
  return rc;
}

int gf_bilinear_gather(int32_t height, int32_t width, int32_t channels, const double* image,
                       const uint8_t* labels, int32_t n, const double* X, const double* Y,
                       int32_t periodic_x, double* vals, uint8_t* ok, void* stream) {
  if (height <= 0 || width <= 0 || channels < 1 || channels > 4)
    return set_error(GF_E_INVALID, "bad geometry");
  return bilinear_launch(height, width, channels, image, labels, n, X, Y, periodic_x, vals, ok,
                         static_cast<cudaStream_t>(stream));
}

int gf_boundary_masks(int32_t height, int32_t width, const uint8_t* labels, int32_t periodic_x,
                      uint8_t* active, uint8_t* inner, uint8_t* outer, void* stream) {
  if (height <= 0 || width <= 0) return set_error(GF_E_INVALID, "bad geometry");
  return boundary_launch(height, width, labels, periodic_x, active, inner, outer,
                         static_cast<cudaStream_t>(stream));
}

size_t gf_coherence_fill_workspace_bytes(int32_t height, int32_t width, int32_t channels,
                                         int64_t capacity) {
  if (height <= 0 || width <= 0 || channels < 1 || channels > 4 || capacity < 0) return 0;
  return coherence_fill_workspace(height, width, channels, capacity);
}

int gf_coherence_fill(int32_t height, int32_t width, int32_t channels, double* image,
                      uint8_t* labels, const gf_fill_params* params, double sigma, double rho,
                      double lam, int64_t capacity, int32_t* fillshell, int32_t* enter,
                      int64_t* rows, int32_t rows_cap, int32_t* report, void* workspace,
                      size_t workspace_bytes, void* stream) {
  if (!params || !image || !labels || !fillshell || !rows || !report || !workspace)
    return set_error(GF_E_INVALID, "NULL argument");
  if (rows_cap < 1 || capacity < 0) return set_error(GF_E_INVALID, "bad rows_cap / capacity");
  if (params->order < 0 || params->order > 2) return set_error(GF_E_INVALID, "bad order");
  BallParams P;
  BallTables* T = new BallTables;
  int rc = build_ball(params, P, *T);
  if (rc == GF_OK) {
    CoherenceFillArgs a{};
    a.height = height;
    a.width = width;
    a.channels = channels;
    a.image = image;
    a.labels = labels;
    a.sigma = sigma;
    a.rho = rho;
    a.lam = lam;
    a.order = params->order;
    a.c = params->c;
    a.c2 = params->c2;
    a.tracked = params->tracked ? 1 : 0;
    a.capacity = capacity;
    a.fillshell = fillshell;
    a.enter = enter;
    a.rows = reinterpret_cast<long long*>(rows);
    a.rows_cap = rows_cap;
    a.report = report;
    a.workspace = workspace;
    a.workspace_bytes = workspace_bytes;
    rc = coherence_fill_launch(a, P, *T, static_cast<cudaStream_t>(stream));
  }
  delete T;
  return rc;
}

void gf_host_exp(const double* x, double* y, int64_t n) {
  for (int64_t i = 0; i < n; ++i) y[i] = exp_np(x[i]);
}

void gf_host_hypot(const double* x, const double* y, double* out, int64_t n) {
  for (int64_t i = 0; i < n; ++i) out[i] = hypot_np(x[i], y[i]);
}

double gf_host_pairwise_sum(const double* a, int32_t n) {
  const PairwisePlan p = make_plan(n);
  return plan_sum(p, a);
}

void gf_host_atan2(const double* y, const double* x, double* out, int64_t n) {
  for (int64_t i = 0; i < n; ++i) out[i] = atan2_np(y[i], x[i]);
}

void gf_host_tanh(const double* x, double* y, int64_t n) {
  for (int64_t i = 0; i < n; ++i) y[i] = tanh_np(x[i]);
}

void gf_host_sincos(const double* x, double* s, double* c, int64_t n) {
  for (int64_t i = 0; i < n; ++i) {
    s[i] = sin_np(x[i]);
    c[i] = cos_np(x[i]);
  }
}

}  // extern "C"
