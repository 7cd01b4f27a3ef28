// Internal declarations shared by the CUDA translation units.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>
#include <string.h>
#include <algorithm>

#include "../../include/guidefill_b200.h"
#include "gf_sampler.cuh"

namespace gf {

constexpr int kMaxFramesPerLaunch = 1024;
constexpr int kIntsPerFrame = 28;  // cnt[4] cntR[4] fills[4] anyg[4] + 11 scalars (+ 1 shared)

// Everything the fill kernels need, passed by value (__grid_constant__).
struct FillArgs {
  int nF, H, W, HW, C, cap;
  unsigned w_mul;  // fast division by W (round-up multiplier, valid below 2^31)
  int w_shr;
  int dtype;
  const void* image;
  const uint8_t* labels;
  const double* gsrc;  // caller's per-pixel guide (g_mode 2 without splines)
  double4* gbuf;       // per Inpaint pixel (gx, gy, ux, uy), written by k_prep, or nullptr
  void* out;
  float4* work;
  float* c3;
  uint32_t* list0;
  uint32_t* list1;
  double* conf;
  float4* gval;    // [nF][HW] sampled value of an unfilled item with rw > 0 (the guard's fill)
  int* cnt;        // [4][nF] frontier list front part (lattice entries)
  int* cntR;       // [4][nF] frontier list back part (rotated-ball entries)
  int* fills;      // [4][nF] pixels filled in the shell
  int* anyg;       // [4][nF] frontier holds a g != 0 pixel (data-term latch)
  int* remaining;  // [nF]
  int* iters;      // [nF]
  int* done;       // [nF] 0 running, 1 complete, 2 unfillable
  int* deadlocks;  // [nF]
  int* filled;     // [nF]
  int* dt_dead;    // [nF] data-term latch released (engine.py:327-329)
  int* best_p;     // [nF]
  int* inpaint;    // [nF]
  int* overflow;   // [nF]
  int* last_f;     // [nF] frontier size of a shell that ended unfilled
  int* badlab;     // [nF] a label outside {0, 128, 255} was seen
  unsigned long long* best_key;  // [nF]
  unsigned long long* hull;      // [nF][2] order-preserving encoded min/max
  int* stats;
  int* rows;
  int rows_cap;
  int* enter;
  int* fillshell;
  int order;
  double c, c2;
  int g_mode;
  double gfx, gfy;
  int periodic;
  int split;       // rotated-ball entries kept in the back part (K <= 128)
  int halo;        // r + 1: farthest pixel a ball sample's corners can touch
  int* clip_next;  // Bystander-clip tile counter (shell loop)
  int clip_total;  // tiles over all frames
  int ntiles;      // 32x32 tiles per frame
  unsigned long long* bys;        // [nF][ntiles][2] Bystander value range per tile (encoded)
  unsigned long long* bys_frame;  // [nF][2] the same per frame
  // fused spline raster (guide.py:286-327), n_seg == 0 when off
  int n_seg;
  const int32_t* frame_seg;  // per-frame segment ranges or nullptr
  const double4* seg;
  const int32_t* seg_spline;
  const double2* dirs;
  double cut;    // 3.0 * eta
  double c2eta;  // 2.0 * eta * eta
  // optional per-shell phase timestamps (globaltimer ns), [trace_cap][6]
  unsigned long long* trace;
  int trace_cap;
};

// thread-local error reporting (gf_abi.cu)
int set_error(int code, const char* msg);
// process-wide count of the kernels this library has launched (gf_launch_count)
void count_launches(int n);

// gf_fill.cu
size_t fill_workspace_bytes(int nF, int H, int W, int C, bool need_g);
int fill_launch(const gf_frames* fr, const gf_fill_params* prm, const gf_fill_outputs* out,
                const gf_splines* spl, void* ws, size_t ws_bytes, cudaStream_t stream,
                const BallParams& P, const BallTables& host_tab);

// gf_points.cu
// a ball beyond the kernels' fixed tables (r > GF_MAX_RADIUS): device arrays
struct BigBall {
  int K;
  const double* n;
  const double* m;
  const double* w0;
  const int* ni;
  const int* mi;
  int n_leaves;
  const int* leaf_lo;  // numpy pairwise plan: leaves (start, length) and the
  const int* leaf_n;   // postfix program (>= 0 push leaf, -1 add the top two)
  int n_prog;
  const int* prog;
  int rotated, periodic, mu_inf;
  double coef, tol_inf;
};
int sample_points_big_launch(int H, int W, int C, const double* image, const uint8_t* labels,
                             int n, const double* points, const double* g, const BigBall& B,
                             double* rw, double* tw, double* vals, cudaStream_t stream);
int sample_points_launch(int H, int W, int C, const double* image, const uint8_t* labels, int n,
                         const double* points, const double* g, const BallParams& P,
                         const BallTables& tab, double* rw, double* tw, double* vals,
                         cudaStream_t stream);
int bilinear_launch(int H, int W, int C, const double* image, const uint8_t* labels, int n,
                    const double* X, const double* Y, int periodic, double* vals, uint8_t* ok,
                    cudaStream_t stream);
int boundary_launch(int H, int W, const uint8_t* labels, int periodic, uint8_t* active,
                    uint8_t* inner, uint8_t* outer, cudaStream_t stream);

// gf_coherence.cu: the whole coherence-transport fill in one persistent kernel
struct CoherenceFillArgs {
  int height, width, channels;
  double* image;        // [H][W][C] f64, filled in place
  uint8_t* labels;      // [H][W], relabelled in place
  double sigma, rho, lam;
  int order;            // GF_ORDER_*
  double c, c2;
  int tracked;
  long long capacity;   // frontier entries (>= Inpaint pixels)
  int32_t* fillshell;   // [H][W], preset to -1
  int32_t* enter;       // [H][W] preset to -1, or nullptr
  long long* rows;      // [rows_cap][5]
  int rows_cap;
  int32_t* report;      // [4]: done (2 unfillable, 3 rows overflow), iterations, deadlocks, filled
  void* workspace;
  size_t workspace_bytes;
};
size_t coherence_fill_workspace(int H, int W, int C, long long capacity);
int coherence_fill_launch(const CoherenceFillArgs& a, const BallParams& P, const BallTables& tab,
                          cudaStream_t stream);

// gf_guide.cu
int guide_launch(int H, int W, const uint8_t* labels, int n_seg, const double* seg,
                 const int32_t* seg_spline, int n_splines, const double* dirs, double eta,
                 double* out, cudaStream_t stream);

}  // namespace gf
