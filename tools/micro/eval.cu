// Microbenchmark: latency of one ball evaluation (lattice / rotated) and of
// the fp64 primitives it is built from, one warp, clock64.
#include <cstdio>
#include <cmath>
#include <vector>
#include "../../paper_1611_05319_b200/csrc/gf_eval.cuh"
using namespace gf;
__device__ __forceinline__ long long clk() { long long t; asm volatile("mov.u64 %0, %%clock64;" : "=l"(t)); return t; }

__global__ void k_prims(double* out, long long* cyc, double a0, double b0) {
  const int N = 128;
  double a = a0, b = b0; long long t0;
  t0 = clk(); for (int i = 0; i < N; ++i) a = b0 / a;                     cyc[0] = (clk() - t0) / N; out[0] = a;
  a = a0; t0 = clk(); for (int i = 0; i < N; ++i) a = sqrt(a) + b;       cyc[1] = (clk() - t0) / N; out[1] = a;
  a = a0; t0 = clk(); for (int i = 0; i < N; ++i) a = hypot_np(a, b);    cyc[2] = (clk() - t0) / N; out[2] = a;
  a = -a0; t0 = clk(); for (int i = 0; i < N; ++i) a = -exp_np(a);       cyc[3] = (clk() - t0) / N; out[3] = a;
  a = a0; t0 = clk(); for (int i = 0; i < N; ++i) a = __shfl_xor_sync(0xffffffffu, a, (i & 3) + 1) + b; cyc[4] = (clk() - t0) / N; out[4] = a;
  a = a0; t0 = clk(); for (int i = 0; i < N; ++i) a = a * b + b;         cyc[5] = (clk() - t0) / N; out[5] = a;
  a = a0; t0 = clk(); for (int i = 0; i < N; ++i) a = floor(a + b);      cyc[6] = (clk() - t0) / N; out[6] = a;
}

__global__ void k_eval(const __grid_constant__ BallParams P, const __grid_constant__ BallTables T,
                       const float4* work, int H, int W, long long* cyc, double* out, double gx, double gy) {
  __shared__ BallTables S;
  for (int i = threadIdx.x; i < P.K; i += blockDim.x) { S.n[i] = T.n[i]; S.m[i] = T.m[i]; S.w0[i] = T.w0[i]; S.ni[i] = T.ni[i]; S.mi[i] = T.mi[i]; }
  __syncthreads();
  const int lane = threadIdx.x & 31;
  WorkSource src{work, nullptr, H, W, 3, 5};
  int p = 1000 * W + 500;
  double accum = 0.0;
  const int N = 32;
  long long t0 = clk();
  for (int i = 0; i < N; ++i) {
    SampleResult r;
    eval_lattice<3, 8>(P, S, src, lane & 7, lane >> 3, true, p % W, p / W, r);
    accum += r.rw;
    p += 7919 + ((int)r.v[0] & 1);  // dependent: next item waits for this one
    if (p >= H * W - 10 * W) p -= (H - 40) * W;
  }
  cyc[0] = (clk() - t0) / N;
  t0 = clk();
  for (int i = 0; i < N; ++i) {
    SampleResult r;
    eval_rot_warp<3>(P, S, src, lane, (double)(p % W), (double)(p / W), gx, gy, gx / 0.5, gy / 0.5, r);
    accum += r.rw;
    p += 7919 + ((int)r.v[0] & 1);
    if (p >= H * W - 10 * W) p -= (H - 40) * W;
  }
  cyc[1] = (clk() - t0) / N;
  // lattice eval timed alone, with a rotated eval (other code) between timings
  long long lat_sum = 0;
  for (int i = 0; i < N; ++i) {
    SampleResult r2;
    eval_rot_warp<3>(P, S, src, lane, (double)(p % W), (double)(p / W), gx, gy, gx / 0.5, gy / 0.5, r2);
    accum += r2.rw;
    p += 7919 + ((int)r2.v[0] & 1);
    if (p >= H * W - 10 * W) p -= (H - 40) * W;
    const long long ta = clk();
    SampleResult r;
    eval_lattice<3, 8>(P, S, src, lane & 7, lane >> 3, true, p % W, p / W, r);
    if (r.rw == -1.0) asm volatile("trap;");
    lat_sum += clk() - ta;
    accum += r.rw;
    p += 7919 + ((int)r.v[0] & 1);
    if (p >= H * W - 10 * W) p -= (H - 40) * W;
  }
  cyc[3] = lat_sum / N;
  // loads only: 4 independent float4 fetches per lane, dependent across iterations
  t0 = clk();
  for (int i = 0; i < N; ++i) {
    float4 v0 = work[p + lane], v1 = work[p + W + lane], v2 = work[p + 2 * W + lane], v3 = work[p + 3 * W + lane];
    p += 7919 + ((int)(v0.x + v1.x + v2.x + v3.x) & 1);
    if (p >= H * W - 10 * W) p -= (H - 40) * W;
  }
  cyc[2] = (clk() - t0) / N;
  out[threadIdx.x] = accum + p;
}

int main() {
  const int r = 3, H = 2048, W = 2048;
  BallParams P{};
  BallTables T{};
  int K = 0;
  for (int m = -r; m <= r; ++m)
    for (int n = -r; n <= r; ++n)
      if (n * n + m * m <= r * r && !(n == 0 && m == 0)) { T.n[K] = n; T.m[K] = m; T.ni[K] = n; T.mi[K] = m; T.w0[K] = 1.0 / std::hypot((double)n, (double)m); ++K; }
  P.r = r; P.K = K; P.rotated = 1; P.periodic = 0; P.mu_inf = 0;
  P.coef = -(50.0 * 50.0) / (2.0 * r * r);
  P.plan.n_leaves = 1; P.plan.leaf_lo[0] = 0; P.plan.leaf_n[0] = K; P.plan.n_prog = 1; P.plan.prog[0] = 0;
  std::vector<float4> h((size_t)H * W);
  for (size_t i = 0; i < h.size(); ++i) h[i] = make_float4(0.3f + (i % 7) * 0.01f, 0.5f, 0.7f, ((i % 5 == 0) ? 1.4e-43f : 0.0f));
  float4* work; long long* cyc; double* out;
  cudaMalloc(&work, h.size() * 16); cudaMalloc(&cyc, 64 * 8); cudaMalloc(&out, 64 * 8);
  cudaMemcpy(work, h.data(), h.size() * 16, cudaMemcpyHostToDevice);
  for (int rep = 0; rep < 3; ++rep) {
    k_prims<<<1, 32>>>(out, cyc, 1.2345, 0.3);
    k_eval<<<1, 32>>>(P, T, work, H, W, cyc + 16, out + 8, 0.4, 0.3);
  }
  cudaDeviceSynchronize();
  long long hc[32];
  cudaMemcpy(hc, cyc, sizeof(hc), cudaMemcpyDeviceToHost);
  const char* pn[] = {"ddiv", "dsqrt+dadd", "hypot_np", "exp_np", "shfl.f64+dadd", "dmul+dadd", "floor+dadd"};
  for (int i = 0; i < 7; ++i) printf("%-16s %lld cycles\n", pn[i], hc[i]);
  printf("%-16s %lld cycles\n", "eval lattice", hc[16]);
  printf("%-16s %lld cycles\n", "eval rotated", hc[17]);
  printf("%-16s %lld cycles\n", "4 fetches", hc[18]);
  printf("%-16s %lld cycles\n", "lattice after rot", hc[19]);
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
}
