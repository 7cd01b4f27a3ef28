// Latency microbenchmark for the fp64 / shuffle / L2 primitives of the shell loop.
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ long long clk() { long long t; asm volatile("mov.u64 %0, %%clock64;" : "=l"(t)); return t; }
__global__ void k(double* out, long long* cyc, const double4* buf, int n, unsigned long long* cnt) {
  double a = out[0], b = out[1];
  long long t0, t1;
  const int N = 256;
  // DADD chain
  t0 = clk();
  for (int i = 0; i < N; ++i) a = a + b;
  t1 = clk(); cyc[0] = (t1 - t0) / N; out[2] = a;
  // DMUL chain
  t0 = clk();
  for (int i = 0; i < N; ++i) a = a * b;
  t1 = clk(); cyc[1] = (t1 - t0) / N; out[3] = a;
  // DDIV chain
  t0 = clk();
  for (int i = 0; i < N; ++i) a = b / a;
  t1 = clk(); cyc[2] = (t1 - t0) / N; out[4] = a;
  // sqrt chain
  t0 = clk();
  for (int i = 0; i < N; ++i) a = sqrt(a + b);
  t1 = clk(); cyc[3] = (t1 - t0) / N; out[5] = a;
  // double shuffle chain
  t0 = clk();
  for (int i = 0; i < N; ++i) a = __shfl_xor_sync(0xffffffffu, a, 1) + b;
  t1 = clk(); cyc[4] = (t1 - t0) / N; out[6] = a;
  // F2F f32->f64 + add
  float f = (float)a;
  t0 = clk();
  for (int i = 0; i < N; ++i) { a = (double)f + b; f = (float)a; }
  t1 = clk(); cyc[5] = (t1 - t0) / N; out[7] = a;
  // dependent global loads (L2, pointer chase through buf of n double4, stride large)
  int idx = 0;
  t0 = clk();
  for (int i = 0; i < 64; ++i) { double4 v = buf[idx]; idx = (int)v.x; }
  t1 = clk(); cyc[6] = (t1 - t0) / 64; out[8] = idx;
  // dependent atomics (L2)
  unsigned long long c = 0;
  t0 = clk();
  for (int i = 0; i < 64; ++i) c = atomicAdd(cnt + (c & 1), 1ull);
  t1 = clk(); cyc[7] = (t1 - t0) / 64; out[9] = (double)c;
  // int dependent IMAD chain
  int x = idx;
  t0 = clk();
  for (int i = 0; i < N; ++i) x = x * 3 + 1;
  t1 = clk(); cyc[8] = (t1 - t0) / N; out[10] = x;
  // globaltimer read cost
  unsigned long long g = 0, gt;
  t0 = clk();
  for (int i = 0; i < 64; ++i) { asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(gt)); g += gt; }
  t1 = clk(); cyc[9] = (t1 - t0) / 64; out[11] = (double)g;
}
int main() {
  double* out; long long* cyc; double4* buf; unsigned long long* cnt;
  const int n = 1 << 22;  // 128 MB of double4 -> L2 misses? use small for L2 hits
  const int nl2 = 1 << 16;   // 2 MB: L2 resident
  cudaMalloc(&out, 64 * 8); cudaMalloc(&cyc, 64 * 8); cudaMalloc(&buf, (size_t)n * 32); cudaMalloc(&cnt, 64);
  double4* h = new double4[nl2];
  for (int i = 0; i < nl2; ++i) h[i] = make_double4((double)((i * 7919 + 104729) % nl2), 0, 0, 0);
  cudaMemcpy(buf, h, (size_t)nl2 * 32, cudaMemcpyHostToDevice);
  double ho[2] = {1.0000001, 1e-9};
  cudaMemcpy(out, ho, 16, cudaMemcpyHostToDevice);
  cudaMemset(cnt, 0, 64);
  for (int rep = 0; rep < 3; ++rep) k<<<1, 32>>>(out, cyc, buf, nl2, cnt);
  cudaDeviceSynchronize();
  long long hc[10];
  cudaMemcpy(hc, cyc, sizeof(hc), cudaMemcpyDeviceToHost);
  const char* names[] = {"dadd", "dmul", "ddiv", "dsqrt", "shfl.f64+dadd", "f2f+dadd+f2f", "ldg L2 chase", "atomicAdd chain", "imad", "globaltimer read"};
  for (int i = 0; i < 10; ++i) printf("%-18s %lld cycles\n", names[i], hc[i]);
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
