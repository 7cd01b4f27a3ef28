// L2 load latency inside a cooperative persistent kernel with grid barriers:
// 'active' warps each load 4 random float4 of a 33 MB buffer (lines written
// by other SMs in the previous round), timed with clock64.  Barrier: cg
// grid.sync (sleep < 0) or a generation barrier polling with __nanosleep.
#include <cstdio>
#include <cooperative_groups.h>
namespace cg = cooperative_groups;
__device__ unsigned hash32(unsigned x) { x ^= x >> 16; x *= 0x7feb352d; x ^= x >> 15; x *= 0x846ca68b; x ^= x >> 16; return x; }
__device__ void my_sync(unsigned* count, unsigned* gen, unsigned nb, int sleep_ns) {
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned g = *(volatile unsigned*)gen;
    __threadfence();
    if (atomicAdd(count, 1u) == nb - 1) { *(volatile unsigned*)count = 0u; __threadfence(); atomicAdd(gen, 1u); }
    else { while (*(volatile unsigned*)gen == g) { if (sleep_ns > 0) __nanosleep(sleep_ns); } }
    __threadfence();
  }
  __syncthreads();
}
__global__ void __launch_bounds__(256, 2) sim(float4* buf, unsigned n, int rounds, int active, unsigned long long* acc,
                                              int sleep_ns, unsigned* bar, int delay, int pattern) {
  cg::grid_group grid = cg::this_grid();
  const int lane = threadIdx.x & 31;
  const int gw = blockIdx.x * 8 + (threadIdx.x >> 5);
  unsigned long long sum = 0, cnt = 0;
  for (int r = 0; r < rounds; ++r) {
    if (gw < active) {
      if (delay) { long long t = clock64(); while (clock64() - t < delay) {} }
      unsigned base = hash32(gw * 7919u + r * 104729u);
      unsigned q[4];
      for (int t = 0; t < 4; ++t) {
        if (pattern == 0) q[t] = hash32(base + t * 31 + lane) % n;            // 32 random lines / instr
        else if (pattern == 1) q[t] = (hash32(base + t) % (n - 64)) + lane;   // 4 contiguous lines / instr
        else q[t] = (hash32(base) % (n - 4096)) + (lane & 7) + 1920 * ((lane >> 3) + 4 * t);  // 7x7-ball-like: 4 rows x 8 px
      }
      long long t0 = clock64();
      float4 v[4];
      for (int t = 0; t < 4; ++t) v[t] = buf[q[t]];
      float s = v[0].x + v[1].x + v[2].x + v[3].x;
      if (s == -1.f) asm volatile("trap;");
      long long t1 = clock64();
      sum += t1 - t0; cnt += 1;
      buf[hash32(base + 999 + lane) % n] = make_float4(s, 1.f, 2.f, 3.f);
    }
    if (sleep_ns < 0) grid.sync(); else my_sync(bar, bar + 1, gridDim.x, sleep_ns);
  }
  if (lane == 0 && cnt) { atomicAdd(acc, sum); atomicAdd(acc + 1, cnt); }
}
int main() {
  const unsigned n = 2073600;  // 1080p pixels
  float4* buf; unsigned long long* acc; unsigned* bar;
  cudaMalloc(&buf, (size_t)n * 16); cudaMemset(buf, 0, (size_t)n * 16);
  cudaMalloc(&acc, 16); cudaMalloc(&bar, 8);
  int dev = 0, sms = 0; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  for (int per : {2}) for (int sleep_ns : {-1}) for (int delay : {0}) for (int pattern : {0, 1, 2}) for (int active : {30, 296, 2368}) {
    int grid = sms * per;
    cudaMemset(acc, 0, 16); cudaMemset(bar, 0, 8);
    int rounds = 50;
    void* args[] = {&buf, (void*)&n, &rounds, &active, &acc, &sleep_ns, &bar, &delay, &pattern};
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0);
    cudaLaunchCooperativeKernel((void*)sim, grid, 256, args, 0, 0);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    unsigned long long h[2];
    cudaMemcpy(h, acc, 16, cudaMemcpyDeviceToHost);
    printf("pattern %d grid %4d active %5d: load %5.0f cycles, %.2f us/round\n", pattern, grid, active,
           (double)h[0] / h[1], ms * 1e3 / rounds); (void)sleep_ns; (void)delay;
  }
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
}
