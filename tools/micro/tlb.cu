// L2-hit load latency vs footprint (TLB reach): pointer chase over a region.
#include <cstdio>
#include <vector>
#include <cuda_runtime.h>
__global__ void chase(const unsigned* buf, int steps, unsigned start, long long* out) {
  unsigned i = start;
  long long t0 = clock64();
  for (int s = 0; s < steps; ++s) i = buf[i];
  long long t1 = clock64();
  out[0] = (t1 - t0) / steps;
  out[1] = i;
}
int main() {
  const size_t maxb = 512ull << 20;
  unsigned* buf; long long* out;
  cudaMalloc(&buf, maxb); cudaMalloc(&out, 16);
  for (size_t mb : {1, 2, 4, 16, 32, 64, 128, 256, 512}) {
    const size_t n = (mb << 20) / 4;
    // chase with a 4 KB+ stride pattern spread over the region
    std::vector<unsigned> h(n);
    const size_t stride = 1031 * 64 + 16;  // elements (~264 KB), odd multiple
    size_t cur = 0;
    for (size_t s = 0; s < n / 1024; ++s) {
      size_t nxt = (cur + stride) % n;
      h[cur] = (unsigned)nxt;
      cur = nxt;
    }
    cudaMemcpy(buf, h.data(), n * 4, cudaMemcpyHostToDevice);
    chase<<<1, 1>>>(buf, 256, 0, out);  // warm (L2)
    chase<<<1, 1>>>(buf, 512, 0, out);
    long long r[2];
    cudaMemcpy(r, out, 16, cudaMemcpyDeviceToHost);
    printf("footprint %4zu MB: %lld cycles per dependent load\n", mb, r[0]);
  }
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
}
