// Output delta: the host half of a fill's result path.
//
// A fill changes only the Inpaint pixels and the Bystanders the value-hull
// clip moves (engine.py:364-376); every Readable pixel comes back bit for bit
// as it went in.  The host API therefore mirrors the input into the caller's
// pinned output buffer with device->host DMA while the frame is still being
// uploaded (full-duplex PCIe), and after the fill this kernel writes only the
// pixels whose output differs bitwise from the input, straight into that
// mapped host buffer.  1080p f64 RGB: ~2 MB crosses the link after the fill
// instead of 50 MB.
#include <cuda_runtime.h>
#include <stdint.h>

#include "gf_internal.cuh"

namespace gf {

constexpr int kDeltaThreads = 256;

// One thread per pixel, grid-stride.  W = channel word (uint32 for f32,
// uint64 for f64): the comparison is on bits, so -0.0 vs 0.0 and NaN
// payloads count as changes exactly like a byte compare of the arrays.
// Writes go to host memory over PCIe, so they are made coalesced: a block
// takes 256 consecutive pixels (C * 256 consecutive words), every thread
// loads words t, t + 256, ... of both images (coalesced), a pixel is marked
// changed in shared memory if any of its words differs bitwise, and each
// thread then stores its own words of the changed pixels -- a run of changed
// pixels leaves the SM as whole contiguous segments instead of one 8-byte
// store per channel at a 24-byte stride.
template <typename Wd>
__global__ void __launch_bounds__(kDeltaThreads)
    k_output_delta(int64_t n_px, int C, const Wd* __restrict__ in, const Wd* __restrict__ out,
                   Wd* host, unsigned long long* n_changed) {
  __shared__ unsigned char s_chg[kDeltaThreads];
  unsigned cnt = 0;
  const int64_t n_tiles = (n_px + kDeltaThreads - 1) / kDeltaThreads;
  for (int64_t tile = blockIdx.x; tile < n_tiles; tile += gridDim.x) {
    const int64_t p0 = tile * kDeltaThreads;
    const int np = n_px - p0 < kDeltaThreads ? (int)(n_px - p0) : kDeltaThreads;
    const int nw = np * C;
    const int64_t w0 = p0 * C;
    s_chg[threadIdx.x] = 0;
    __syncthreads();
    Wd o[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int w = threadIdx.x + k * kDeltaThreads;
      if (k < C && w < nw) {
        o[k] = __ldg(out + w0 + w);
        if (o[k] != __ldg(in + w0 + w)) s_chg[w / C] = 1;
      }
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int w = threadIdx.x + k * kDeltaThreads;
      if (k < C && w < nw && s_chg[w / C]) host[w0 + w] = o[k];
    }
    if (threadIdx.x < np) cnt += s_chg[threadIdx.x];
    __syncthreads();
  }
  if (n_changed) {
    const unsigned w = __reduce_add_sync(0xffffffffu, cnt);
    if ((threadIdx.x & 31) == 0 && w) atomicAdd(n_changed, (unsigned long long)w);
  }
}

}  // namespace gf

using namespace gf;

extern "C" int gf_output_delta(int64_t n_px, int32_t channels, int32_t dtype, const void* input,
                               const void* output, void* host_out,
                               unsigned long long* n_changed, void* stream) {
  if (n_px < 0 || channels < 1 || channels > 4 || (dtype != GF_F32 && dtype != GF_F64))
    return set_error(GF_E_INVALID, "bad geometry or dtype");
  if (n_px == 0) return GF_OK;
  if (!input || !output || !host_out) return set_error(GF_E_INVALID, "NULL buffer");
  void* dev_host = nullptr;
  cudaError_t e = cudaHostGetDevicePointer(&dev_host, host_out, 0);
  if (e != cudaSuccess) {
    cudaGetLastError();
    return set_error(GF_E_INVALID, "host_out is not mapped pinned memory");
  }
  int sms = 148;
  int dev = 0;
  if (cudaGetDevice(&dev) == cudaSuccess)
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t want = (n_px + kDeltaThreads - 1) / kDeltaThreads;
  const int grid = (int)std::min<int64_t>(want, (int64_t)sms * 8);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (dtype == GF_F64)
    k_output_delta<unsigned long long><<<grid, kDeltaThreads, 0, s>>>(
        n_px, channels, static_cast<const unsigned long long*>(input),
        static_cast<const unsigned long long*>(output), static_cast<unsigned long long*>(dev_host),
        n_changed);
  else
    k_output_delta<uint32_t><<<grid, kDeltaThreads, 0, s>>>(
        n_px, channels, static_cast<const uint32_t*>(input), static_cast<const uint32_t*>(output),
        static_cast<uint32_t*>(dev_host), n_changed);
  count_launches(1);
  e = cudaPeekAtLastError();
  if (e != cudaSuccess) return set_error(GF_E_CUDA, cudaGetErrorString(e));
  return GF_OK;
}

namespace {
// Per-(thread, device) ring of timing-free events for the chunk hand-off: a
// record is consumed by the stream wait enqueued right after it, so reuse is
// safe.  Events belong to the device current at creation, so each device has
// its own ring (a single host thread may drive several GPUs).
constexpr int kRing = 64;
constexpr int kMaxDevices = 64;
struct EventRing {
  cudaEvent_t ev[kRing] = {};
  int pos = 0;
};
thread_local EventRing g_rings[kMaxDevices];
}  // namespace

extern "C" int gf_upload_mirrored(const void* host_src, void* dev_dst, void* host_mirror,
                                  int64_t nbytes, int64_t chunk, void* stream,
                                  void* side_stream) {
  if (nbytes < 0 || chunk <= 0) return set_error(GF_E_INVALID, "bad size");
  if (nbytes == 0) return GF_OK;
  if (!host_src || !dev_dst || !host_mirror) return set_error(GF_E_INVALID, "NULL buffer");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  cudaStream_t side = static_cast<cudaStream_t>(side_stream);
  const char* src = static_cast<const char*>(host_src);
  char* dst = static_cast<char*>(dev_dst);
  char* mir = static_cast<char*>(host_mirror);
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= kMaxDevices)
    return set_error(GF_E_CUDA, "no usable current device");
  EventRing& ring = g_rings[dev];
  for (int64_t lo = 0; lo < nbytes; lo += chunk) {
    const size_t n = (size_t)std::min(chunk, nbytes - lo);
    cudaEvent_t& ev = ring.ev[ring.pos];
    ring.pos = (ring.pos + 1) % kRing;
    cudaError_t e = cudaSuccess;
    if (!ev) e = cudaEventCreateWithFlags(&ev, cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaMemcpyAsync(dst + lo, src + lo, n, cudaMemcpyHostToDevice, s);
    if (e == cudaSuccess) e = cudaEventRecord(ev, s);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(side, ev, 0);
    if (e == cudaSuccess) e = cudaMemcpyAsync(mir + lo, dst + lo, n, cudaMemcpyDeviceToHost, side);
    if (e != cudaSuccess) return set_error(GF_E_CUDA, cudaGetErrorString(e));
  }
  return GF_OK;
}
