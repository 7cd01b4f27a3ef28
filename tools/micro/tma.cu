// Standalone check of the TMA helpers used by k_prep_tma (3-D tile load into
// shared memory with an mbarrier, then a 3-D tile store back out).
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <stdio.h>
#include <string.h>

__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }

struct Maps { CUtensorMap in, out, lab; int bw; };

template <int V>
__global__ void k(const __grid_constant__ Maps M, int* flag) {
  __shared__ __align__(128) float tile[32 * 96];
  __shared__ __align__(128) unsigned char labs[64 * 64];
  __shared__ __align__(8) unsigned long long bar;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&bar)), "r"(1) : "memory");
    if (V >= 1) asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bar)), "r"(32 * 96 * 4 + (V >= 1 ? 48 * 40 : 0)) : "memory");
    if (V >= 1)
    asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];"
                 ::"r"(smem_u32(labs)), "l"(reinterpret_cast<unsigned long long>(&M.lab)), "r"((int)blockIdx.x * 32 - 4), "r"(-4), "r"(0), "r"(smem_u32(&bar)) : "memory");
    asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];"
                 ::"r"(smem_u32(tile)), "l"(reinterpret_cast<unsigned long long>(&M.in)), "r"((int)blockIdx.x * 96), "r"(0), "r"(0), "r"(smem_u32(&bar)) : "memory");
  }
  if (V >= 2) {
    asm volatile("{\n.reg .pred p;\nWAIT_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra.uni WAIT_%=;\n}\n" ::"r"(smem_u32(&bar)), "r"(0) : "memory");
  } else {
    // plain spin with test_wait
    unsigned done = 0;
    while (!done) asm volatile("{\n.reg .pred p;\nmbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\nselp.u32 %0, 1, 0, p;\n}\n" : "=r"(done) : "r"(smem_u32(&bar)), "r"(0) : "memory");
  }
  if (threadIdx.x == 0) {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%1, %2, %3}], [%4];" ::"l"(reinterpret_cast<unsigned long long>(&M.out)), "r"((int)blockIdx.x * 96), "r"(0), "r"(0), "r"(smem_u32(tile)) : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
  }
  if (threadIdx.x == 0) atomicAdd(flag, 1);
}

int main() {
  const int W = 128, H = 64, C = 3;
  float *a, *b; int* flag;
  cudaMalloc(&a, W * H * C * 4); cudaMalloc(&b, W * H * C * 4); cudaMalloc(&flag, 4);
  float* h = (float*)malloc(W * H * C * 4);
  for (int i = 0; i < W * H * C; ++i) h[i] = (float)i;
  cudaMemcpy(a, h, W * H * C * 4, cudaMemcpyHostToDevice);
  void* ptr; cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPointByVersion("cuTensorMapEncodeTiled", &ptr, 12000, cudaEnableDefault, &q);
  auto enc = (PFN_cuTensorMapEncodeTiled_v12000)ptr;
  Maps M;
  cuuint64_t dims[3] = {(cuuint64_t)W * C, (cuuint64_t)H, 1};
  cuuint64_t str[2] = {(cuuint64_t)W * C * 4, (cuuint64_t)W * C * H * 4};
  cuuint32_t box[3] = {96, 32, 1}, es[3] = {1, 1, 1};
  int r1 = enc(&M.in, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, a, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  cuuint64_t ldims[3] = {(cuuint64_t)W, (cuuint64_t)H, 1};
  cuuint64_t lstr[2] = {(cuuint64_t)W, (cuuint64_t)W * H};
  cuuint32_t lbox[3] = {48, 40, 1};
  unsigned char* lb; cudaMalloc(&lb, W * H);
  int r3 = enc(&M.lab, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, lb, ldims, lstr, lbox, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("lab encode %d\n", r3);
  int r2 = enc(&M.out, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, b, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("encode %d %d\n", r1, r2);
  for (int v = 0; v < 3; ++v) {
    cudaMemset(b, 0, W * H * C * 4); cudaMemset(flag, 0, 4);
    if (v == 0) k<0><<<4, 128>>>(M, flag);
    if (v == 1) k<1><<<4, 128>>>(M, flag);
    if (v == 2) k<2><<<4, 128>>>(M, flag);
    cudaError_t e = cudaDeviceSynchronize();
    printf("variant %d: %s\n", v, cudaGetErrorString(e));
    if (e != cudaSuccess) return 1;
    cudaMemcpy(h, b, W * 32 * C * 4, cudaMemcpyDeviceToHost);
    int bad = 0; for (int i = 0; i < W * 32 * C; ++i) bad += h[i] != (float)i;
    printf("  bad %d\n", bad);
  }
  return 0;
}
