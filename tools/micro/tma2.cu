// Which u8 TMA box / coordinate combinations are legal on sm_100a.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <stdio.h>
__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
struct Maps { CUtensorMap lab; };
__global__ void k(const __grid_constant__ Maps M, int x, int y, unsigned bytes, int* out) {
  __shared__ __align__(128) unsigned char labs[64 * 64];
  __shared__ __align__(8) unsigned long long bar;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&bar)), "r"(1) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bar)), "r"(bytes) : "memory");
    asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];"
                 ::"r"(smem_u32(labs)), "l"(reinterpret_cast<unsigned long long>(&M.lab)), "r"(x), "r"(y), "r"(0), "r"(smem_u32(&bar)) : "memory");
  }
  asm volatile("{\n.reg .pred p;\nWAIT_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra.uni WAIT_%=;\n}\n" ::"r"(smem_u32(&bar)), "r"(0) : "memory");
  if (threadIdx.x == 0) out[0] = labs[0] + labs[100];
}
int main() {
  const int W = 128, H = 64;
  unsigned char* lb; cudaMalloc(&lb, W * H); cudaMemset(lb, 7, W * H);
  int* out; cudaMalloc(&out, 4);
  void* ptr; cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPointByVersion("cuTensorMapEncodeTiled", &ptr, 12000, cudaEnableDefault, &q);
  auto enc = (PFN_cuTensorMapEncodeTiled_v12000)ptr;
  int cfg[][4] = {{64, 40, 0, -4}, {64, 40, -16, -4}, {64, 40, -16, 0}, {64, 40, 16, 0}, {64, 40, 112, 60}, {64, 40, 4, 0}};
  for (auto& c : cfg) {
    Maps M;
    cuuint64_t d[3] = {(cuuint64_t)W, (cuuint64_t)H, 1}, s[2] = {(cuuint64_t)W, (cuuint64_t)W * H};
    cuuint32_t box[3] = {(cuuint32_t)c[0], (cuuint32_t)c[1], 1}, es[3] = {1, 1, 1};
    int r = enc(&M.lab, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, lb, d, s, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    k<<<1, 128>>>(M, c[2], c[3], c[0] * c[1], out);
    cudaError_t e = cudaDeviceSynchronize();
    printf("box %dx%d at (%d,%d): encode %d -> %s\n", c[0], c[1], c[2], c[3], r, cudaGetErrorString(e));
    if (e != cudaSuccess) return 1;
  }
  return 0;
}
