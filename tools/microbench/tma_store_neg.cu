// Does a TMA tensor store with negative / fully-OOB coordinates complete?
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <cstring>
#include "sm100_ptx.cuh"
using namespace tec_sm100;
__global__ void k(const __grid_constant__ CUtensorMap tm, int c1, int c2, int c3) {
  __shared__ __align__(1024) uint16_t box[32 * 32];
  for (int i = threadIdx.x; i < 32 * 32; i += blockDim.x) box[i] = (uint16_t)(i + 1);
  fence_proxy_async_smem();
  __syncthreads();
  if (threadIdx.x == 0) {
    tma_store_4d(&tm, smem_u32(box), 0, c1, c2, c3);
    bulk_commit();
    bulk_wait_all();
  }
  __syncthreads();
}
int main() {
  const int OC = 64, OW = 8, OH = 8, N = 1;
  uint16_t* y; cudaMalloc(&y, OC * OW * OH * N * 2); cudaMemset(y, 0, OC * OW * OH * N * 2);
  void* fn; cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  auto enc = (CUresult(*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill))fn;
  CUtensorMap tm;
  cuuint64_t dims[4] = {OC, OW, OH, N};
  cuuint64_t str[3] = {OC * 2, OC * 2 * OW, OC * 2 * OW * OH};
  cuuint32_t box[4] = {32, 32, 1, 1}, es[4] = {1, 1, 1, 1};
  for (int sw = 0; sw < 2; ++sw) {
  CUresult r = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, y, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   sw ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("swz %d encode %d\n", sw, (int)r);
  int cases[][3] = {{0, 0, 0}, {-3, 1, 0}, {-40, 2, 0}, {0, 9, 0}, {2, 3, 0}};
  for (auto& c : cases) {
    k<<<1, 128>>>(tm, c[0], c[1], c[2]);
    cudaError_t e = cudaDeviceSynchronize();
    printf("coord ow=%d oh=%d n=%d -> %s\n", c[0], c[1], c[2], cudaGetErrorString(e));
    if (e) return 1;
  }
  }
  uint16_t h[OC * OW * OH];
  cudaMemcpy(h, y, sizeof(h), cudaMemcpyDeviceToHost);
  for (int oh = 0; oh < 4; ++oh) { for (int ow = 0; ow < OW; ++ow) printf("%5d", h[(oh * OW + ow) * OC]); printf("\n"); }
  return 0;
}
