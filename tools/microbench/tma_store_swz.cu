// Is the TMA-store swizzle a function of the absolute smem address?
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include "sm100_ptx.cuh"
using namespace tec_sm100;
__global__ void k(const __grid_constant__ CUtensorMap tm, int off_rows) {
  __shared__ __align__(1024) uint16_t buf[64 * 32];
  const uint32_t base = smem_u32(buf);
  for (int i = threadIdx.x; i < 64 * 4; i += blockDim.x) {
    const int r = i / 4, c = i % 4;
    const uint32_t lin = base + r * 64 + c * 16;
    const uint32_t addr = lin ^ (((lin >> 7) & 3u) << 4);
    uint16_t* p = buf + (addr - base) / 2;
    for (int e = 0; e < 8; ++e) p[e] = (uint16_t)(r * 32 + c * 8 + e);
  }
  fence_proxy_async_smem();
  __syncthreads();
  if (threadIdx.x == 0) {
    tma_store_2d(&tm, base + off_rows * 64, 0, 0);
    bulk_commit();
    bulk_wait_all();
  }
}
int main() {
  uint16_t* y; cudaMalloc(&y, 64 * 32 * 2);
  void* fn; cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  auto enc = (CUresult(*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill))fn;
  CUtensorMap tm;
  cuuint64_t dims[2] = {32, 64}, str[1] = {64};
  cuuint32_t box[2] = {32, 32}, es[2] = {1, 1};
  printf("encode %d\n", (int)enc(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, y, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE));
  for (int off : {0, 2, 4, 6, 8, 1}) {
    cudaMemset(y, 0xff, 64 * 32 * 2);
    k<<<1, 128>>>(tm, off);
    cudaError_t e = cudaDeviceSynchronize();
    if (e) { printf("off %d -> %s\n", off, cudaGetErrorString(e)); return 1; }
    uint16_t h[32 * 32];
    cudaMemcpy(h, y, sizeof(h), cudaMemcpyDeviceToHost);
    int bad_abs = 0;
    for (int j = 0; j < 32; ++j)
      for (int c = 0; c < 32; ++c)
        if (h[j * 32 + c] != (uint16_t)((off + j) * 32 + c)) ++bad_abs;
    printf("off %d rows: mismatches vs absolute-address swizzle = %d  (row0: %d %d %d ... row1: %d)\n", off, bad_abs,
           h[0], h[8], h[16], h[32]);
  }
  return 0;
}
