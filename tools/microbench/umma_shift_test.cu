// Micro-experiment: can a K-major SWIZZLE_128B UMMA operand start at a row
// offset that is not a multiple of 8 rows (1024 B)? Variants: base_offset 0
// vs (row & 7). Also SWIZZLE_NONE planar layout with 16 B row shifts.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include "sm100_ptx.cuh"
using namespace tec_sm100;

__device__ uint64_t desc_sw128(uint32_t saddr, uint32_t base_off) {
  uint64_t d = make_smem_desc<128>(saddr, 1024);
  d |= (uint64_t)(base_off & 7) << 49;
  return d;
}
// SWIZZLE_NONE K-major: core matrix 8 rows x 16 B contiguous; SBO = M-dir
// core matrix stride, LBO = K-dir core matrix stride.
__device__ uint64_t desc_none(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;
  return d;
}

// mode 0: SW128 base_off=0; 1: SW128 base_off=row&7; 2: SWIZZLE_NONE planar
__global__ void k(const __grid_constant__ CUtensorMap ta, const __grid_constant__ CUtensorMap tb,
                  const __nv_bfloat16* a_plain, const __nv_bfloat16* b_plain,
                  float* out, int shift, int mode) {
  extern __shared__ uint8_t raw[];
  uint8_t* sm = (uint8_t*)(((uintptr_t)raw + 1023) & ~(uintptr_t)1023);
  uint8_t* sA = sm;                  // 256 rows x 128 B (SW128) or planar 8 x 256 x 16 B
  uint8_t* sB = sm + 32768;          // 64 rows x 128 B
  uint64_t* bar = (uint64_t*)(sm + 32768 + 8192 + 32768);
  uint32_t* slot = (uint32_t*)(bar + 2);
  int warp = threadIdx.x / 32;
  if (threadIdx.x == 0) { mbar_init(&bar[0], 1); mbar_init(&bar[1], 1); fence_barrier_init(); }
  if (warp == 1) tmem_alloc<64>(slot);
  tc_fence_before(); __syncthreads(); tc_fence_after();
  uint32_t tmem = *slot;
  if (mode < 2) {
    if (threadIdx.x == 0) {
      mbar_arrive_expect_tx(&bar[0], 32768 + 8192);
      tma_load_2d(sA, &ta, &bar[0], 0, 0);
      tma_load_2d(sA + 16384, &ta, &bar[0], 0, 128);
      tma_load_2d(sB, &tb, &bar[0], 0, 0);
    }
    mbar_wait(&bar[0], 0);
  } else {
    // planar: chunk j (8 ch) of pixel p at j*256*16 + p*16; B also no-swizzle:
    // B core matrices: n-group g (8 rows), k-chunk j: at j*(64*16) + n*16
    for (int i = threadIdx.x; i < 256 * 8; i += blockDim.x) {
      int p = i / 8, j = i % 8;
      *(uint4*)(sA + j * 256 * 16 + p * 16) = *(const uint4*)(a_plain + p * 64 + j * 8);
    }
    for (int i = threadIdx.x; i < 64 * 8; i += blockDim.x) {
      int n = i / 8, j = i % 8;
      *(uint4*)(sB + j * 64 * 16 + n * 16) = *(const uint4*)(b_plain + n * 64 + j * 8);
    }
    asm volatile("fence.proxy.async.shared::cta;");
    __syncthreads();
  }
  tc_fence_after();
  if (threadIdx.x == 32) {
    uint32_t idesc = make_idesc<MmaKind::kF16>(128, 64);
    for (int kk = 0; kk < 4; ++kk) {
      uint64_t ad, bd;
      if (mode < 2) {
        uint32_t a = smem_u32(sA) + shift * 128 + kk * 32;
        ad = desc_sw128(a, mode == 1 ? (uint32_t)shift : 0u);
        bd = make_smem_desc<128>(smem_u32(sB) + kk * 32, 1024);
      } else {
        // K16 step = 2 chunks of 8 channels
        ad = desc_none(smem_u32(sA) + (2 * kk) * 256 * 16 + shift * 16, 256 * 16, 128);
        bd = desc_none(smem_u32(sB) + (2 * kk) * 64 * 16, 64 * 16, 128);
      }
      tc_mma<MmaKind::kF16>(tmem, ad, bd, idesc, kk > 0);
    }
    tc_commit(&bar[1]);
  }
  mbar_wait(&bar[1], 0);
  tc_fence_after();
  if (warp < 4) {
    uint32_t v[32];
    for (int c = 0; c < 64; c += 32) {
      tmem_ld32(tmem + ((warp * 32) << 16) + c, v);
      tmem_ld_wait();
      int row = warp * 32 + threadIdx.x % 32;
      for (int j = 0; j < 32; ++j) out[row * 64 + c + j] = __uint_as_float(v[j]);
    }
  }
  tc_fence_before(); __syncthreads(); tc_fence_after();
  if (warp == 1) tmem_dealloc<64>(tmem);
}

typedef CUresult (*EncFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                          const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                          CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main() {
  void* fp; cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fp, cudaEnableDefault, &q);
  EncFn enc = (EncFn)fp;
  std::vector<__nv_bfloat16> A(256 * 64), B(64 * 64);
  std::vector<float> Af(256 * 64);
  for (int i = 0; i < 256 * 64; ++i) { float v = (float)((i * 37) % 251 - 125); A[i] = __float2bfloat16(v); Af[i] = v; }
  for (int n = 0; n < 64; ++n) for (int k = 0; k < 64; ++k) B[n * 64 + k] = __float2bfloat16(n == k ? 1.f : 0.f);
  __nv_bfloat16 *dA, *dB; float* dO;
  cudaMalloc(&dA, A.size() * 2); cudaMalloc(&dB, B.size() * 2); cudaMalloc(&dO, 128 * 64 * 4);
  cudaMemcpy(dA, A.data(), A.size() * 2, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, B.data(), B.size() * 2, cudaMemcpyHostToDevice);
  CUtensorMap ta, tb;
  cuuint64_t da[2] = {64, 256}, sa[1] = {128}; cuuint32_t box[2] = {64, 128}, es[2] = {1, 1};
  enc(&ta, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, dA, da, sa, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
      CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  cuuint64_t db[2] = {64, 64}; cuuint32_t boxb[2] = {64, 64};
  enc(&tb, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, dB, db, sa, boxb, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
      CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 100000);
  int shifts[] = {0, 1, 3, 5, 8, 13, 58, 117};
  std::vector<float> O(128 * 64);
  for (int mode = 0; mode < 3; ++mode)
    for (int s : shifts) {
      cudaMemset(dO, 0, 128 * 64 * 4);
      k<<<1, 256, 100000>>>(ta, tb, dA, dB, dO, s, mode);
      cudaError_t e = cudaDeviceSynchronize();
      if (e) { printf("mode %d shift %d: CUDA error %s\n", mode, s, cudaGetErrorString(e)); return 1; }
      cudaMemcpy(O.data(), dO, O.size() * 4, cudaMemcpyDeviceToHost);
      int bad = 0;
      for (int m = 0; m < 128; ++m) for (int n = 0; n < 64; ++n)
        if (O[m * 64 + n] != Af[(m + s) * 64 + n]) ++bad;
      printf("mode %d (%s) shift %3d: %s (%d mismatches)\n", mode,
             mode == 0 ? "SW128 base_off=0" : mode == 1 ? "SW128 base_off=row&7" : "NONE planar",
             s, bad ? "FAIL" : "ok", bad);
    }
  return 0;
}
