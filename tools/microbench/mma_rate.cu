// Micro-benchmark: tcgen05.mma (kind::f16, cta_group::1, SS operands)
// throughput per SM vs N and A-start alignment. 148 CTAs, each issues
// ITERS x 4 MMAs (K=16 each) back to back from one thread on static smem.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include "sm100_ptx.cuh"
using namespace tec_sm100;

template <int N, int SWZ, int NACC = 1, int M = 128, MmaKind KIND = MmaKind::kF16>
__global__ void __launch_bounds__(128, 1) k(int iters, int shift_rows, long long* cyc) {
  extern __shared__ uint8_t raw[];
  uint8_t* sm = (uint8_t*)(((uintptr_t)raw + 1023) & ~(uintptr_t)1023);
  uint8_t* sA = sm;              // 512 rows x 128 B
  uint8_t* sB = sm + 65536;      // 256 rows x 128 B
  uint64_t* bar = (uint64_t*)(sm + 65536 + 32768);
  uint32_t* slot = (uint32_t*)(bar + 1);
  int warp = threadIdx.x / 32;
  for (int i = threadIdx.x; i < (65536 + 32768) / 16; i += blockDim.x)
    ((uint4*)sm)[i] = make_uint4(0x3f803f80u, 0, 0, 0);
  asm volatile("fence.proxy.async.shared::cta;");
  if (threadIdx.x == 0) { mbar_init(bar, 1); fence_barrier_init(); }
  if (warp == 1) tmem_alloc<512>(slot);
  tc_fence_before(); __syncthreads(); tc_fence_after();
  uint32_t tmem = *slot;
  if (threadIdx.x == 0) {
    uint32_t idesc = make_idesc<KIND>(M, N);
    long long t0 = clock64();
    uint32_t a0 = smem_u32(sA) + shift_rows * 128, b0 = smem_u32(sB);
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int kk = 0; kk < 4; ++kk) {
        uint64_t ad = SWZ == 128 ? make_smem_desc<128>(a0 + (it & 1) * 16384 + kk * 32, 1024)
                                 : make_smem_desc<SWZ>(a0 + (it & 1) * 16384 + kk * 128 * SWZ, 8 * SWZ);
        uint64_t bd = SWZ == 128 ? make_smem_desc<128>(b0 + kk * 32, 1024)
                                 : make_smem_desc<SWZ>(b0 + kk * 256 * SWZ, 8 * SWZ);
        tc_mma<KIND>(tmem + (NACC > 1 ? (kk % NACC) * N : 0), ad, bd, idesc, 1);
      }
    }
    tc_commit(bar);
    mbar_wait(bar, 0);
    long long t1 = clock64();
    cyc[blockIdx.x] = t1 - t0;
  }
  tc_fence_before(); __syncthreads(); tc_fence_after();
  if (warp == 1) tmem_dealloc<512>(tmem);
}

template <int N, int SWZ = 128, int NACC = 1, int M = 128, MmaKind KIND = MmaKind::kF16>
void run(int shift) {
  long long* d; cudaMalloc(&d, 148 * 8);
  auto f = k<N, SWZ, NACC, M, KIND>;
  cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, 110000);
  int iters = 4000;
  f<<<148, 128, 110000>>>(iters, shift, d);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  f<<<148, 128, 110000>>>(iters, shift, d);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  long long h[148]; cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  const int kdim = KIND == MmaKind::kI8 ? 32 : 16;  // 32 bytes of K per MMA either way
  double flops = 2.0 * M * N * kdim * 4 * (double)iters * 148;
  printf("%s M=%d N=%3d shift=%d SWZ=%d NACC=%d: %.1f cycles/MMA (ideal %d), %.0f T(FL)OP/s\n",
         KIND == MmaKind::kI8 ? "i8  " : "bf16", M, N, shift, SWZ, NACC, (double)h[0] / (iters * 4),
         KIND == MmaKind::kI8 ? M * N / 512 : M * N / 256, flops / (ms * 1e-3) / 1e12);
  cudaFree(d);
}

int main() {
  run<64, 128, 1, 128, MmaKind::kI8>(0); run<128, 128, 1, 128, MmaKind::kI8>(0);
  run<256, 128, 1, 128, MmaKind::kI8>(0);
  run<64, 128, 1>(0); run<128, 128, 1>(0); run<256, 128, 1>(0);
  run<64, 128, 1, 64>(0); run<128, 128, 1, 64>(0); run<256, 128, 1, 64>(0); run<256, 128, 2, 64>(0);
  return 0;
}
