// Halo-kernel MMA pattern micro-benchmark (no loads, no epilogue): per "tile",
// TAPS taps x MS sub-tiles x KK k-steps; A start shifts by (rh*WP + rw) rows,
// B advances one weight tile per tap (resident weights). Compare cycles/MMA
// with the static-operand rate of mma_rate.cu.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include "sm100_ptx.cuh"
using namespace tec_sm100;
template <int SWZ, int MS, int KK, int R, int BN, bool kCommit, bool kKOuter = false, bool kResetB = true, int ACCS = BN, bool kMsOuter = false>
__global__ void __launch_bounds__(128, 1) k(int tiles, int wp, long long* cyc, int boff, int aoff, int bstride) {
  extern __shared__ uint8_t raw[];
  uint8_t* sm = (uint8_t*)(((uintptr_t)raw + 1023) & ~(uintptr_t)1023);
  uint8_t* sA = sm + aoff;          // halo: up to 96 KB (aoff: base shift)
  uint8_t* sB = sm + 96 * 1024 + boff;  // weights: R*R*BN*SWZ (boff: base shift, bytes)
  uint64_t* bar = (uint64_t*)(sm + 200 * 1024);
  uint32_t* slot = (uint32_t*)(bar + 2);
  static_assert((kResetB ? R : R * R) * BN * SWZ <= 72 * 1024, "B tiles must fit the B region");
  if (boff > 32 * 1024 || aoff > 32 * 1024) return;
  if (bstride && (kResetB ? R : R * R) * bstride + boff > 104 * 1024) return;
  for (int i = threadIdx.x; i < 200 * 1024 / 16; i += blockDim.x)
    ((uint4*)sm)[i] = make_uint4(0x3f803f80u, 0, 0, 0);
  asm volatile("fence.proxy.async.shared::cta;");
  if (threadIdx.x == 0) { mbar_init(&bar[0], 1); mbar_init(&bar[1], 1); fence_barrier_init(); }
  if (threadIdx.x / 32 == 1) tmem_alloc<512>(slot);
  tc_fence_before(); __syncthreads(); tc_fence_after();
  uint32_t tmem = *slot;
  if (threadIdx.x == 0) {
    constexpr uint32_t idesc = make_idesc<MmaKind::kF16>(128, BN);
    const uint64_t a0 = make_smem_desc<SWZ>(smem_u32(sA), 8 * SWZ);
    const uint64_t b0 = make_smem_desc<SWZ>(smem_u32(sB), 8 * SWZ);
    const uint32_t row_skip = (uint32_t)((wp - R) * SWZ) >> 4;
    long long t0 = clock64();
    for (int t = 0; t < tiles; ++t) {
      const uint32_t d0 = tmem + (t & 1) * MS * ACCS;
      if constexpr (kMsOuter) {
        for (int ms = 0; ms < MS; ++ms) {
          uint64_t ad = a0 + ((ms * 128 * SWZ) >> 4), bd = b0;
          uint32_t accum = 0;
          for (int rh = 0; rh < R; ++rh) {
            for (int rw = 0; rw < R; ++rw) {
#pragma unroll
              for (int kk = 0; kk < KK; ++kk)
                tc_mma<MmaKind::kF16>(d0 + ms * ACCS, ad + ((kk * 32) >> 4), bd + ((kk * 32) >> 4),
                                      idesc, kk == 0 ? accum : 1u);
              accum = 1;
              ad += SWZ >> 4;
              bd += (bstride ? bstride : BN * SWZ) >> 4;
            }
            ad += row_skip;
            if (kResetB) bd = b0;
          }
        }
        if (kCommit) tc_commit(&bar[t & 1]);
        continue;
      }
      uint64_t ad = a0, bd = b0;
      uint32_t accum = 0;
      for (int rh = 0; rh < R; ++rh) {
        for (int rw = 0; rw < R; ++rw) {
          if constexpr (kKOuter) {
#pragma unroll
            for (int kk = 0; kk < KK; ++kk)
#pragma unroll
              for (int ms = 0; ms < MS; ++ms)
                tc_mma<MmaKind::kF16>(d0 + ms * ACCS, ad + ((ms * 128 * SWZ + kk * 32) >> 4),
                                      bd + ((kk * 32) >> 4), idesc, kk == 0 ? accum : 1u);
          } else {
#pragma unroll
            for (int ms = 0; ms < MS; ++ms)
#pragma unroll
              for (int kk = 0; kk < KK; ++kk)
                tc_mma<MmaKind::kF16>(d0 + ms * ACCS, ad + ((ms * 128 * SWZ + kk * 32) >> 4),
                                      bd + ((kk * 32) >> 4), idesc, kk == 0 ? accum : 1u);
          }
          accum = 1;
          ad += SWZ >> 4;
          bd += (bstride ? bstride : BN * SWZ) >> 4;
        }
        ad += row_skip;
        if (kResetB) bd = b0;  // one filter row of weight tiles, reused
      }
      if (kCommit) tc_commit(&bar[t & 1]);
    }
    tc_commit(&bar[0]);
    long long t1 = clock64();
    cyc[blockIdx.x] = t1 - t0;
    // drain
    mbar_wait(&bar[0], (kCommit ? ((tiles + 1) / 2) : 0) & 1);
  }
  tc_fence_before(); __syncthreads(); tc_fence_after();
  if (threadIdx.x / 32 == 1) tmem_dealloc<512>(tmem);
}
template <int SWZ, int MS, int KK, int R, int BN, bool kC, bool kKO = false, bool kRB = true, int ACCS = BN, bool kMO = false>
void run(const char* name, int wp, int boff = 0, int aoff = 0, int bstride = 0) {
  long long* d; cudaMalloc(&d, 148 * 8);
  auto f = k<SWZ, MS, KK, R, BN, kC, kKO, kRB, ACCS, kMO>;
  const int smem = 200 * 1024 + 2048;
  cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int tiles = 400;
  f<<<148, 128, smem>>>(tiles, wp, d, boff, aoff, bstride);
  if (cudaDeviceSynchronize() != cudaSuccess) { printf("%s: kernel failed\n", name); exit(1); }
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  f<<<148, 128, smem>>>(tiles, wp, d, boff, aoff, bstride);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  const double mmas = (double)tiles * R * R * MS * KK;
  printf("%s boff=%d aoff=%d bstride=%d: %.1f us, %.1f ns/MMA/SM -> %.2f GHz-equiv at 54 cyc  (%s)\n", name, boff, aoff, bstride, ms * 1e3,
         ms * 1e6 / mmas, 54.0 / (ms * 1e6 / mmas), cudaGetErrorString(cudaGetLastError()));
  long long h[148]; cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  printf("   issue-side cycles/MMA (thread 0 loop) %.1f\n", (double)h[0] / mmas);
  cudaFree(d);
}
int main() {
  run<128, 2, 4, 3, 64, true, false, false>("C2 MS2 B72KB (ms inside the tap loop)", 58);
  run<128, 2, 4, 3, 64, true, false, false, 64, true>("C2 MS2 B72KB (ms outermost)", 58);
  run<128, 1, 4, 3, 64, true, false, false>("C2 MS1 B72KB", 58);
  run<32, 4, 1, 4, 64, true, false, false>("C1 MS4 SW32 B32KB (ms inside)", 116);
  run<32, 4, 1, 4, 64, true, false, false, 64, true>("C1 MS4 SW32 B32KB (ms outermost)", 116);
  return 0;
}
