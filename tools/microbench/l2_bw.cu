// Micro-benchmark: L2 -> SM TMA read throughput (tiled 2D boxes of
// 128 rows x 128 B = 16 KB) from an L2-resident buffer, 148 CTAs.
// mode 0: each CTA reads its own region; mode 1: all CTAs read the same
// region (same lines at about the same time); mode 2: pairs of CTAs share.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <vector>
#include "sm100_ptx.cuh"
using namespace tec_sm100;

__device__ __forceinline__ bool try_nohint(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred P1;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2;\n\t"
      "selp.b32 %0, 1, 0, P1;\n\t}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ bool test_w(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred P1;\n\t"
      "mbarrier.test_wait.parity.shared::cta.b64 P1, [%1], %2;\n\t"
      "selp.b32 %0, 1, 0, P1;\n\t}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}
__device__ int g_wait_kind;
// issuers: thread i * tstride (i < nissuers) issues iterations i, i + n, ...
__global__ void __launch_bounds__(128, 1) k(const __grid_constant__ CUtensorMap tm, int iters,
                                            int rows_per_cta, int mode, long long* cyc,
                                            int box_rows, int kStages, int nissuers, int tstride) {
  extern __shared__ uint8_t raw[];
  uint8_t* sm = (uint8_t*)(((uintptr_t)raw + 1023) & ~(uintptr_t)1023);
  const int bbytes = box_rows * 128;
  uint64_t* full = (uint64_t*)(sm + 200 * 1024);
  if (threadIdx.x == 0) {
    for (int i = 0; i < kStages; ++i) mbar_init(&full[i], 1);
    fence_barrier_init();
  }
  __syncthreads();
  const int me = (int)threadIdx.x / tstride;
  if (tstride == 32 && me < nissuers && elect_one()) {
    int region = mode == 0 ? blockIdx.x : mode == 1 ? 0 : blockIdx.x / 2;
    int base = region * rows_per_cta;
    int nblk = rows_per_cta / box_rows;
    long long t0 = clock64();
    for (int it = me; it < iters + kStages; it += nissuers) {
      int s = it % kStages;
      if (it >= kStages) {
        const uint32_t ph = ((it / kStages) - 1) & 1;
        if (g_wait_kind == 0) mbar_wait(&full[s], ph);
        else if (g_wait_kind == 1) { while (!try_nohint(&full[s], ph)) {} }
        else { while (!test_w(&full[s], ph)) {} }
      }
      if (it < iters) {
        mbar_arrive_expect_tx(&full[s], bbytes);
        tma_load_2d(sm + s * bbytes, &tm, &full[s], 0, base + (it % nblk) * box_rows);
      }
    }
    if (me == 0) cyc[blockIdx.x] = clock64() - t0;
  }
}
__global__ void __launch_bounds__(256, 1) kldg(const uint4* buf, int iters, int rows_per_cta,
                                               long long* cyc, uint4* sink) {
  uint4 acc = make_uint4(0, 0, 0, 0);
  const uint4* p = buf + (size_t)blockIdx.x * rows_per_cta * 8;
  const int n = rows_per_cta * 8;
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll 8
    for (int j = 0; j < 8; ++j) {
      uint4 v = __ldcg(p + ((it * 8 + j) * 256 + threadIdx.x) % n);
      acc.x ^= v.x; acc.y ^= v.y; acc.z ^= v.z; acc.w ^= v.w;
    }
  }
  if (threadIdx.x == 0) cyc[blockIdx.x] = clock64() - t0;
  if (acc.x == 12345) sink[0] = acc;
}

int main() {
  typedef CUresult (*Enc)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                          const cuuint64_t*, const cuuint32_t*, const cuuint32_t*,
                          CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion,
                          CUtensorMapFloatOOBfill);
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  Enc enc = (Enc)fn;
  const int rows_per_cta = 1024;  // 128 KB per CTA region -> 19 MB total, L2 resident
  const size_t rows = (size_t)148 * rows_per_cta;
  void* buf;
  cudaMalloc(&buf, rows * 128);
  cudaMemset(buf, 1, rows * 128);
  CUtensorMap tm;
  cuuint64_t dims[2] = {64, rows};
  cuuint64_t strides[1] = {128};
  long long* d;
  cudaMalloc(&d, 148 * 8);
  const int smem = 200 * 1024 + 2048;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  struct V { int box_rows, stages, issuers, tstride; };
  std::vector<V> vs = {
    {128, 8, 1, 32}, {128, 12, 1, 32}, {256, 6, 1, 32}, {64, 16, 1, 32}, {128, 8, 2, 32}, {128, 8, 4, 32}, {128, 12, 4, 32},
  };
  int wk = 1;
  cudaMemcpyToSymbol(g_wait_kind, &wk, 4);
  for (const V& v : vs) {
    CUtensorMap tm;
    cuuint32_t box[2] = {64, (cuuint32_t)v.box_rows};
    cuuint32_t es[2] = {1, 1};
    CUresult r = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, buf, dims, strides, box, es,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                     CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r) { printf("encode %d\n", r); return 1; }
    const int iters = 2000 * 128 / v.box_rows;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    k<<<148, 128, smem>>>(tm, iters, rows_per_cta, 0, d, v.box_rows, v.stages, v.issuers, v.tstride);
    cudaEventRecord(e0);
    k<<<148, 128, smem>>>(tm, iters, rows_per_cta, 0, d, v.box_rows, v.stages, v.issuers, v.tstride);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    std::vector<long long> h(148);
    cudaMemcpy(h.data(), d, 148 * 8, cudaMemcpyDeviceToHost);
    double avg = 0;
    for (auto x : h) avg += x;
    avg /= 148;
    printf("box %3d rows stages %2d issuers %2d stride %2d: %.1f B/cycle/SM, %.2f TB/s chip\n",
           v.box_rows, v.stages, v.issuers, v.tstride, (double)iters * v.box_rows * 128 / avg,
           148.0 * iters * v.box_rows * 128 / (ms * 1e-3) / 1e12);
  }
  {
    uint4* sink; cudaMalloc(&sink, 64);
    const int iters = 4000;
    for (int rep = 0; rep < 2; ++rep)
      kldg<<<148, 256>>>((const uint4*)buf, iters, rows_per_cta, d, sink);
    cudaDeviceSynchronize();
    std::vector<long long> h(148);
    cudaMemcpy(h.data(), d, 148 * 8, cudaMemcpyDeviceToHost);
    double avg = 0;
    for (auto x : h) avg += x;
    avg /= 148;
    printf("LDG.128 256 threads: %.1f B/cycle/SM\n", (double)iters * 8 * 256 * 16 / avg);
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
