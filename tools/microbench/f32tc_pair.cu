// The f32tc BN=128 main loop (six N=128 products per K16 slice, A and B in
// three bf16 planes, a 2-stage TMA ring of 64-channel k-iterations) with and
// without a CTA pair (cta_group::2, M = 256: each CTA loads its own 128 A
// rows and HALF of the B rows; the leader issues the MMAs, both CTAs' TMA
// bytes land on the leader's full barrier, the commit multicasts the stage
// release to both). Measures MMA-thread cycles per K16 slice with the real
// TMA traffic into shared memory (LOAD) and without it, to size how much of
// the f32tc layers' time is the shared-memory bandwidth the operand reads
// and the TMA writes share.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include "sm100_ptx.cuh"
using namespace tec_sm100;

__device__ __forceinline__ void mma2(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
      "l"(a), "l"(b), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void commit2_mc(uint64_t* bar, uint16_t mask) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;"
      ::"r"(smem_u32(bar)), "h"(mask) : "memory");
}

template <bool PAIR, bool LOAD, int BN = 128, int PROD = 6, int NST = 2>
__global__ void __launch_bounds__(128, 1) k(const __grid_constant__ CUtensorMap tm16,
                                            const __grid_constant__ CUtensorMap tm8,
                                            const __grid_constant__ CUtensorMap tm4, int iters,
                                            long long* cyc) {
  extern __shared__ uint8_t raw[];
  uint8_t* sm = (uint8_t*)(((uintptr_t)raw + 1023) & ~(uintptr_t)1023);
  constexpr int kA = 16384, kBP = (PAIR ? BN / 2 : BN) * 128;
  constexpr int kPl = PROD == 1 ? 1 : 3;  // operand planes (f32tc: h, m, l)
  // grouped (PROD 3, BN 64): a pair CTA holds R1 = its half of [h m l] (rank
  // order h m l / m l h) + R2 = its half of [h m] -- 5 boxes of 32 rows
  constexpr int kBBoxes = PROD == 3 && PAIR ? 5 : kPl;
  constexpr int kStage = kPl * kA + kBBoxes * kBP;
  uint64_t* bars = (uint64_t*)(sm + NST * kStage);
  uint64_t* full = bars;
  uint64_t* empty = bars + NST;
  uint64_t* done = bars + 2 * NST;
  uint32_t* slot = (uint32_t*)(bars + 2 * NST + 1);
  const uint32_t rank = PAIR ? cluster_ctarank() : 0;
  const int warp = threadIdx.x / 32;
  if (threadIdx.x == 0) {
    for (int i = 0; i < NST; ++i) { mbar_init(&full[i], 1); mbar_init(&empty[i], 1); }
    mbar_init(done, 1);
    fence_barrier_init();
  }
  if (warp == 2) {
    if (PAIR) {
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(slot)));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    } else {
      tmem_alloc<512>(slot);
    }
  }
  tc_fence_before();
  if (PAIR) cluster_sync(); else __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *slot;
  if (warp == 0 && elect_one()) {
    const uint32_t full_leader0 = PAIR ? mapa_u32(smem_u32(&full[0]), 0) : 0;
    for (int it = 0; it < iters; ++it) {
      const int s = it % NST;
      if (it >= NST) mbar_wait(&empty[s], ((it / NST) - 1) & 1);
      uint8_t* st = sm + s * kStage;
      if (rank == 0) {
        if (LOAD) mbar_arrive_expect_tx(&full[s], (PAIR ? 2 : 1) * kStage);
        else mbar_arrive(&full[s]);
      }
      if (LOAD) {
        const int base = (blockIdx.x / (PAIR ? 2 : 1)) * 37 + it * 11;
        for (int pl = 0; pl < kBBoxes; ++pl) {
          const int ra = ((base + pl * 5 + rank * 3) % 1000) * 128;
          const int rb = ((base + pl * 7 + 500) % 1000) * 128 + (PAIR ? rank * (BN / 2) : 0);
          if (PAIR) {
            const uint32_t fb = full_leader0 + s * 8;
            if (pl < kPl) tma_load_2d_pair(st + pl * kA, &tm16, fb, 0, ra);
            tma_load_2d_pair(st + kPl * kA + pl * kBP, BN == 128 ? &tm8 : &tm4, fb, 0, rb);
          } else {
            if (pl < kPl) tma_load_2d(st + pl * kA, &tm16, &full[s], 0, ra);
            tma_load_2d(st + kPl * kA + pl * kBP, BN == 128 ? &tm16 : &tm8, &full[s], 0, rb);
          }
        }
      }
    }
  } else if (warp == 1 && rank == 0 && elect_one()) {
    constexpr uint32_t id = make_idesc<MmaKind::kF16>(PAIR ? 256 : 128, BN);
    const uint32_t S = tmem, T = tmem + 128;
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
      const int s = it % NST;
      mbar_wait(&full[s], (it / NST) & 1);
      tc_fence_after();
      const uint32_t a = smem_u32(sm + s * kStage), b = a + kPl * kA;
      for (int kk = 0; kk < 4; ++kk) {
        const uint64_t ah = make_smem_desc<128>(a + kk * 32, 1024), am = make_smem_desc<128>(a + kA + kk * 32, 1024),
                       al = make_smem_desc<128>(a + 2 * kA + kk * 32, 1024);
        const uint64_t bh = make_smem_desc<128>(b + kk * 32, 1024), bm = make_smem_desc<128>(b + kBP + kk * 32, 1024),
                       bl = make_smem_desc<128>(b + 2 * kBP + kk * 32, 1024);
        const uint32_t acc = (it | kk) ? 1u : 0u;
        if (PROD == 1) {
          if (PAIR) mma2(S, ah, bh, id, acc); else tc_mma<MmaKind::kF16>(S, ah, bh, id, acc);
        } else if (PROD == 3) {
          // X = [hh0 hm0 hl0 hm1 hl1 hh1] (pair) / [hh hm hl] (one CTA)
          constexpr uint32_t i3 = make_idesc<MmaKind::kF16>(PAIR ? 256 : 128, 3 * BN);
          constexpr uint32_t i2 = make_idesc<MmaKind::kF16>(PAIR ? 256 : 128, 2 * BN);
          constexpr uint32_t i1 = make_idesc<MmaKind::kF16>(PAIR ? 256 : 128, BN);
          if (PAIR) {
            const uint64_t r2 = make_smem_desc<128>(b + 3 * kBP + kk * 32, 1024);
            mma2(S, ah, bh, i3, acc);
            mma2(S + BN / 2, am, r2, i2, 1u);
            mma2(S + BN, al, r2, i1, 1u);
          } else {
            tc_mma<MmaKind::kF16>(S, ah, bh, i3, acc);
            tc_mma<MmaKind::kF16>(S + BN, am, bh, i2, 1u);
            tc_mma<MmaKind::kF16>(S + BN, al, bh, i1, 1u);
          }
        } else if (PAIR) {
          mma2(S, ah, bh, id, acc); mma2(T, ah, bm, id, acc); mma2(T, am, bh, id, 1u);
          mma2(T, ah, bl, id, 1u); mma2(T, al, bh, id, 1u); mma2(T, am, bm, id, 1u);
        } else {
          tc_mma<MmaKind::kF16>(S, ah, bh, id, acc); tc_mma<MmaKind::kF16>(T, ah, bm, id, acc);
          tc_mma<MmaKind::kF16>(T, am, bh, id, 1u); tc_mma<MmaKind::kF16>(T, ah, bl, id, 1u);
          tc_mma<MmaKind::kF16>(T, al, bh, id, 1u); tc_mma<MmaKind::kF16>(T, am, bm, id, 1u);
        }
      }
      if (PAIR) commit2_mc(&empty[s], 3); else tc_commit(&empty[s]);
    }
    if (PAIR) commit2_mc(done, 1); else tc_commit(done);
    mbar_wait(done, 0);
    cyc[blockIdx.x] = clock64() - t0;
  }
  tc_fence_before();
  if (PAIR) cluster_sync(); else __syncthreads();
  tc_fence_after();
  if (warp == 2) {
    if (PAIR) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tmem));
    else tmem_dealloc<512>(tmem);
  }
}

static CUtensorMap make_map(void* base, int rows, int box_rows) {
  CUtensorMap m;
  cuuint64_t dims[2] = {64, (cuuint64_t)rows};
  cuuint64_t strides[1] = {128};
  cuuint32_t box[2] = {64, (cuuint32_t)box_rows};
  cuuint32_t es[2] = {1, 1};
  CUresult r = cuTensorMapEncodeTiled(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, base, dims, strides, box, es,
                                      CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                      CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) { printf("encode failed %d\n", (int)r); exit(1); }
  return m;
}

template <bool PAIR, bool LOAD, int BN = 128, int PROD = 6, int NST = 2>
void run(const char* name, const CUtensorMap& m16, const CUtensorMap& m8, const CUtensorMap& m4) {
  auto f = k<PAIR, LOAD, BN, PROD, NST>;
  constexpr int kPl = PROD == 1 ? 1 : 3;
  constexpr int kStage = kPl * 16384 + (PROD == 3 && PAIR ? 5 : kPl) * (PAIR ? BN / 2 : BN) * 128;
  const int smem = NST * kStage + 2048;
  cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  long long* d; cudaMalloc(&d, 148 * 8); cudaMemset(d, 0, 148 * 8);
  const int iters = 400;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(148); cfg.blockDim = dim3(128); cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = PAIR ? 2 : 1; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
  cfg.attrs = at; cfg.numAttrs = 1;
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaLaunchKernelEx(&cfg, f, m16, m8, m4, iters, d);  // warm
  cudaEventRecord(e0);
  cudaLaunchKernelEx(&cfg, f, m16, m8, m4, iters, d);
  cudaEventRecord(e1);
  cudaError_t err = cudaDeviceSynchronize();
  if (err != cudaSuccess) { printf("%s: %s\n", name, cudaGetErrorString(err)); exit(1); }
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  std::vector<long long> h(148); cudaMemcpy(h.data(), d, 148 * 8, cudaMemcpyDeviceToHost);
  long long mx = 0; for (auto v : h) mx = v > mx ? v : mx;
  // per SM: iters x 4 K16 slices of a 128-row tile x N=128 x 6 products
  const double flops = 148.0 * iters * 4 * (PROD == 3 ? 6 : PROD) * 2.0 * 128 * BN * 16;
  printf("%-44s %7.1f cycles per K16 (ideal %d), %6.0f bf16 TFLOP/s\n", name, (double)mx / (iters * 4), PROD * BN / 2,
         flops / (ms * 1e-3) / 1e12);
  cudaFree(d);
}

int main() {
  const int rows = 131072;  // 16 MB of bf16 rows of 128 B (L2-resident)
  void* buf; cudaMalloc(&buf, (size_t)rows * 128);
  std::vector<uint16_t> h((size_t)rows * 64);
  for (size_t i = 0; i < h.size(); ++i) h[i] = 0x3f80 | (uint16_t)((i * 2654435761u >> 7) & 0x807f);
  cudaMemcpy(buf, h.data(), h.size() * 2, cudaMemcpyHostToDevice);
  CUtensorMap m16 = make_map(buf, rows, 128), m8 = make_map(buf, rows, 64), m4 = make_map(buf, rows, 32);
  run<false, false>("f32tc N=128: 1 CTA, no loads", m16, m8, m4);
  run<false, true>("f32tc N=128: 1 CTA, A 48 KB + B 48 KB / stage", m16, m8, m4);
  run<true, false>("f32tc N=128: CTA pair, no loads", m16, m8, m4);
  run<true, true>("f32tc N=128: CTA pair, A 48 KB + B 24 KB / CTA", m16, m8, m4);
  run<false, false, 64, 3>("f32tc grouped N=64: 1 CTA, no loads", m16, m8, m4);
  run<false, true, 64, 3>("f32tc grouped N=64: 1 CTA, A 48 KB + B 24 KB", m16, m8, m4);
  run<true, false, 64, 3>("f32tc grouped N=64: CTA pair, no loads", m16, m8, m4);
  run<true, true, 64, 3>("f32tc grouped N=64: CTA pair, A 48 KB + B 20 KB", m16, m8, m4);
  run<false, false, 64, 1, 8>("bf16 N=64 x8 stages: 1 CTA, no loads", m16, m8, m4);
  run<false, true, 64, 1, 8>("bf16 N=64 x8: 1 CTA, A 16 KB + B 8 KB", m16, m8, m4);
  run<true, false, 64, 1, 8>("bf16 N=64 x8: CTA pair, no loads", m16, m8, m4);
  run<true, true, 64, 1, 8>("bf16 N=64 x8: CTA pair, A 16 KB + B 4 KB", m16, m8, m4);
  run<false, true, 128, 1, 6>("bf16 N=128 x6: 1 CTA, A 16 KB + B 16 KB", m16, m8, m4);
  run<true, true, 128, 1, 6>("bf16 N=128 x6: CTA pair, A 16 KB + B 8 KB", m16, m8, m4);
  return 0;
}
