// f32tc MMA issue patterns without loads or epilogue (the C1 shape: 16 taps
// per tile, BN = 64): cycles per tile for
//   grp3   A_h x [B_h|B_m|B_l] (N=192) + A_m x [B_h|B_m] (N=128) + A_l x B_h
//   six    the six N=64 products
// with A at the shifted-window row offsets (tap (ri, sj) at row ri*WP + sj)
// or aligned (every tap at row 0), and B in the 32-B (3-D box) layout or
// the 128-B-row layout. Answers which of these costs the f32tc C1 kernel
// its missing tensor-core throughput.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#include "sm100_ptx.cuh"
using namespace tec_sm100;

__device__ __forceinline__ bool mbar_test_wait(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile("{\n\t.reg .pred P1;\n\tmbarrier.test_wait.parity.shared::cta.b64 P1, [%1], %2;\n\t"
               "selp.b32 %0, 1, 0, P1;\n\t}" : "=r"(ok) : "r"(smem_u32(bar)), "r"(parity) : "memory");
  return ok != 0;
}

__device__ __forceinline__ uint32_t rnd_bf16x2(uint32_t i) {
  // two finite bf16 values in [-2, 2) with random mantissas
  uint32_t h = i * 2654435761u;
  h ^= h >> 13; h *= 0x5bd1e995u; h ^= h >> 15;
  const uint32_t a = 0x3f80u | (h & 0x807fu), b = 0x3f80u | ((h >> 16) & 0x807fu);
  return a | (b << 16);
}

template <int BSW, bool kGrp, bool kShift, int kLayout = 0, int kCommits = 0>
__global__ void __launch_bounds__(128, 1) k(int tiles, int wp, long long* cyc, int random) {
  extern __shared__ uint8_t raw[];
  uint8_t* sm = (uint8_t*)(((uintptr_t)raw + 1023) & ~(uintptr_t)1023);
  uint8_t* sA = sm;                 // 64 KB halo (SW128 rows)
  uint8_t* sB = sm + 64 * 1024;     // 16 taps x 3 planes x 64 rows x BSW bytes
  uint64_t* bar = (uint64_t*)(sm + 200 * 1024);
  uint32_t* slot = (uint32_t*)(bar + 2);
  for (int i = threadIdx.x; i < 200 * 1024 / 16; i += blockDim.x)
    ((uint4*)sm)[i] = random ? make_uint4(rnd_bf16x2(4 * i), rnd_bf16x2(4 * i + 1), rnd_bf16x2(4 * i + 2),
                                          rnd_bf16x2(4 * i + 3))
                             : make_uint4(0x3f803f80u, 0, 0, 0);
  asm volatile("fence.proxy.async.shared::cta;");
  if (threadIdx.x == 0) { mbar_init(&bar[0], 1); mbar_init(&bar[1], 1); fence_barrier_init(); }
  if (threadIdx.x / 32 == 1) tmem_alloc<512>(slot);
  tc_fence_before(); __syncthreads(); tc_fence_after();
  const uint32_t tmem = *slot;
  if (threadIdx.x == 0) {
    constexpr uint32_t id64 = make_idesc<MmaKind::kF16>(128, 64);
    constexpr uint32_t id128 = make_idesc<MmaKind::kF16>(128, 128);
    constexpr uint32_t id192 = make_idesc<MmaKind::kF16>(128, 192);
    constexpr int kBPlane = 64 * BSW, kBTap = 3 * kBPlane;
    long long t0 = clock64();
    for (int t = 0; t < tiles; ++t) {
      for (int tap = 0; tap < 16; ++tap) {
        const int ri = tap / 4, sj = tap % 4;
        const uint32_t a = smem_u32(sA) + (kShift ? (ri * wp + sj) * 128 : 0);
        const uint32_t b = smem_u32(sB) + tap * kBTap;
        const uint64_t ah = make_smem_desc<128>(a, 1024), am = make_smem_desc<128>(a + 32, 1024),
                       al = make_smem_desc<128>(a + 64, 1024);
        const uint64_t bh = make_smem_desc<BSW>(b, 8 * BSW), bm = make_smem_desc<BSW>(b + kBPlane, 8 * BSW),
                       bl = make_smem_desc<BSW>(b + 2 * kBPlane, 8 * BSW);
        const uint32_t acc = tap ? 1u : 0u;
        if (kGrp && kLayout == 1) {
          // the kernel's GRP targets: X = [hh|hm|hl] (192 columns), the A_m
          // product onto X[64:192] and the A_l product onto X[64:128] --
          // overlapping accumulators of consecutive MMAs
          const uint32_t x = tmem + (t & 1) * 192;
          tc_mma<MmaKind::kF16>(x, ah, bh, id192, acc);
          tc_mma<MmaKind::kF16>(x + 64, am, bh, id128, 1u);
          tc_mma<MmaKind::kF16>(x + 64, al, bh, id64, 1u);
        } else if (kGrp && kLayout == 2) {
          // reordered: the A_l product first (X[64:128]), then A_h (all of
          // X), then A_m (X[64:192])
          const uint32_t x = tmem + (t & 1) * 192;
          tc_mma<MmaKind::kF16>(x + 64, al, bh, id64, tap ? 1u : 0u);
          tc_mma<MmaKind::kF16>(x, ah, bh, id192, 1u);
          tc_mma<MmaKind::kF16>(x + 64, am, bh, id128, 1u);
        } else if (kGrp) {
          tc_mma<MmaKind::kF16>(tmem, ah, bh, id192, acc);
          tc_mma<MmaKind::kF16>(tmem + 192, am, bh, id128, acc);
          tc_mma<MmaKind::kF16>(tmem + 192, al, bh, id64, 1u);
        } else {
          tc_mma<MmaKind::kF16>(tmem, ah, bh, id64, acc);
          tc_mma<MmaKind::kF16>(tmem + 64, ah, bm, id64, acc);
          tc_mma<MmaKind::kF16>(tmem + 64, am, bh, id64, 1u);
          tc_mma<MmaKind::kF16>(tmem + 64, ah, bl, id64, 1u);
          tc_mma<MmaKind::kF16>(tmem + 64, al, bh, id64, 1u);
          tc_mma<MmaKind::kF16>(tmem + 64, am, bm, id64, 1u);
        }
      }
      // kCommits per tile: tcgen05.commit to an mbarrier nobody waits on
      // (the kernel commits the chunk and the released halo rows per tile)
      for (int c = 0; c < kCommits; ++c) tc_commit(&bar[1]);
    }
    tc_commit(&bar[0]);
    mbar_wait(&bar[0], 0);
    cyc[blockIdx.x] = clock64() - t0;
  }
  tc_fence_before(); __syncthreads(); tc_fence_after();
  if (threadIdx.x / 32 == 1) tmem_dealloc<512>(tmem);
}

// The kernel's chunk handshake: the MMA thread commits sfull[b] per tile
// and, before tile t, waits sempty[b] (arrived by 256 "epilogue" threads
// once they see sfull[b] of tile t - 2) -- no TMEM reads.
__global__ void __launch_bounds__(384, 1) hs(int tiles, long long* cyc, int sleep_wait, int tap_waits = 0) {
  extern __shared__ uint8_t raw[];
  uint8_t* sm = (uint8_t*)(((uintptr_t)raw + 1023) & ~(uintptr_t)1023);
  uint8_t* sA = sm;
  uint8_t* sB = sm + 64 * 1024;
  uint64_t* bar = (uint64_t*)(sm + 200 * 1024);
  uint64_t* sfull = bar + 2;
  uint64_t* sempty = bar + 4;
  uint32_t* slot = (uint32_t*)(bar + 8);
  for (int i = threadIdx.x; i < 200 * 1024 / 16; i += blockDim.x)
    ((uint4*)sm)[i] = make_uint4(rnd_bf16x2(4 * i), rnd_bf16x2(4 * i + 1), rnd_bf16x2(4 * i + 2), rnd_bf16x2(4 * i + 3));
  asm volatile("fence.proxy.async.shared::cta;");
  if (threadIdx.x == 0) {
    mbar_init(&bar[0], 1);
    for (int i = 0; i < 2; ++i) { mbar_init(&sfull[i], 1); mbar_init(&sempty[i], 256); }
    mbar_init(&bar[1], 1);
    fence_barrier_init();
    mbar_arrive(&bar[1]);  // phase 0 completes
  }
  if (threadIdx.x / 32 == 2) tmem_alloc<512>(slot);
  tc_fence_before(); __syncthreads(); tc_fence_after();
  const uint32_t tmem = *slot;
  const int warp = threadIdx.x / 32;
  if (warp == 1 && elect_one()) {
    constexpr uint32_t id64 = make_idesc<MmaKind::kF16>(128, 64);
    constexpr uint32_t id128 = make_idesc<MmaKind::kF16>(128, 128);
    constexpr uint32_t id192 = make_idesc<MmaKind::kF16>(128, 192);
    long long t0 = clock64();
    for (int t = 0; t < tiles; ++t) {
      const int b = t & 1;
      mbar_wait(&sempty[b], ((t >> 1) & 1) ^ 1);
      tc_fence_after();
      const uint32_t x = tmem + b * 192;
      for (int tap = 0; tap < 16; ++tap) {
        const int ri = tap / 4, sj = tap % 4;
        const uint32_t a = smem_u32(sA) + (ri * 115 + sj) * 128;
        const uint32_t bb = smem_u32(sB) + tap * 6144;
        const uint64_t ah = make_smem_desc<128>(a, 1024);
        const uint64_t bh = make_smem_desc<32>(bb, 256);
        tc_mma<MmaKind::kF16>(x, ah, bh, id192, tap ? 1u : 0u);
        tc_mma<MmaKind::kF16>(x + 64, ah + 2, bh, id128, 1u);
        tc_mma<MmaKind::kF16>(x + 64, ah + 4, bh, id64, 1u);
        // the kernels' per-stage operand wait, on an already completed phase
        for (int w = 0; w < tap_waits; ++w) {
          mbar_wait(&bar[1], 0);
          tc_fence_after();
        }
      }
      tc_commit(&sfull[b]);
    }
    tc_commit(&bar[0]);
    mbar_wait(&bar[0], 0);
    cyc[blockIdx.x] = clock64() - t0;
  } else if (warp >= 4) {
    for (int t = 0; t < tiles; ++t) {
      const int b = t & 1;
      if (sleep_wait) mbar_wait(&sfull[b], (t >> 1) & 1);
      else while (!mbar_test_wait(&sfull[b], (t >> 1) & 1)) {}
      tc_fence_before();
      mbar_arrive(&sempty[b]);
    }
  }
  tc_fence_before(); __syncthreads(); tc_fence_after();
  if (warp == 2) tmem_dealloc<512>(tmem);
}

void run_hs(const char* name, int sleep_wait, int tap_waits = 0) {
  long long* d; cudaMalloc(&d, 148 * 8);
  const int smem = 200 * 1024 + 2048;
  cudaFuncSetAttribute(hs, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int tiles = 200;
  hs<<<148, 384, smem>>>(tiles, d, sleep_wait, tap_waits);
  long long h[148];
  if (cudaDeviceSynchronize() != cudaSuccess) { printf("%s: kernel failed\n", name); exit(1); }
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  long long mx = 0;
  for (int i = 0; i < 148; ++i) mx = h[i] > mx ? h[i] : mx;
  printf("%-44s %8.1f cycles/tile (16 taps), %6.1f per tap\n", name, (double)mx / tiles, (double)mx / tiles / 16);
  cudaFree(d);
}

template <int BSW, bool kGrp, bool kShift, int kLayout = 0, int kCommits = 0>
void run(const char* name, int random = 0) {
  long long* d; cudaMalloc(&d, 148 * 8);
  auto f = k<BSW, kGrp, kShift, kLayout, kCommits>;
  const int smem = 200 * 1024 + 2048;
  cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int tiles = 200;
  f<<<148, 128, smem>>>(tiles, 115, d, random);
  if (cudaDeviceSynchronize() != cudaSuccess) { printf("%s: kernel failed\n", name); exit(1); }
  long long h[148]; cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  printf("%-44s %8.1f cycles/tile (16 taps), %6.1f per tap\n", name, (double)h[0] / tiles, (double)h[0] / tiles / 16);
  cudaFree(d);
}

int main() {
  run_hs("handshake + 1 completed-barrier wait per tap", 1, 1);
  run_hs("handshake + 2 completed-barrier waits per tap", 1, 2);
  run_hs("handshake sfull/sempty, sleeping waits", 1);
  run_hs("handshake sfull/sempty, spinning waits", 0);
  run<32, true, true, 1, 1>("grp3, X targets, 1 commit per tile", 1);
  run<32, true, true, 1, 2>("grp3, X targets, 2 commits per tile", 1);
  run<32, true, true, 1>("grp3, the kernel's overlapping X targets", 1);
  run<32, true, true, 2>("grp3, overlapping targets, A_l first", 1);
  run<32, true, true>("grp3, B 32-B rows, A shifted, RANDOM data", 1);
  run<32, false, true>("six N=64, B 32-B rows, A shifted, RANDOM data", 1);
  run<32, true, true>("grp3, B 32-B rows, A shifted (C1 halo)");
  run<32, true, false>("grp3, B 32-B rows, A aligned");
  run<128, true, true>("grp3, B 128-B rows, A shifted");
  run<128, true, false>("grp3, B 128-B rows, A aligned");
  run<32, false, true>("six N=64, B 32-B rows, A shifted");
  run<128, false, false>("six N=64, B 128-B rows, A aligned");
  return 0;
}
