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

template <int BSW, bool kGrp, bool kShift>
__global__ void __launch_bounds__(128, 1) k(int tiles, int wp, long long* cyc) {
  extern __shared__ uint8_t raw[];
  uint8_t* sm = (uint8_t*)(((uintptr_t)raw + 1023) & ~(uintptr_t)1023);
  uint8_t* sA = sm;                 // 64 KB halo (SW128 rows)
  uint8_t* sB = sm + 64 * 1024;     // 16 taps x 3 planes x 64 rows x BSW bytes
  uint64_t* bar = (uint64_t*)(sm + 200 * 1024);
  uint32_t* slot = (uint32_t*)(bar + 2);
  for (int i = threadIdx.x; i < 200 * 1024 / 16; i += blockDim.x)
    ((uint4*)sm)[i] = make_uint4(0x3f803f80u, 0, 0, 0);
  asm volatile("fence.proxy.async.shared::cta;");
  if (threadIdx.x == 0) { mbar_init(&bar[0], 1); fence_barrier_init(); }
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
        if (kGrp) {
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
    }
    tc_commit(&bar[0]);
    mbar_wait(&bar[0], 0);
    cyc[blockIdx.x] = clock64() - t0;
  }
  tc_fence_before(); __syncthreads(); tc_fence_after();
  if (threadIdx.x / 32 == 1) tmem_dealloc<512>(tmem);
}

template <int BSW, bool kGrp, bool kShift>
void run(const char* name) {
  long long* d; cudaMalloc(&d, 148 * 8);
  auto f = k<BSW, kGrp, kShift>;
  const int smem = 200 * 1024 + 2048;
  cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int tiles = 200;
  f<<<148, 128, smem>>>(tiles, 115, d);
  if (cudaDeviceSynchronize() != cudaSuccess) { printf("%s: kernel failed\n", name); exit(1); }
  long long h[148]; cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  printf("%-44s %8.1f cycles/tile (16 taps), %6.1f per tap\n", name, (double)h[0] / tiles, (double)h[0] / tiles / 16);
  cudaFree(d);
}

int main() {
  run<32, true, true>("grp3, B 32-B rows, A shifted (C1 halo)");
  run<32, true, false>("grp3, B 32-B rows, A aligned");
  run<128, true, true>("grp3, B 128-B rows, A shifted");
  run<128, true, false>("grp3, B 128-B rows, A aligned");
  run<32, false, true>("six N=64, B 32-B rows, A shifted");
  run<128, false, false>("six N=64, B 128-B rows, A aligned");
  return 0;
}
