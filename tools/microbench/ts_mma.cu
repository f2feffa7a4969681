// A operand from tensor memory (tcgen05.mma ... [a_tmem], the "ts" form)
// for the f32tc products: (1) correctness -- A staged smem -> TMEM with
// tcgen05.cp.128x256b (one K16 slice of a 128-B-swizzled K-major tile per
// copy) then ts-MMAs must equal the ss-MMAs bit for bit; (2) rate -- the six
// N=128 products of one K16 step (hh hm mh hl lh mm) with A read from shared
// memory six times (ss) vs copied once per plane and read from TMEM (ts):
// the ss form moves 48 KB of operands per step through the tensor core's
// shared-memory path (~128 B/cycle, its limit), the ts form 3 KB + 24 KB.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include "sm100_ptx.cuh"
using namespace tec_sm100;

// smem: A planes h, m, l (3 x 16 KB: 128 rows x 64 bf16, SW128 K-major),
// B planes h, m, l (3 x 16 KB: 128 rows x 64 bf16)
__global__ void __launch_bounds__(128, 1) check(const uint4* a_g, const uint4* b_g, float* out) {
  extern __shared__ uint8_t raw[];
  uint8_t* sm = (uint8_t*)(((uintptr_t)raw + 1023) & ~(uintptr_t)1023);
  uint64_t* bar = (uint64_t*)(sm + 96 * 1024);
  uint32_t* slot = (uint32_t*)(bar + 2);
  // swizzled fill: element row r, 16-B chunk c of plane p at r*128 + ((c ^ (r & 7)) << 4)
  for (int i = threadIdx.x; i < 3 * 128 * 8; i += blockDim.x) {
    const int p = i / 1024, r = (i / 8) % 128, c = i % 8;
    *(uint4*)(sm + p * 16384 + r * 128 + ((c ^ (r & 7)) << 4)) = a_g[i];
    *(uint4*)(sm + 49152 + p * 16384 + r * 128 + ((c ^ (r & 7)) << 4)) = b_g[i];
  }
  asm volatile("fence.proxy.async.shared::cta;");
  if (threadIdx.x == 0) { mbar_init(&bar[0], 1); fence_barrier_init(); }
  if (threadIdx.x / 32 == 0) tmem_alloc<512>(slot);
  tc_fence_before(); __syncthreads(); tc_fence_after();
  const uint32_t tmem = *slot;
  if (threadIdx.x == 0) {
    constexpr uint32_t id = make_idesc<MmaKind::kF16>(128, 128);
    const uint32_t sa = smem_u32(sm), sb = smem_u32(sm + 49152);
    // ss: D0 = sum over planes products hh+hm+mh over K = 64
    for (int kk = 0; kk < 4; ++kk) {
      const uint64_t ah = make_smem_desc<128>(sa + kk * 32, 1024), am = make_smem_desc<128>(sa + 16384 + kk * 32, 1024);
      const uint64_t bh = make_smem_desc<128>(sb + kk * 32, 1024), bm = make_smem_desc<128>(sb + 16384 + kk * 32, 1024);
      tc_mma<MmaKind::kF16>(tmem, ah, bh, id, kk ? 1u : 0u);
      tc_mma<MmaKind::kF16>(tmem, ah, bm, id, 1u);
      tc_mma<MmaKind::kF16>(tmem, am, bh, id, 1u);
    }
    // ts: the same with A_h / A_m copied to TMEM columns 256 / 264 per K16
    for (int kk = 0; kk < 4; ++kk) {
      const uint64_t ah = make_smem_desc<128>(sa + kk * 32, 1024), am = make_smem_desc<128>(sa + 16384 + kk * 32, 1024);
      const uint64_t bh = make_smem_desc<128>(sb + kk * 32, 1024), bm = make_smem_desc<128>(sb + 16384 + kk * 32, 1024);
      const uint32_t th = tmem + 256 + kk * 16, tm = th + 8;
      tc_cp_128x256b(th, ah);
      tc_cp_128x256b(tm, am);
      tc_mma_ts(tmem + 128, th, bh, id, kk ? 1u : 0u);
      tc_mma_ts(tmem + 128, th, bm, id, 1u);
      tc_mma_ts(tmem + 128, tm, bh, id, 1u);
    }
    tc_commit(&bar[0]);
  }
  mbar_wait(&bar[0], 0);
  tc_fence_after();
  const uint32_t q = threadIdx.x / 32;
  for (int c0 = 0; c0 < 256; c0 += 32) {
    uint32_t v[32];
    tmem_ld32(tmem + ((q * 32) << 16) + c0, v);
    tmem_ld_wait();
    for (int j = 0; j < 32; ++j) out[(threadIdx.x) * 256 + c0 + j] = __uint_as_float(v[j]);
  }
  tc_fence_before(); __syncthreads(); tc_fence_after();
  if (threadIdx.x / 32 == 0) tmem_dealloc<512>(tmem);
}

template <bool kTs>
__global__ void __launch_bounds__(128, 1) rate(int steps, long long* cyc) {
  extern __shared__ uint8_t raw[];
  uint8_t* sm = (uint8_t*)(((uintptr_t)raw + 1023) & ~(uintptr_t)1023);
  uint64_t* bar = (uint64_t*)(sm + 96 * 1024);
  uint32_t* slot = (uint32_t*)(bar + 2);
  for (int i = threadIdx.x; i < 96 * 1024 / 16; i += blockDim.x)
    ((uint4*)sm)[i] = make_uint4(0x3f803f81u ^ i, 0x3f003f00u, 0x3e803e80u ^ (i << 3), 0x3c003c00u);
  asm volatile("fence.proxy.async.shared::cta;");
  if (threadIdx.x == 0) { mbar_init(&bar[0], 1); fence_barrier_init(); }
  if (threadIdx.x / 32 == 0) tmem_alloc<512>(slot);
  tc_fence_before(); __syncthreads(); tc_fence_after();
  const uint32_t tmem = *slot;
  if (threadIdx.x == 0) {
    constexpr uint32_t id = make_idesc<MmaKind::kF16>(128, 128);
    const uint32_t sa = smem_u32(sm), sb = smem_u32(sm + 49152);
    const uint32_t S = tmem, T = tmem + 128, A = tmem + 256;
    long long t0 = clock64();
    for (int st = 0; st < steps; ++st) {
      for (int kk = 0; kk < 4; ++kk) {
        const uint64_t ah = make_smem_desc<128>(sa + kk * 32, 1024), am = make_smem_desc<128>(sa + 16384 + kk * 32, 1024),
                       al = make_smem_desc<128>(sa + 32768 + kk * 32, 1024);
        const uint64_t bh = make_smem_desc<128>(sb + kk * 32, 1024), bm = make_smem_desc<128>(sb + 16384 + kk * 32, 1024),
                       bl = make_smem_desc<128>(sb + 32768 + kk * 32, 1024);
        const uint32_t acc = (st | kk) ? 1u : 0u;
        if (kTs) {
          const uint32_t th = A + (kk & 1) * 32, tm = th + 8, tl = th + 16;  // 2 slices in flight
          tc_cp_128x256b(th, ah);
          tc_cp_128x256b(tm, am);
          tc_cp_128x256b(tl, al);
          tc_mma_ts(S, th, bh, id, acc);
          tc_mma_ts(T, th, bm, id, acc);
          tc_mma_ts(T, tm, bh, id, 1u);
          tc_mma_ts(T, th, bl, id, 1u);
          tc_mma_ts(T, tl, bh, id, 1u);
          tc_mma_ts(T, tm, bm, id, 1u);
        } else {
          tc_mma<MmaKind::kF16>(S, ah, bh, id, acc);
          tc_mma<MmaKind::kF16>(T, ah, bm, id, acc);
          tc_mma<MmaKind::kF16>(T, am, bh, id, 1u);
          tc_mma<MmaKind::kF16>(T, ah, bl, id, 1u);
          tc_mma<MmaKind::kF16>(T, al, bh, id, 1u);
          tc_mma<MmaKind::kF16>(T, am, bm, id, 1u);
        }
      }
    }
    tc_commit(&bar[0]);
    mbar_wait(&bar[0], 0);
    cyc[blockIdx.x] = clock64() - t0;
  }
  tc_fence_before(); __syncthreads(); tc_fence_after();
  if (threadIdx.x / 32 == 0) tmem_dealloc<512>(tmem);
}

int main() {
  const int smem = 96 * 1024 + 2048;
  // (1) correctness
  std::vector<uint4> a(3 * 1024), b(3 * 1024);
  srand(7);
  auto rbf = [] { uint32_t m = rand() & 0x7f, s = rand() & 1, e = 120 + rand() % 10;
                  return (s << 15) | (e << 7) | m; };
  for (auto* v : {&a, &b})
    for (auto& x : *v) x = make_uint4(rbf() | (rbf() << 16), rbf() | (rbf() << 16), rbf() | (rbf() << 16), rbf() | (rbf() << 16));
  uint4 *da, *db; float* dout;
  cudaMalloc(&da, a.size() * 16); cudaMalloc(&db, b.size() * 16); cudaMalloc(&dout, 128 * 256 * 4);
  cudaMemcpy(da, a.data(), a.size() * 16, cudaMemcpyHostToDevice);
  cudaMemcpy(db, b.data(), b.size() * 16, cudaMemcpyHostToDevice);
  cudaFuncSetAttribute(check, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  check<<<1, 128, smem>>>(da, db, dout);
  if (cudaDeviceSynchronize() != cudaSuccess) { printf("check: kernel failed\n"); return 1; }
  std::vector<float> o(128 * 256);
  cudaMemcpy(o.data(), dout, o.size() * 4, cudaMemcpyDeviceToHost);
  int diff = 0; double mx = 0;
  for (int r = 0; r < 128; ++r)
    for (int c = 0; c < 128; ++c) {
      const float s = o[r * 256 + c], t = o[r * 256 + 128 + c];
      if (s != t) ++diff;
      mx = fabs(s) > mx ? fabs(s) : mx;
    }
  printf("ts vs ss: %d of %d outputs differ (max |ss| %.3g)\n", diff, 128 * 128, mx);
  // (2) rate
  long long* d; cudaMalloc(&d, 148 * 8);
  for (int ts = 0; ts < 2; ++ts) {
    const int steps = 200;
    if (ts) { cudaFuncSetAttribute(rate<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem); rate<true><<<148, 128, smem>>>(steps, d); }
    else { cudaFuncSetAttribute(rate<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem); rate<false><<<148, 128, smem>>>(steps, d); }
    if (cudaDeviceSynchronize() != cudaSuccess) { printf("rate: kernel failed\n"); return 1; }
    long long h[148], mx2 = 0;
    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    for (int i = 0; i < 148; ++i) mx2 = h[i] > mx2 ? h[i] : mx2;
    printf("%s six N=128 products per K16: %.1f cycles per K16 (ideal 384)\n", ts ? "ts (A in TMEM)" : "ss (A in smem)",
           (double)mx2 / (steps * 4));
  }
  return 0;
}
