// conv_stem.cu -- the network stem (conv 7x7 / stride 2 / pad 3 on <= 4
// input channels, ResNet's C1) as a DENSE-K implicit GEMM.
//
// Why: every generic formulation wastes the tensor cores on this layer. TMA
// im2col needs >= 8 channels per pixel (49 taps x 8 = 392 K for 147 useful)
// and the space-to-depth form is 4x4 taps x 16 = 256 K. Here K is the exact
// (rh, rw, c) stream of 7*7*3 = 147 products, padded to 160 = 10 MMA steps:
// 1.6x fewer MMAs than space-to-depth.
//
// A tile is one output row (OW <= 128 pixels = the 128 MMA rows; rows past
// OW are junk and never stored). Roles (384 threads):
//   warp 0     loader: the 7 input rows the tile needs (NHWC, 4 bf16 channels
//              = 8 B per pixel) -> shared memory with cp.async, zero-filled
//              outside the image (the conv padding), one 16-B pixel pair per
//              copy (the halo is shifted by 4 pixels so pairs never straddle
//              the image border);
//   warps 2-3  gather: build the A tile [128 rows][160 K] in the UMMA
//              SWIZZLE_128B K-major layout from the halo (each pixel's taps
//              in the reference reduction order (rh, rw, c));
//   warp 1     MMA issuer: 10 x tcgen05.mma (M=128, N=64, K=16) per tile;
//   warps 4-11 epilogue (two groups, one per TMEM accumulator): the shared
//              fused-member code of conv_epilogue.cuh, TMA-store fast path.
// Weights [OC][160] (same K order) stay resident in shared memory.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <type_traits>
#include <utility>

#include "conv_epilogue.cuh"
#include "conv_params.h"
#include "sm100_ptx.cuh"

namespace tec_sm100 {

namespace {

// Warp roles: 1 loader... see the kernel. The gather and the loader are
// latency bound per warp, so they get several warps per SM sub-partition.
constexpr int kLoadWarp0 = 1, kLoadWarps = 2;
constexpr int kGatherWarp0 = 3, kGatherWarps = 8;
constexpr int kEpiWarp0 = 11;
constexpr int kThreads = (kEpiWarp0 + 8) * 32;  // 608
constexpr int kEpiThreads = 256;
constexpr int kGather = kGatherWarps * 32;      // two threads per A row
constexpr int kLoaders = kLoadWarps * 32;
constexpr int kBN = 64;              // output channels per CTA tile (= OC for the stem)
constexpr int kK = 160;              // 7*7*3 = 147 padded to 10 x 16
constexpr int kKBlocks = 3;          // 64-element SW128 K blocks (the last half used)
constexpr int kABlock = 128 * 128;   // one K block of A: 128 rows x 128 B
constexpr int kAStage = kKBlocks * kABlock;
constexpr int kWBlock = kBN * 128;
constexpr int kHaloCols = 232;       // smem col = image col + 4; covers [-4, 227]
constexpr int kHaloRowBytes = kHaloCols * 8;
constexpr int kHaloBytes = 7 * kHaloRowBytes;  // 12992
constexpr int kHaloStride = (kHaloBytes + 127) & ~127;
constexpr int kHaloStages = 4;  // deep enough to cover the halo load latency
constexpr int kStageOff = (kHaloStages * kHaloStride + 1023) & ~1023;  // from sH (1024-aligned)

__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src, bool valid) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src),
               "r"(valid ? 16 : 0)
               : "memory");
}
__device__ __forceinline__ void cp_async_arrive(uint64_t* bar) {
  asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}
// Gather helpers: the loads are plain (non-volatile, no memory clobber) so
// the compiler can issue a whole group of them before the first use -- the
// gather is otherwise bound by shared-memory load latency; the halo they read
// is ordered by the mbarrier waits (memory clobbers) around the loop.
__device__ __forceinline__ void sts128(uint32_t addr, uint32_t a, uint32_t b, uint32_t c,
                                       uint32_t d) {
  asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "r"(a), "r"(b), "r"(c),
               "r"(d));
}
__device__ __forceinline__ uint2 lds64(uint32_t addr) {
  uint2 v;
  asm("ld.shared.v2.b32 {%0, %1}, [%2];" : "=r"(v.x), "=r"(v.y) : "r"(addr));
  return v;
}

// Element e (0..2) of the 4-channel pixel held as two 32-bit words.
__device__ __forceinline__ uint32_t chan(uint2 px, int e) {
  return e == 0 ? (px.x & 0xFFFFu) : e == 1 ? (px.x >> 16) : (px.y & 0xFFFFu);
}

template <int OUT_ES>
__global__ void __launch_bounds__(kThreads, 1)
    conv_stem_kernel(const __grid_constant__ CUtensorMap tm_w,
                     const __grid_constant__ CUtensorMap tm_y, const StemParams p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;                              // 2 A stages (1024-aligned)
  uint8_t* sW = sA + 2 * kAStage;                  // resident weights
  uint8_t* sH = sW + kKBlocks * kWBlock;           // 2 halo stages
  // 8 warps x 4 KB epilogue stage; 1024-aligned: the TMA-store box swizzle
  // (SW128 for f32 rows) is a function of the absolute address.
  uint8_t* sStage = sH + kStageOff;
  uint64_t* bars = reinterpret_cast<uint64_t*>(sStage + 8 * 4096);
  uint64_t* h_full = bars;       // [kHaloStages] loader -> gather (32 cp.async arrivals)
  uint64_t* h_empty = bars + 4;  // [kHaloStages] gather -> loader
  uint64_t* a_full = bars + 8;   // [2] gather -> MMA
  uint64_t* a_empty = bars + 10; // [2] MMA -> gather (commit)
  uint64_t* w_full = bars + 12;  // weights landed
  uint64_t* tfull = bars + 13;   // [2]
  uint64_t* tempty = bars + 15;  // [2] (128 each)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 17);
  uint32_t* sBias = reinterpret_cast<uint32_t*>(reinterpret_cast<uint8_t*>(bars) + 256);

  const uint32_t warp = warp_id();
  const uint32_t lane = threadIdx.x & 31;
  const int tiles = p.n * p.oh;
  long long dbg_wait[5] = {0, 0, 0, 0, 0};
  const long long t_start = p.dbg ? clock64() : 0;

  if (warp == 0 && elect_one()) {
    tma_prefetch_desc(&tm_w);
    if (p.tma_store) tma_prefetch_desc(&tm_y);
    for (int i = 0; i < kHaloStages; ++i) {
      mbar_init(&h_full[i], kLoaders);
      mbar_init(&h_empty[i], kGather);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&a_full[i], kGather);
      mbar_init(&a_empty[i], 1);
      mbar_init(&tfull[i], 1);
      mbar_init(&tempty[i], 128);
    }
    mbar_init(w_full, 1);
    fence_barrier_init();
  }
  if (warp == 0) tmem_alloc<128>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  pdl_launch_dependents();
  pdl_wait();

  if (warp >= kLoadWarp0 && warp < kLoadWarp0 + kLoadWarps) {
    // ------------------------------------------------------------ loader
    const __nv_bfloat16* x = static_cast<const __nv_bfloat16*>(p.x);
    const int lt = static_cast<int>(threadIdx.x) - kLoadWarp0 * 32;
    int hs = 0;
    uint32_t hph = 0;
    if (lt == 0) {  // resident weights: three 64-element K blocks
      mbar_arrive_expect_tx(w_full, kKBlocks * kWBlock);
      for (int kb = 0; kb < kKBlocks; ++kb) tma_load_2d(sW + kb * kWBlock, &tm_w, w_full, kb * 64, 0);
    }
    for (int tile = blockIdx.x; tile < tiles; tile += gridDim.x) {
      const int img = tile / p.oh, oh = tile - img * p.oh;
      mbar_wait(&h_empty[hs], hph ^ 1);
      const uint32_t dst0 = smem_u32(sH + hs * kHaloStride);
      // 7 rows x 116 pixel pairs, walked with incremental (row, pair)
      int row = lt / (kHaloCols / 2), pr = lt - row * (kHaloCols / 2);
      for (int j = lt; j < 7 * (kHaloCols / 2); j += kLoaders) {
        const int ih = oh * 2 - p.ph + row;
        const int iw = pr * 2 - 4;  // first image column of the pixel pair
        const bool ok = ih >= 0 && ih < p.h && iw >= 0 && iw + 1 < p.w;
        const __nv_bfloat16* src =
            x + ((static_cast<int64_t>(img) * p.h + (ok ? ih : 0)) * p.w + (ok ? iw : 0)) * 4;
        cp_async16(dst0 + row * kHaloRowBytes + pr * 16, src, ok);
        pr += kLoaders;
        while (pr >= kHaloCols / 2) { pr -= kHaloCols / 2; ++row; }
      }
      cp_async_arrive(&h_full[hs]);
      if (++hs == kHaloStages) { hs = 0; hph ^= 1; }
    }
  } else if (warp >= kGatherWarp0 && warp < kGatherWarp0 + kGatherWarps) {
    // ------------------------------------------------------------ gather
    // Two threads per A row: half 0 builds taps 0..23 (words 0..35,
    // chunks 0..8), half 1 taps 24..48 (words 36..79, chunks 9..19).
    const int gt = static_cast<int>(threadIdx.x) - kGatherWarp0 * 32;  // 0..255
    const int half = gt & 1;
    long long g_aw = 0, g_busy = 0;
    int hs = 0, as = 0;
    uint32_t hph = 0, aph = 0;
    for (int tile = blockIdx.x; tile < tiles; tile += gridDim.x) {
      const long long g0 = p.dbg ? clock64() : 0;
      mbar_wait(&h_full[hs], hph);
      const long long g1 = p.dbg ? clock64() : 0;
      mbar_wait(&a_empty[as], aph ^ 1);
      if (p.dbg && gt == 0) { dbg_wait[0] += g1 - g0; dbg_wait[1 + 0] += 0; g_aw += clock64() - g1; }
      const uint32_t hbase = smem_u32(sH + hs * kHaloStride);
      const uint32_t abase = smem_u32(sA + as * kAStage);
      {
        const int m = gt >> 1;
        if (m < p.ow) {
          // K stream k = (rh*7 + rw)*3 + c as 32-bit words (bf16 pairs):
          // taps t (even) and t+1 give words (c0,c1)_t, (c2_t, c0_t+1),
          // (c1,c2)_t+1 -- one move and two byte permutes per two taps.
          // Words 0..73 hold elements 0..147 (147 = pad), 74..79 are zero.
          // Words stream out in order; each completed 16-B chunk is stored
          // at once (a 4-word rolling buffer keeps register use small).
          const uint32_t pix0 = hbase + (2 * m + 1) * 8;
          const uint32_t arow = abase + m * 128;
          const uint32_t msw = static_cast<uint32_t>(m & 7);
          uint32_t buf[4];
          auto emit = [&](auto w_c, uint32_t v) {
            constexpr int W = decltype(w_c)::value;
            buf[W & 3] = v;
            if constexpr ((W & 3) == 3) {
              constexpr int c = W >> 2;
              sts128(arow + (c >> 3) * kABlock + (((c & 7) ^ msw) << 4), buf[0], buf[1], buf[2],
                     buf[3]);
            }
          };
          // Phase 1 loads every tap pixel of this half-row (up to 25
          // independent LDS in flight), phase 2 permutes and stores: the
          // interleaved form exposed the shared-memory latency per chunk.
          auto build = [&](auto t0_c, auto t1_c) {
            constexpr int T0 = decltype(t0_c)::value, T1 = decltype(t1_c)::value;
            constexpr int NT = T1 - T0;
            uint2 px[NT];
            [&]<int... I>(std::integer_sequence<int, I...>) {
              ((px[I] = lds64(pix0 + ((T0 + I) / 7) * kHaloRowBytes + ((T0 + I) % 7) * 8)), ...);
            }(std::make_integer_sequence<int, NT>{});
            [&]<int... I>(std::integer_sequence<int, I...>) {
              (([&] {
                 constexpr int t = T0 + 2 * I;
                 const uint2 a = px[t - T0];
                 emit(std::integral_constant<int, (3 * t) / 2>{}, a.x);
                 if constexpr (t + 1 < 49) {
                   const uint2 bb = px[t + 1 - T0];
                   emit(std::integral_constant<int, (3 * t) / 2 + 1>{}, __byte_perm(a.y, bb.x, 0x5410));
                   emit(std::integral_constant<int, (3 * t) / 2 + 2>{}, __byte_perm(bb.x, bb.y, 0x5432));
                 } else {
                   emit(std::integral_constant<int, (3 * t) / 2 + 1>{}, a.y & 0xFFFFu);  // (c2_48, 0)
                 }
               }()),
               ...);
            }(std::make_integer_sequence<int, (NT + 1) / 2>{});
          };
          if (half == 0) {
            build(std::integral_constant<int, 0>{}, std::integral_constant<int, 24>{});  // words 0..35
          } else {
            build(std::integral_constant<int, 24>{}, std::integral_constant<int, 49>{});  // words 36..73
            emit(std::integral_constant<int, 74>{}, 0u);
            emit(std::integral_constant<int, 75>{}, 0u);
            emit(std::integral_constant<int, 76>{}, 0u);
            emit(std::integral_constant<int, 77>{}, 0u);
            emit(std::integral_constant<int, 78>{}, 0u);
            emit(std::integral_constant<int, 79>{}, 0u);
          }
        }
      }
      fence_proxy_async_smem();  // generic-proxy writes -> tensor core operand
      if (p.dbg && gt == 0) g_busy += clock64() - g1;
      mbar_arrive(&a_full[as]);
      mbar_arrive(&h_empty[hs]);
      if (++hs == kHaloStages) { hs = 0; hph ^= 1; }
      if (++as == 2) { as = 0; aph ^= 1; }
    }
    if (p.dbg && gt == 0) {
      atomicAdd(&p.dbg[0], static_cast<unsigned long long>(dbg_wait[0]));
      atomicAdd(&p.dbg[7], static_cast<unsigned long long>(g_aw));
      atomicAdd(&p.dbg[8], static_cast<unsigned long long>(g_busy));
    }
  } else if (warp == 0) {
    // --------------------------------------------------------- MMA issuer
    if (elect_one()) {
      constexpr uint32_t idesc = make_idesc<MmaKind::kF16>(128, kBN);
      mbar_wait(w_full, 0);
      const uint64_t wdesc = make_smem_desc<128>(smem_u32(sW), 1024);
      int as = 0;
      uint32_t aph = 0;
      int local = 0;
      for (int tile = blockIdx.x; tile < tiles; tile += gridDim.x, ++local) {
        const int acc = local & 1;
        const uint32_t use = static_cast<uint32_t>(local >> 1);
        { const long long t0 = p.dbg ? clock64() : 0;
          mbar_wait(&tempty[acc], (use & 1) ^ 1);
          if (p.dbg) dbg_wait[2] += clock64() - t0; }
        { const long long t0 = p.dbg ? clock64() : 0;
          mbar_wait(&a_full[as], aph);
          if (p.dbg) dbg_wait[1] += clock64() - t0; }
        tc_fence_after();
        const uint64_t adesc = make_smem_desc<128>(smem_u32(sA + as * kAStage), 1024);
        const uint32_t d = tmem_base + acc * kBN;
#pragma unroll
        for (int s = 0; s < kK / 16; ++s) {
          const uint32_t kb = s >> 2, kk = s & 3;
          tc_mma<MmaKind::kF16>(d, adesc + ((kb * kABlock + kk * 32) >> 4),
                                wdesc + ((kb * kWBlock + kk * 32) >> 4), idesc, s ? 1u : 0u);
        }
        tc_commit(&a_empty[as]);
        tc_commit(&tfull[acc]);
        if (++as == 2) { as = 0; aph ^= 1; }
      }
    }
  } else if (warp >= kEpiWarp0) {
    // ------------------------------------------------------------ epilogue
    // warp w reads TMEM lane quadrant w % 4; each group of 4 consecutive
    // warps covers all four quadrants.
    const uint32_t q = warp & 3;
    const int grp = static_cast<int>(warp - kEpiWarp0) >> 2;
    const int gtid = static_cast<int>(threadIdx.x) - (kThreads - kEpiThreads) - grp * 128;
    uint8_t* stage = sStage + (warp - kEpiWarp0) * 4096;
    const uint32_t stage_u32 = smem_u32(stage);
    const epi::EpiProg prog = epi::make_prog(p.epi);
    const int fast = epi::classify_prog(p.epi);
    const bool tma_epi = p.tma_store && fast != epi::kProgGeneric && fast != epi::kProgBiasAddRelu;
    uint32_t* bias_s = sBias + grp * kBN;
    epi::stage_bias(bias_s, p.epi.bias, 0, kBN, p.oc, gtid, 128);
    epi::named_bar_sync(1 + grp, 128);
    uint32_t box_cnt = 0;
    bool overflow = false;
    int local = 0;
    for (int tile = blockIdx.x; tile < tiles; tile += gridDim.x, ++local) {
      const int acc = local & 1;
      if (acc != grp) continue;
      const uint32_t use = static_cast<uint32_t>(local >> 1);
      const long long tw0 = p.dbg ? clock64() : 0;
      mbar_wait(&tfull[acc], use & 1);
      const long long tw1 = p.dbg ? clock64() : 0;
      if (p.dbg) dbg_wait[3] += tw1 - tw0;
      tc_fence_after();
      const uint32_t taddr0 = tmem_base + ((q * 32) << 16) + acc * kBN;
      if (tma_epi) {
        // 3-D map [N*OH][OW][OC]: the box's pixels >= OW are clipped.
        auto run = [&](auto prog_c) {
          constexpr int kProg = decltype(prog_c)::value;
          epi::epi_rows_tma<kProg, OUT_ES, kBN, false>(
              taddr0, static_cast<int>(lane), bias_s, stage_u32, p.oc, box_cnt, &overflow,
              [&](uint32_t box, int c0) {
                tma_store_3d(&tm_y, box, c0, static_cast<int>(q) * 32, tile);
              });
        };
        if (fast == epi::kProgNone) run(std::integral_constant<int, epi::kProgNone>{});
        else if (fast == epi::kProgBias) run(std::integral_constant<int, epi::kProgBias>{});
        else run(std::integral_constant<int, epi::kProgBiasRelu>{});
      } else {
        const int m = static_cast<int>(q * 32 + lane);
        const int my_row = m < p.ow ? tile * p.ow + m : -1;
#pragma unroll 1
        for (int c0 = 0; c0 < kBN; c0 += epi::kChunk)
          epi::epi_block<false>(p, prog, fast, taddr0 + c0, c0, static_cast<int>(lane), my_row,
                                bias_s + c0, stage, &overflow);
      }
      tc_fence_before();
      mbar_arrive(&tempty[acc]);
      if (p.dbg) dbg_wait[4] += clock64() - tw1;
    }
    if (lane == 0) bulk_wait_all();
    if (overflow && p.err) atomicOr(p.err, 1);
  }

  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 0) tmem_dealloc<128>(tmem_base);
  if (p.dbg) {
    const bool rep = (warp == 0 && lane == 0) || threadIdx.x == kThreads - kEpiThreads;
    if (rep)
      for (int i = 1; i < 5; ++i)
        if (dbg_wait[i]) atomicAdd(&p.dbg[i], static_cast<unsigned long long>(dbg_wait[i]));
    if (threadIdx.x == 0) {
      atomicAdd(&p.dbg[5], static_cast<unsigned long long>(clock64() - t_start));
      atomicAdd(&p.dbg[6], static_cast<unsigned long long>((tiles - blockIdx.x + gridDim.x - 1) / gridDim.x));
    }
  }
}

// NCHW f32 (c <= 4) -> NHWC bf16 with 4 channels (zero padded).
__global__ void pack_stem_kernel(const float* __restrict__ x, __nv_bfloat16* __restrict__ y,
                                 int n, int c, int hw) {
  const int64_t total = static_cast<int64_t>(n) * hw;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t img = i / hw, px = i - img * hw;
    __nv_bfloat16 v[4];
#pragma unroll
    for (int ch = 0; ch < 4; ++ch)
      v[ch] = __float2bfloat16_rn(ch < c ? x[(img * c + ch) * hw + px] : 0.0f);
    *reinterpret_cast<uint2*>(y + i * 4) = *reinterpret_cast<const uint2*>(v);
  }
}

// OIHW f32 [k][c][7][7] -> [k][160] bf16, K order (rh, rw, c), zero tail.
__global__ void pack_stem_weights_kernel(const float* __restrict__ w, __nv_bfloat16* __restrict__ o,
                                         int k, int c) {
  const int total = k * kK;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x) {
    const int oc = i / kK, kk = i - oc * kK;
    float v = 0.0f;
    if (kk < 49 * 3) {
      const int tap = kk / 3, ch = kk - tap * 3;
      const int rh = tap / 7, rw = tap - rh * 7;
      if (ch < c) v = w[((oc * c + ch) * 7 + rh) * 7 + rw];
    }
    o[i] = __float2bfloat16_rn(v);
  }
}

}  // namespace

int stem_smem_bytes() {
  return 1024 + 2 * kAStage + kKBlocks * kWBlock + kStageOff + 8 * 4096 + 256 + 2 * kBN * 4;
}

int launch_conv_stem(const CUtensorMap& tm_w, const CUtensorMap& tm_y, const StemParams& p,
                     int grid, cudaStream_t st) {
  const int smem = stem_smem_bytes();
  auto go = [&](auto kfn) -> int {
    cudaError_t e = cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    e = launch_pdl(kfn, dim3(grid), dim3(kThreads), smem, st, tm_w, tm_y, p);
    if (e != cudaSuccess) return e;
    return cudaGetLastError();
  };
  return p.out_type == kBF16 ? go(conv_stem_kernel<2>) : go(conv_stem_kernel<4>);
}

int launch_pack_stem(const float* x, void* y, int64_t n, int64_t c, int64_t hw,
                     cudaStream_t st) {
  const int64_t total = n * hw;
  const int grid = static_cast<int>(total / 256 + 1 < 148 * 16 ? total / 256 + 1 : 148 * 16);
  pack_stem_kernel<<<grid, 256, 0, st>>>(x, static_cast<__nv_bfloat16*>(y), static_cast<int>(n),
                                         static_cast<int>(c), static_cast<int>(hw));
  return cudaGetLastError();
}

int launch_pack_stem_weights(const float* w, void* o, int64_t k, int64_t c, cudaStream_t st) {
  pack_stem_weights_kernel<<<64, 256, 0, st>>>(w, static_cast<__nv_bfloat16*>(o),
                                               static_cast<int>(k), static_cast<int>(c));
  return cudaGetLastError();
}

}  // namespace tec_sm100
