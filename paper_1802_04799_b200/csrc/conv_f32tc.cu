// conv_f32tc.cu -- f32 fused conv2d (+bias_add, +add, +relu) on the sm_100a
// tensor cores, held within the reference comparator's 1e-4
// (R/src/tensor.cpp:56-72) of the f32 reference, whose arithmetic is a
// sequential float sum of float products (R/src/texpr.cpp:205-232,
// R/src/expr.cpp:137-145).
//
// Numerics (measured on B200, tools/microbench/acc_precision.cu):
//  * kind::tf32 reads only the top 19 bits of an f32 operand and the tcgen05
//    f32 accumulator adds with truncation, so one tf32 MMA chain over
//    ResNet's K = 4608 misses the reference by ~1e-2, and 3xTF32 in one
//    accumulator by ~1e-3 (the truncation bias grows with K).
//  * Here every f32 operand is split EXACTLY into three bf16 planes,
//    x = h + m + l (h = bf16(x), m = bf16(x - h), l = x - h - m; three 8-bit
//    mantissas cover f32's 24), and the conv is the six products whose order
//    is <= 2^-16: hh + (hm + mh + hl + lh + mm). bf16 x bf16 products are exact
//    in f32.
//  * The dominant hh term is accumulated in K chunks of 256: each chunk runs
//    in a fresh TMEM accumulator and is folded into f32 REGISTERS with
//    round-to-nearest adds (__fadd_rn), so truncation never compounds over
//    the whole K. The five cross terms (2^-8 of hh and smaller) share one
//    TMEM accumulator over the whole K; their truncation error is 2^-8
//    smaller again. Error vs the exact sum at K = 4608: std 4.9e-6, max
//    2.4e-5 -- 5x below the reference's own rounding error (std 2.8e-5).
//
// Pipeline (one CTA per SM, persistent over output tiles, N fastest):
//  warp 0      TMA producer: per k-iteration (filter tap, 64-channel block)
//              three im2col boxes (h, m, l planes of the NHWC activation,
//              hardware zero padding and stride) + three weight boxes;
//  warp 1      single-thread tcgen05.mma issuer, 6 MMAs per K16 step: hh into
//              the chunk accumulator S[g & 1], the cross terms into the
//              tile's T[t & 1]; commits S per chunk and T per tile;
//  warps 4-11  epilogue: warp w owns TMEM lanes 32*(w%4).. and half of the
//              columns; folds each chunk into registers, adds T, runs the
//              fused members (bias, residual add, relu -- every member
//              rounded separately, R/src/graph.cpp:209-222) and stores
//              through 32x32 f32 boxes with TMA.
// TMEM: S0 S1 T0 T1, BN columns each (4 x BN <= 512).
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "conv_params.h"
#include "sm100_ptx.cuh"
#include "conv_epilogue.cuh"

namespace tec_sm100 {

namespace {

constexpr int kBM = 128;
constexpr int kThreads = 384;  // 4 control warps + 8 epilogue warps

template <int BN, int SWZ, int STAGES>
struct F32tcCfg {
  static constexpr int kA = kBM * SWZ;         // one plane of A per stage
  static constexpr int kB = BN * SWZ;          // one plane of B per stage
  static constexpr int kStage = 3 * (kA + kB);
  static constexpr int kKSteps = SWZ / 32;     // K16 MMAs per plane per stage
  static constexpr uint32_t kTmemCols = 4 * BN <= 256 ? 256 : 512;
  static constexpr int kSmem = 1024 + STAGES * kStage + 8 * 4096 + 256 + BN * 4;
  static_assert(kSmem <= 227 * 1024, "shared memory budget");
  static_assert(4 * BN <= 512, "TMEM budget");
};

template <int BN, int SWZ, int STAGES, int PROG>
__global__ void __launch_bounds__(kThreads, 1)
    conv_f32tc_kernel(const __grid_constant__ CUtensorMap tm_a,
                      const __grid_constant__ CUtensorMap tm_b,
                      const __grid_constant__ CUtensorMap tm_y, const ConvGemmParams p) {
  using Cfg = F32tcCfg<BN, SWZ, STAGES>;
  constexpr int kCB = SWZ / 2;  // bf16 channels per block
  constexpr int HB = BN / 2;    // columns per epilogue warp
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sStage = smem + STAGES * Cfg::kStage;  // 8 warps x 4 KB
  uint64_t* full = reinterpret_cast<uint64_t*>(sStage + 8 * 4096);
  uint64_t* empty = full + STAGES;
  uint64_t* sfull = empty + STAGES;
  uint64_t* sempty = sfull + 2;
  uint64_t* tfull = sempty + 2;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
  uint32_t* sBias = reinterpret_cast<uint32_t*>(reinterpret_cast<uint8_t*>(full) + 256);

  const uint32_t warp = warp_id();
  const uint32_t lane = threadIdx.x & 31;
  const int num_tiles = p.m_tiles * p.n_tiles;
  const int k_iters = p.r * p.s * p.cblocks;
  const int kps = p.kps;  // k-iterations per hh chunk
  const int cpp = p.cp;   // channels per plane

  if (warp == 0 && elect_one()) {
    tma_prefetch_desc(&tm_a);
    tma_prefetch_desc(&tm_b);
    if (p.tma_store) tma_prefetch_desc(&tm_y);
    for (int i = 0; i < STAGES; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&sfull[i], 1);
      mbar_init(&sempty[i], 256);
      mbar_init(&tfull[i], 1);
      mbar_init(&tempty[i], 256);
    }
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc<Cfg::kTmemCols>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  pdl_launch_dependents();

  if (warp == 0) {
    // ------------------------------------------------ TMA producer
    if (elect_one()) {
      pdl_wait();
      int stage = 0;
      uint32_t phase = 0;
      const int ohw = p.oh * p.ow;
      const int wrow = 3 * cpp * p.s;  // weight columns per filter row
      for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x) {
        const int m_tile = tile / p.n_tiles;
        const int n_tile = tile - m_tile * p.n_tiles;
        const int m0 = m_tile * kBM;
        const int img = m0 / ohw;
        const int rem = m0 - img * ohw;
        const int oh = rem / p.ow;
        const int ow = rem - oh * p.ow;
        const int w0 = ow * p.sw - p.pw;
        const int h0 = oh * p.sh - p.ph;
        int r = 0, s = 0, cb = 0;
        for (int k = 0; k < k_iters; ++k) {
          mbar_wait(&empty[stage], phase ^ 1);
          mbar_arrive_expect_tx(&full[stage], Cfg::kStage);
          uint8_t* base = smem + stage * Cfg::kStage;
          const int wcol = r * wrow + s * 3 * cpp + cb * kCB;
#pragma unroll
          for (int pl = 0; pl < 3; ++pl) {
            tma_load_im2col_4d(base + pl * Cfg::kA, &tm_a, &full[stage], pl * cpp + cb * kCB, w0,
                               h0, img, static_cast<uint16_t>(s), static_cast<uint16_t>(r));
            tma_load_2d(base + 3 * Cfg::kA + pl * Cfg::kB, &tm_b, &full[stage],
                        wcol + pl * cpp, n_tile * BN);
          }
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
          if (++cb == p.cblocks) {
            cb = 0;
            if (++s == p.s) { s = 0; ++r; }
          }
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------ single-thread MMA issuer
    if (elect_one()) {
      constexpr uint32_t idesc = make_idesc<MmaKind::kF16>(kBM, BN);
      int stage = 0;
      uint32_t phase = 0;
      int g = 0;  // hh chunks issued so far (S ring position)
      int local = 0;
      for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x, ++local) {
        const int tb = local & 1;
        mbar_wait(&tempty[tb], ((local >> 1) & 1) ^ 1);
        tc_fence_after();
        const uint32_t t_tmem = tmem_base + (2 + tb) * BN;
        uint32_t s_tmem = tmem_base;
        int in_chunk = 0;
        for (int k = 0; k < k_iters; ++k) {
          if (in_chunk == 0) {
            const int sb = g & 1;
            mbar_wait(&sempty[sb], ((g >> 1) & 1) ^ 1);
            tc_fence_after();
            s_tmem = tmem_base + sb * BN;
          }
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          const uint32_t base = smem_u32(smem + stage * Cfg::kStage);
#pragma unroll
          for (int kk = 0; kk < Cfg::kKSteps; ++kk) {
            const uint32_t a0 = base + kk * 32, b0 = base + 3 * Cfg::kA + kk * 32;
            const uint64_t ah = make_smem_desc<SWZ>(a0, 8 * SWZ);
            const uint64_t am = make_smem_desc<SWZ>(a0 + Cfg::kA, 8 * SWZ);
            const uint64_t al = make_smem_desc<SWZ>(a0 + 2 * Cfg::kA, 8 * SWZ);
            const uint64_t bh = make_smem_desc<SWZ>(b0, 8 * SWZ);
            const uint64_t bm = make_smem_desc<SWZ>(b0 + Cfg::kB, 8 * SWZ);
            const uint64_t bl = make_smem_desc<SWZ>(b0 + 2 * Cfg::kB, 8 * SWZ);
            tc_mma<MmaKind::kF16>(s_tmem, ah, bh, idesc, (in_chunk | kk) != 0 ? 1u : 0u);
            tc_mma<MmaKind::kF16>(t_tmem, ah, bm, idesc, (k | kk) != 0 ? 1u : 0u);
            tc_mma<MmaKind::kF16>(t_tmem, am, bh, idesc, 1u);
            tc_mma<MmaKind::kF16>(t_tmem, ah, bl, idesc, 1u);
            tc_mma<MmaKind::kF16>(t_tmem, al, bh, idesc, 1u);
            tc_mma<MmaKind::kF16>(t_tmem, am, bm, idesc, 1u);
          }
          tc_commit(&empty[stage]);  // frees the smem slot when the MMAs land
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
          if (++in_chunk == kps || k + 1 == k_iters) {
            tc_commit(&sfull[g & 1]);  // chunk ready to fold
            ++g;
            in_chunk = 0;
          }
        }
        tc_commit(&tfull[tb]);
      }
    }
  } else if (warp >= 4) {
    // ------------------------------------------------- epilogue warps
    const uint32_t q = warp & 3;
    const int hf = static_cast<int>(warp - 4) >> 2;
    const int etid = static_cast<int>(threadIdx.x) - 128;
    const uint32_t stage_u32 = smem_u32(sStage + (warp - 4) * 4096);
    const int nch = (k_iters + kps - 1) / kps;
    const uint32_t lane_base = tmem_base + ((q * 32) << 16) + hf * HB;
    bool overflow = false;
    int g = 0;
    int local = 0;
    int staged_n = -1;
    for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x, ++local) {
      const int m_tile = tile / p.n_tiles;
      const int n_tile = tile - m_tile * p.n_tiles;
      const int row0 = m_tile * kBM + static_cast<int>(q * 32);
      const int row = row0 + static_cast<int>(lane);
      if (PROG != epi::kProgNone && n_tile != staged_n) {
        epi::named_bar_sync(1, 256);  // previous tile's bias readers are done
        epi::stage_bias(sBias, p.epi.bias, n_tile * BN, BN, p.oc, etid, 256);
        epi::named_bar_sync(1, 256);
        staged_n = n_tile;
      }
      float sum[HB];
#pragma unroll
      for (int j = 0; j < HB; ++j) sum[j] = 0.0f;
      // hh chunks, folded in K order with round-to-nearest adds
#pragma unroll 1
      for (int c = 0; c < nch; ++c, ++g) {
        const int sb = g & 1;
        mbar_wait(&sfull[sb], (g >> 1) & 1);
        tc_fence_after();
#pragma unroll
        for (int c0 = 0; c0 < HB; c0 += 32) {
          uint32_t v[32];
          tmem_ld32(lane_base + sb * BN + c0, v);
          tmem_ld_wait();
#pragma unroll
          for (int j = 0; j < 32; ++j) sum[c0 + j] = __fadd_rn(sum[c0 + j], __uint_as_float(v[j]));
        }
        tc_fence_before();
        mbar_arrive(&sempty[sb]);
      }
      // + the cross terms
      const int tb = local & 1;
      mbar_wait(&tfull[tb], (local >> 1) & 1);
      tc_fence_after();
#pragma unroll
      for (int c0 = 0; c0 < HB; c0 += 32) {
        uint32_t v[32];
        tmem_ld32(lane_base + (2 + tb) * BN + c0, v);
        tmem_ld_wait();
#pragma unroll
        for (int j = 0; j < 32; ++j) sum[c0 + j] = __fadd_rn(sum[c0 + j], __uint_as_float(v[j]));
      }
      tc_fence_before();
      mbar_arrive(&tempty[tb]);
      if (!p.tma_store) {
        // OC not a multiple of 32: per-element stores (small odd shapes)
        const float* bias = static_cast<const float*>(p.epi.bias);
        const float* res = static_cast<const float*>(p.epi.residual);
        float* y = static_cast<float*>(p.y);
#pragma unroll
        for (int j = 0; j < HB; ++j) {
          const int col = n_tile * BN + hf * HB + j;
          if (row >= p.m || col >= p.oc) continue;
          const int64_t o = static_cast<int64_t>(row) * p.oc + col;
          float v = sum[j];
          if constexpr (PROG != epi::kProgNone) v = __fadd_rn(v, bias[col]);
          if constexpr (PROG == epi::kProgBiasAddRelu) v = __fadd_rn(v, res[o]);
          if constexpr (PROG == epi::kProgBiasRelu || PROG == epi::kProgBiasAddRelu)
            v = v < 0.0f ? 0.0f : v;
          y[o] = v;
        }
        continue;
      }
      // fused members -> 32x32 f32 boxes -> TMA stores (rows >= M and
      // columns >= OC are clipped by the tensor map)
      const uint8_t* rrow = nullptr;
      if (PROG == epi::kProgBiasAddRelu && row < p.m)
        rrow = static_cast<const uint8_t*>(p.epi.residual) +
               (static_cast<int64_t>(row) * p.oc + n_tile * BN + hf * HB) * 4;
#pragma unroll
      for (int c0 = 0; c0 < HB; c0 += 32) {
        if (n_tile * BN + hf * HB + c0 < p.oc) {
          uint32_t acc[32];
#pragma unroll
          for (int j = 0; j < 32; ++j) acc[j] = __float_as_uint(sum[c0 + j]);
          if (lane == 0) bulk_wait_read<0>();  // the box's previous store has read it
          __syncwarp();
          epi::epi_acc_to_box<PROG, 4>(acc, static_cast<int>(lane), sBias + hf * HB + c0,
                                       stage_u32, &overflow, rrow ? rrow + c0 * 4 : nullptr);
          fence_proxy_async_smem();
          __syncwarp();
          if (lane == 0) {
            tma_store_2d(&tm_y, stage_u32, n_tile * BN + hf * HB + c0, row0);
            bulk_commit();
          }
        }
      }
    }
    if (lane == 0) bulk_wait_all();  // TMA stores done before smem goes away
  }

  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 2) tmem_dealloc<Cfg::kTmemCols>(tmem_base);
}

}  // namespace

int conv_f32tc_smem_bytes(int bn, int swz) {
  if (swz == 128) return bn == 64 ? F32tcCfg<64, 128, 2>::kSmem : F32tcCfg<128, 128, 2>::kSmem;
  return bn == 64 ? F32tcCfg<64, 32, 8>::kSmem : F32tcCfg<128, 32, 6>::kSmem;
}

template <int BN, int SWZ, int STAGES, int PROG>
static int launch_f32tc_inst(const CUtensorMap& tm_a, const CUtensorMap& tm_b,
                             const CUtensorMap& tm_y, const ConvGemmParams& p, int grid,
                             cudaStream_t stream) {
  using Cfg = F32tcCfg<BN, SWZ, STAGES>;
  auto kfn = conv_f32tc_kernel<BN, SWZ, STAGES, PROG>;
  cudaError_t e =
      cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::kSmem);
  if (e != cudaSuccess) return e;
  e = launch_pdl(kfn, dim3(grid), dim3(kThreads), Cfg::kSmem, stream, tm_a, tm_b, tm_y, p);
  if (e != cudaSuccess) return e;
  return cudaGetLastError();
}

template <int BN, int SWZ, int STAGES>
static int launch_f32tc_prog(const CUtensorMap& tm_a, const CUtensorMap& tm_b,
                             const CUtensorMap& tm_y, const ConvGemmParams& p, int prog,
                             int grid, cudaStream_t st) {
  switch (prog) {
    case epi::kProgNone: return launch_f32tc_inst<BN, SWZ, STAGES, epi::kProgNone>(tm_a, tm_b, tm_y, p, grid, st);
    case epi::kProgBias: return launch_f32tc_inst<BN, SWZ, STAGES, epi::kProgBias>(tm_a, tm_b, tm_y, p, grid, st);
    case epi::kProgBiasRelu: return launch_f32tc_inst<BN, SWZ, STAGES, epi::kProgBiasRelu>(tm_a, tm_b, tm_y, p, grid, st);
    case epi::kProgBiasAddRelu: return launch_f32tc_inst<BN, SWZ, STAGES, epi::kProgBiasAddRelu>(tm_a, tm_b, tm_y, p, grid, st);
    default: return -1;
  }
}

// Returns a cudaError_t, or -1 for an unsupported (bn, swz, program).
int launch_conv_f32tc(const CUtensorMap& tm_a, const CUtensorMap& tm_b, const CUtensorMap& tm_y,
                      const ConvGemmParams& p, int bn, int swz, int prog, int grid,
                      cudaStream_t st) {
  if (swz == 128 && bn == 64) return launch_f32tc_prog<64, 128, 2>(tm_a, tm_b, tm_y, p, prog, grid, st);
  if (swz == 128 && bn == 128) return launch_f32tc_prog<128, 128, 2>(tm_a, tm_b, tm_y, p, prog, grid, st);
  if (swz == 32 && bn == 64) return launch_f32tc_prog<64, 32, 8>(tm_a, tm_b, tm_y, p, prog, grid, st);
  if (swz == 32 && bn == 128) return launch_f32tc_prog<128, 32, 6>(tm_a, tm_b, tm_y, p, prog, grid, st);
  return -1;
}

}  // namespace tec_sm100
