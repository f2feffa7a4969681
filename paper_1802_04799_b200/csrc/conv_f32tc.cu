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
//
// Plane layouts: 64+ channels per plane -> the three planes are separate
// 128-B channel blocks ([h | m | l], one TMA box each per k-iteration);
// <= 16 channels per plane (the space-to-depth stem C1) -> INTERLEAVED: one
// 64-channel pixel [h16 | m16 | l16 | 0], one box per k-iteration, and the
// planes are the three K16 slices (32-B offsets) of the same swizzled row --
// a third of the im2col requests.
//
// Split-K (deep layers whose output has too few tiles for 148 SMs): work
// item = (tile, split); a split folds its own hh chunks and cross terms into
// an f32 partial, the last split to arrive sums the partials IN SPLIT ORDER
// with RN adds (the same promotion as the chunk fold -- deterministic and
// independent of scheduling) and runs the fused members.
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

template <int BN, int SWZ, int STAGES, bool INTER>
struct F32tcCfg {
  static constexpr int kPlanes = INTER ? 1 : 3;  // TMA boxes per operand per k-iteration
  static constexpr int kA = kBM * SWZ;           // one box of A
  static constexpr int kB = BN * SWZ;            // one box of B
  static constexpr int kStage = kPlanes * (kA + kB);
  static constexpr int kKSteps = INTER ? 1 : SWZ / 32;  // K16 steps per plane per stage
  static constexpr uint32_t kTmemCols = 4 * BN <= 256 ? 256 : 512;
  static constexpr int kSmem = 1024 + STAGES * kStage + 8 * 4096 + 256 + BN * 4;
  static_assert(kSmem <= 227 * 1024, "shared memory budget");
  static_assert(4 * BN <= 512, "TMEM budget");
  static_assert(!INTER || SWZ == 128, "interleaved planes live in one 128-B row");
};

template <int BN, int SWZ, int STAGES, bool INTER, int PROG>
__global__ void __launch_bounds__(kThreads, 1)
    conv_f32tc_kernel(const __grid_constant__ CUtensorMap tm_a,
                      const __grid_constant__ CUtensorMap tm_b,
                      const __grid_constant__ CUtensorMap tm_y, const ConvGemmParams p) {
  using Cfg = F32tcCfg<BN, SWZ, STAGES, INTER>;
  constexpr int kCB = SWZ / 2;  // bf16 channels per box row
  constexpr int HB = BN / 2;    // columns per epilogue warp
  // byte offset of plane q inside an operand stage: its own box, or its
  // K16 slice of the interleaved row
  constexpr int kPlaneA = INTER ? 32 : Cfg::kA;
  constexpr int kPlaneB = INTER ? 32 : Cfg::kB;
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
  int* s_last = reinterpret_cast<int*>(tmem_slot + 1);
  uint32_t* sBias = reinterpret_cast<uint32_t*>(reinterpret_cast<uint8_t*>(full) + 256);

  const uint32_t warp = warp_id();
  const uint32_t lane = threadIdx.x & 31;
  const int splits = p.splits > 1 ? p.splits : 1;
  const int num_items = p.m_tiles * p.n_tiles * splits;
  const int k_iters = p.r * p.s * p.cblocks;
  const int kps = splits > 1 ? p.kps : k_iters;  // k-iterations per split
  const int chunk = p.chunk_iters;               // k-iterations per hh chunk
  const int cpp = p.cp;                          // channels per plane
  const int pix = INTER ? 64 : 3 * cpp;          // packed channels per pixel

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
      const int sc = p.s * p.cblocks;
      for (int item = blockIdx.x; item < num_items; item += gridDim.x) {
        const int mn = item / splits;
        const int split = item - mn * splits;
        const int m_tile = mn / p.n_tiles;
        const int n_tile = mn - m_tile * p.n_tiles;
        const int m0 = m_tile * kBM;
        const int img = m0 / ohw;
        const int rem = m0 - img * ohw;
        const int oh = rem / p.ow;
        const int ow = rem - oh * p.ow;
        const int w0 = ow * p.sw - p.pw;
        const int h0 = oh * p.sh - p.ph;
        const int kb = split * kps, ke = min(k_iters, kb + kps);
        int r = kb / sc, rem_k = kb - r * sc;
        int s = rem_k / p.cblocks, cb = rem_k - s * p.cblocks;
        for (int k = kb; k < ke; ++k) {
          mbar_wait(&empty[stage], phase ^ 1);
          mbar_arrive_expect_tx(&full[stage], Cfg::kStage);
          uint8_t* base = smem + stage * Cfg::kStage;
          const int wcol = (r * p.s + s) * pix + cb * kCB;
#pragma unroll
          for (int pl = 0; pl < Cfg::kPlanes; ++pl) {
            tma_load_im2col_4d(base + pl * Cfg::kA, &tm_a, &full[stage], pl * cpp + cb * kCB, w0,
                               h0, img, static_cast<uint16_t>(s), static_cast<uint16_t>(r));
            tma_load_2d(base + Cfg::kPlanes * Cfg::kA + pl * Cfg::kB, &tm_b, &full[stage],
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
      for (int item = blockIdx.x; item < num_items; item += gridDim.x, ++local) {
        const int tb = local & 1;
        mbar_wait(&tempty[tb], ((local >> 1) & 1) ^ 1);
        tc_fence_after();
        const uint32_t t_tmem = tmem_base + (2 + tb) * BN;
        uint32_t s_tmem = tmem_base;
        const int kb = (item % splits) * kps, ke = min(k_iters, kb + kps);
        int in_chunk = 0;
        for (int k = kb; k < ke; ++k) {
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
            const uint32_t a0 = base + kk * 32, b0 = base + Cfg::kPlanes * Cfg::kA + kk * 32;
            const uint64_t ah = make_smem_desc<SWZ>(a0, 8 * SWZ);
            const uint64_t am = make_smem_desc<SWZ>(a0 + kPlaneA, 8 * SWZ);
            const uint64_t al = make_smem_desc<SWZ>(a0 + 2 * kPlaneA, 8 * SWZ);
            const uint64_t bh = make_smem_desc<SWZ>(b0, 8 * SWZ);
            const uint64_t bm = make_smem_desc<SWZ>(b0 + kPlaneB, 8 * SWZ);
            const uint64_t bl = make_smem_desc<SWZ>(b0 + 2 * kPlaneB, 8 * SWZ);
            tc_mma<MmaKind::kF16>(s_tmem, ah, bh, idesc, (in_chunk | kk) != 0 ? 1u : 0u);
            tc_mma<MmaKind::kF16>(t_tmem, ah, bm, idesc, (k != kb || kk != 0) ? 1u : 0u);
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
          if (++in_chunk == chunk || k + 1 == ke) {
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
    const int ew = static_cast<int>(warp) - 4;
    const int hf = ew >> 2;
    const int etid = static_cast<int>(threadIdx.x) - 128;
    const uint32_t stage_u32 = smem_u32(sStage + ew * 4096);
    const uint32_t lane_base = tmem_base + ((q * 32) << 16) + hf * HB;
    bool overflow = false;
    int g = 0;
    int local = 0;
    int staged_n = -1;
    for (int item = blockIdx.x; item < num_items; item += gridDim.x, ++local) {
      const int mn = item / splits;
      const int split = item - mn * splits;
      const int m_tile = mn / p.n_tiles;
      const int n_tile = mn - m_tile * p.n_tiles;
      const int row0 = m_tile * kBM + static_cast<int>(q * 32);
      const int row = row0 + static_cast<int>(lane);
      const int kb = split * kps, ke = min(k_iters, kb + kps);
      const int nch = (ke - kb + chunk - 1) / chunk;
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
      // p.fault == 1 (tests only): lose one arrive -- the MMA warp then waits
      // for this accumulator forever and the mbarrier watchdog must trap
      if (!(p.fault == 1 && local == 0)) mbar_arrive(&tempty[tb]);
      if (splits > 1) {
        // publish this split's partial ([item][warp][column][lane]: one
        // 128-B line per column); the last split of the tile sums them all
        // in split order
        float* mine = p.ws + ((static_cast<size_t>(mn) * splits + split) * 8 + ew) * HB * 32 + lane;
#pragma unroll
        for (int j = 0; j < HB; ++j) __stcg(mine + j * 32, sum[j]);
        __threadfence();
        epi::named_bar_sync(1, 256);
        if (etid == 0) *s_last = atomicAdd(&p.tile_cnt[mn], 1) == splits - 1;
        epi::named_bar_sync(1, 256);
        if (!*s_last) continue;
        __threadfence();
        const float* part = p.ws + (static_cast<size_t>(mn) * splits * 8 + ew) * HB * 32 + lane;
#pragma unroll
        for (int j = 0; j < HB; ++j) sum[j] = __ldcg(part + j * 32);
#pragma unroll 1
        for (int sp = 1; sp < splits; ++sp) {
          const float* ps = part + static_cast<size_t>(sp) * 8 * HB * 32;
#pragma unroll
          for (int j = 0; j < HB; ++j) sum[j] = __fadd_rn(sum[j], __ldcg(ps + j * 32));
        }
        if (etid == 0) p.tile_cnt[mn] = 0;  // ready for the next launch
      }
      if (PROG != epi::kProgNone && n_tile != staged_n) {
        // only the tiles this CTA finishes stage their bias (uniform over the
        // 256 epilogue threads: s_last is shared)
        epi::named_bar_sync(2, 256);  // previous tile's bias readers are done
        epi::stage_bias(sBias, p.epi.bias, n_tile * BN, BN, p.oc, etid, 256);
        epi::named_bar_sync(2, 256);
        staged_n = n_tile;
      }
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

template <int BN, int SWZ, int STAGES, bool INTER, int PROG>
int launch_f32tc_inst(const CUtensorMap& tm_a, const CUtensorMap& tm_b, const CUtensorMap& tm_y,
                      const ConvGemmParams& p, int grid, cudaStream_t stream) {
  using Cfg = F32tcCfg<BN, SWZ, STAGES, INTER>;
  auto kfn = conv_f32tc_kernel<BN, SWZ, STAGES, INTER, PROG>;
  cudaError_t e =
      cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::kSmem);
  if (e != cudaSuccess) return e;
  e = launch_pdl(kfn, dim3(grid), dim3(kThreads), Cfg::kSmem, stream, tm_a, tm_b, tm_y, p);
  if (e != cudaSuccess) return e;
  return cudaGetLastError();
}

template <int BN, int SWZ, int STAGES, bool INTER>
int launch_f32tc_prog(const CUtensorMap& tm_a, const CUtensorMap& tm_b, const CUtensorMap& tm_y,
                      const ConvGemmParams& p, int prog, int grid, cudaStream_t st) {
  switch (prog) {
    case epi::kProgNone: return launch_f32tc_inst<BN, SWZ, STAGES, INTER, epi::kProgNone>(tm_a, tm_b, tm_y, p, grid, st);
    case epi::kProgBias: return launch_f32tc_inst<BN, SWZ, STAGES, INTER, epi::kProgBias>(tm_a, tm_b, tm_y, p, grid, st);
    case epi::kProgBiasRelu: return launch_f32tc_inst<BN, SWZ, STAGES, INTER, epi::kProgBiasRelu>(tm_a, tm_b, tm_y, p, grid, st);
    case epi::kProgBiasAddRelu: return launch_f32tc_inst<BN, SWZ, STAGES, INTER, epi::kProgBiasAddRelu>(tm_a, tm_b, tm_y, p, grid, st);
    default: return -1;
  }
}

// The instantiated (BN, block, stages, interleaved) set.
#define TEC_F32TC_INSTANCES(X) \
  X(64, 128, 2, false)         \
  X(128, 128, 2, false)        \
  X(64, 32, 8, false)          \
  X(128, 32, 6, false)         \
  X(64, 128, 6, true)          \
  X(128, 128, 5, true)

}  // namespace

int conv_f32tc_smem_bytes(int bn, int swz, bool inter) {
#define TEC_X(BN, SW, ST, IN) \
  if (bn == BN && swz == SW && inter == IN) return F32tcCfg<BN, SW, ST, IN>::kSmem;
  TEC_F32TC_INSTANCES(TEC_X)
#undef TEC_X
  return -1;
}

int conv_f32tc_stages(int bn, int swz, bool inter) {
#define TEC_X(BN, SW, ST, IN) \
  if (bn == BN && swz == SW && inter == IN) return ST;
  TEC_F32TC_INSTANCES(TEC_X)
#undef TEC_X
  return -1;
}

// Returns a cudaError_t, or -1 for an unsupported (bn, swz, program).
int launch_conv_f32tc(const CUtensorMap& tm_a, const CUtensorMap& tm_b, const CUtensorMap& tm_y,
                      const ConvGemmParams& p, int bn, int swz, bool inter, int prog, int grid,
                      cudaStream_t st) {
#define TEC_X(BN, SW, ST, IN)   \
  if (bn == BN && swz == SW && inter == IN) \
    return launch_f32tc_prog<BN, SW, ST, IN>(tm_a, tm_b, tm_y, p, prog, grid, st);
  TEC_F32TC_INSTANCES(TEC_X)
#undef TEC_X
  return -1;
}

}  // namespace tec_sm100
