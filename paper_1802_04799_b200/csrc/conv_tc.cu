// conv_tc.cu -- fused conv2d (+scale/bias_add/add/mul/relu) as a
// warp-specialised implicit GEMM on the sm_100a 5th-generation tensor cores.
//
// Reference semantics: make_conv (R/src/ops.cpp:120-161) followed by the
// fused epilogue members (R/src/ops.cpp:216-305) exactly as fuse_pass groups
// them (R/src/graph_passes.cpp:240-244) and eval_graph_node runs them
// (R/src/graph.cpp:209-222).
//
// B200 design (the paper's schedule primitives, realised in hardware):
//  * GEMM view: M = N*OH*OW output pixels (NHWC), N = OC, K = R*S*Cp.
//  * "cache_read(shared) + compute_at": A tiles (128 output pixels x one
//    channel block of one filter tap) are produced by the TMA engine in
//    im2col mode straight from the NHWC activation -- the hardware applies
//    the zero padding of select(...) and the stride; B tiles (BN output
//    channels x the same K slice) by tiled TMA from the KRSC weights.
//  * "virtual_thread" latency hiding: a STAGES-deep shared-memory ring
//    guarded by full/empty mbarriers decouples the TMA warp (load), the
//    single-thread MMA issuer (compute) and 4 epilogue warps (store) --
//    the decoupled access-execute pipeline of the paper's VDLA, with
//    mbarriers in place of its dependence tokens.
//  * "tensorize": tcgen05.mma (M=128, N=BN, K=32 bytes) accumulating in
//    TMEM; two TMEM accumulators let the epilogue of tile i overlap the
//    MMAs of tile i+1.
//  * epilogue "compute_at": TMEM -> registers (32 columns per tcgen05.ld)
//    -> scale/bias/residual/relu on 32-wide register vectors with 128-bit
//    operand loads -> 128-bit global stores; intermediates never touch HBM.
//  * persistent grid (one CTA per SM), tiles strided by gridDim.x.
//  * CTA pairs (knob cluster_n = 2): tcgen05 cta_group::2, a 256-row tile
//    per pair with half of the weight rows in each CTA (`PAIR` below).
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <type_traits>

#include "conv_params.h"
#include "sm100_ptx.cuh"
#include "conv_epilogue.cuh"

namespace tec_sm100 {

namespace {

constexpr int kBM = 128;
constexpr int kThreads = 384;  // 4 control warps + 8 epilogue warps
constexpr int kEpiThreads = 256;
using epi::kChunk;

template <MmaKind KIND, int BN, int STAGES, int SWZ, bool PAIR = false>
struct ConvCfg {
  static constexpr int kABytes = kBM * SWZ;  // one stage of A
  // one stage of B (a CTA of a pair holds half of the tile's weight rows)
  static constexpr int kBBytes = (PAIR ? BN / 2 : BN) * SWZ;
  static constexpr int kStageBytes = kABytes + kBBytes;
  static constexpr int kMmaPerStage = SWZ / 32;  // each MMA eats 32 B of K
  // TMEM accumulator ring: 4 buffers when they fit (knob acc_bufs), else 2
  static constexpr int kMaxAcc = 4 * BN <= 512 ? 4 : 2;
  static constexpr uint32_t kTmemCols = kMaxAcc * BN <= 32    ? 32
                                        : kMaxAcc * BN <= 64  ? 64
                                        : kMaxAcc * BN <= 128 ? 128
                                        : kMaxAcc * BN <= 256 ? 256
                                                              : 512;
  static constexpr int kSmemBytes = 1024 /*align slack*/ + STAGES * kStageBytes +
                                    8 * 4096 /*epilogue stage*/ + 256 /*barriers*/ +
                                    2 * BN * 4 /*bias*/;
  static_assert(kSmemBytes <= 227 * 1024, "shared memory budget");
};

template <MmaKind KIND, int BN, int STAGES, int SWZ, bool PAIR>
__global__ void __launch_bounds__(kThreads, 1)
    conv_fprop_tc_kernel(const __grid_constant__ CUtensorMap tm_a,
                         const __grid_constant__ CUtensorMap tm_b,
                         const __grid_constant__ CUtensorMap tm_y,
                         const ConvGemmParams p) {
  using Cfg = ConvCfg<KIND, BN, STAGES, SWZ, PAIR>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + STAGES * Cfg::kABytes;
  uint8_t* sStage = sB + STAGES * Cfg::kBBytes;  // 8 warps x 4 KB epilogue stage
  uint64_t* full = reinterpret_cast<uint64_t*>(sStage + 8 * 4096);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint64_t* tempty = tfull + 4;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 4);
  uint32_t* sBias = reinterpret_cast<uint32_t*>(
      reinterpret_cast<uint8_t*>(full) + 256);  // [2][BN] f32 / i32

  const uint32_t warp = warp_id();
  const uint32_t lane = threadIdx.x & 31;
  // tile `local` -> accumulator local % nacc, drained by epilogue group local % 2
  const int nacc = p.nacc == 4 && Cfg::kMaxAcc == 4 ? 4 : 2;
  const int acc_shift = nacc == 4 ? 2 : 1;
  const int splits = p.splits > 1 ? p.splits : 1;
  const int num_tiles = p.m_tiles * p.n_tiles * splits;  // work items
  const int k_iters = p.r * p.s * p.cblocks;
  const int kps = splits > 1 ? p.kps : k_iters;  // k-iterations per split
  const int sc = p.s * p.cblocks;
  int* s_last = reinterpret_cast<int*>(reinterpret_cast<uint8_t*>(full) + 240);  // [2]
  long long dbg_wait[5] = {0, 0, 0, 0, 0};
  const long long t_start = p.dbg ? clock64() : 0;
  constexpr int kCB =
      SWZ / (KIND == MmaKind::kF16 ? 2 : KIND == MmaKind::kTF32 ? 4 : 1);
  // CTA pair (PAIR, cta_group::2, cluster of 2): the pair computes a 256-row
  // M tile -- rows [0,128) in the leader's TMEM from its A, [128,256) in the
  // peer's -- with one MMA stream issued by the leader; each CTA loads its
  // own A rows and HALF of the BN weight rows, so a CTA's shared memory
  // feeds the tensor cores A + B/2 per K step instead of A + B. Both CTAs'
  // TMA bytes complete on the leader's full barrier, the leader's commits
  // release both CTAs' stages and accumulators, and the peer's epilogue
  // hands its accumulator back through the leader's tempty barrier. Work
  // unit u = (M-tile pair, N tile); splits == 1.
  const uint32_t rank = PAIR ? cluster_ctarank() : 0u;
  const int t_first = PAIR ? static_cast<int>(blockIdx.x >> 1) : static_cast<int>(blockIdx.x);
  const int t_step = PAIR ? static_cast<int>(gridDim.x >> 1) : static_cast<int>(gridDim.x);
  const int t_count = PAIR ? ((p.m_tiles + 1) / 2) * p.n_tiles : num_tiles;
  auto tile_of = [&](int u) -> int {  // work unit -> this CTA's tile index
    if constexpr (!PAIR) return u;
    const int mp = u / p.n_tiles;
    return (2 * mp + static_cast<int>(rank)) * p.n_tiles + (u - mp * p.n_tiles);
  };
  constexpr uint32_t kStageTx = PAIR ? 2 * Cfg::kStageBytes : Cfg::kStageBytes;

  if (warp == 0 && elect_one()) {
    tma_prefetch_desc(&tm_a);
    tma_prefetch_desc(&tm_b);
    if (p.tma_store) tma_prefetch_desc(&tm_y);
    for (int i = 0; i < STAGES; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    for (int i = 0; i < 4; ++i) {
      mbar_init(&tfull[i], 1);
      // the epilogue group (4 warps) of the accumulator; a pair: both CTAs'
      mbar_init(&tempty[i], PAIR ? 256 : 128);
    }
    fence_barrier_init();
  }
  if (warp == 2) {
    if constexpr (PAIR) tmem_alloc_pair<Cfg::kTmemCols>(tmem_slot);
    else tmem_alloc<Cfg::kTmemCols>(tmem_slot);
  }
  tc_fence_before();
  if constexpr (PAIR) cluster_sync();  // barriers initialised in both CTAs
  else __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  // Prologue done: let the next layer launch. Only the producer waits for
  // the previous layer (pdl_wait below), after issuing the weight (B) boxes
  // of the first ring pass -- parameters; the activation loads follow the
  // wait and every later step is ordered after them by mbarriers.
  pdl_launch_dependents();

  if (warp == 0) {
    // ------------------------------------------------ TMA producer warp
    if (elect_one()) {
      int pre = 0;  // stages whose B box went out before the wait
      // the full barrier the loads complete on: the leader's for a pair
      const uint32_t full_l = PAIR ? mapa_u32(smem_u32(full), 0) : 0u;
      const int b_row = PAIR ? static_cast<int>(rank) * (BN / 2) : 0;
      auto load_b = [&](int st, int kcol, int n_tile) {
        if constexpr (PAIR)
          tma_load_2d_pair(sB + st * Cfg::kBBytes, &tm_b, full_l + 8 * st, kcol, n_tile * BN + b_row);
        else
          tma_load_2d(sB + st * Cfg::kBBytes, &tm_b, &full[st], kcol, n_tile * BN);
      };
      if (t_first < t_count) {
        const int t0 = tile_of(t_first);
        const int mn = t0 / splits;
        const int n_tile0 = mn % p.n_tiles;
        const int kb = (t0 - mn * splits) * kps;
        const int ke = min(k_iters, kb + kps);
        for (int k = kb; k < ke && pre < STAGES; ++k, ++pre) {
          if (!PAIR || rank == 0) mbar_arrive_expect_tx(&full[pre], kStageTx);
          // k = (r * S + s) * cblocks + cb -> weight column k * kCB
          load_b(pre, k * kCB, n_tile0);
        }
      }
      pdl_wait();
      int stage = 0;
      uint32_t phase = 0;
      const int ohw = p.oh * p.ow;
      for (int u = t_first; u < t_count; u += t_step) {
        const int tile = tile_of(u);
        const int mn = tile / splits;
        const int split = tile - mn * splits;
        const int m_tile = mn / p.n_tiles;
        const int n_tile = mn - m_tile * p.n_tiles;
        // a pair's phantom tile (odd m_tiles) reads its partner's rows
        const int m0 = min(m_tile, p.m_tiles - 1) * kBM;
        const int img = m0 / ohw;
        const int rem = m0 - img * ohw;
        const int oh = rem / p.ow;
        const int ow = rem - oh * p.ow;
        const int w0 = ow * p.sw - p.pw;
        const int h0 = oh * p.sh - p.ph;
        const int kb = split * kps, ke = min(k_iters, kb + kps);
        // k index = (r * S + s) * cblocks + cb, walked incrementally
        int r = kb / sc, rem_k = kb - r * sc;
        int s = rem_k / p.cblocks, cb = rem_k - s * p.cblocks;
        for (int k = kb; k < ke; ++k) {
          auto load_a = [&]() {
            if constexpr (PAIR)
              tma_load_im2col_4d_pair(sA + stage * Cfg::kABytes, &tm_a, full_l + 8 * stage,
                                      cb * kCB, w0, h0, img, static_cast<uint16_t>(s),
                                      static_cast<uint16_t>(r));
            else
              tma_load_im2col_4d(sA + stage * Cfg::kABytes, &tm_a, &full[stage], cb * kCB, w0,
                                 h0, img, static_cast<uint16_t>(s), static_cast<uint16_t>(r));
          };
          if (pre > 0) {  // B already in flight, the stage known free
            --pre;
            load_a();
          } else {
          { const long long t0 = p.dbg ? clock64() : 0;
            mbar_wait(&empty[stage], phase ^ 1);
            if (p.dbg) dbg_wait[0] += clock64() - t0; }
          if (!PAIR || rank == 0) mbar_arrive_expect_tx(&full[stage], kStageTx);
          load_a();
          load_b(stage, (r * p.s + s) * p.cp + cb * kCB, n_tile);
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
  } else if (warp == 1 && (!PAIR || rank == 0)) {
    // ------------------------------------------ single-thread MMA issuer
    if (elect_one()) {
      constexpr uint32_t idesc = make_idesc<KIND>(PAIR ? 2 * kBM : kBM, BN);
      int stage = 0;
      uint32_t phase = 0;
      int local = 0;
      // The tensor pipe queues only about one group of MMAs, so the scalar
      // work between stages on this thread is pipe idle time: descriptors
      // are advanced by adding to their 16-byte address field (shared
      // addresses < 256 KB), parameters live in registers (the asm "memory"
      // clobbers would re-read them from the constant bank), the split of a
      // tile is stepped instead of divided.
      const uint64_t adesc0 = make_smem_desc<SWZ>(smem_u32(sA), 8 * SWZ);
      const uint64_t bdesc0 = make_smem_desc<SWZ>(smem_u32(sB), 8 * SWZ);
      const int nsplit = splits, kps_ = kps, kit = k_iters;
      const bool dbg = p.dbg != nullptr;
      int split = static_cast<int>(blockIdx.x) % nsplit;
      const int dsplit = static_cast<int>(gridDim.x) % nsplit;
      for (int u = t_first; u < t_count; u += t_step, ++local) {
        const int acc = local & (nacc - 1);
        const uint32_t use = static_cast<uint32_t>(local >> acc_shift);
        { const long long t0 = dbg ? clock64() : 0;
          mbar_wait(&tempty[acc], (use & 1) ^ 1);
          if (dbg) dbg_wait[2] += clock64() - t0; }
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * BN;
        const int kb = split * kps_, ke = min(kit, kb + kps_);
        split += dsplit;
        if (split >= nsplit) split -= nsplit;
        for (int k = kb; k < ke; ++k) {
          { const long long t0 = dbg ? clock64() : 0;
            mbar_wait(&full[stage], phase);
            if (dbg) dbg_wait[1] += clock64() - t0; }
          tc_fence_after();
          const uint64_t ad = adesc0 + static_cast<uint64_t>(stage * (Cfg::kABytes >> 4));
          const uint64_t bd = bdesc0 + static_cast<uint64_t>(stage * (Cfg::kBBytes >> 4));
#pragma unroll
          for (int kk = 0; kk < Cfg::kMmaPerStage; ++kk) {
            if constexpr (PAIR)
              tc_mma_pair<KIND>(d_tmem, ad + 2 * kk, bd + 2 * kk, idesc,
                                (k != kb || kk != 0) ? 1u : 0u);
            else
              tc_mma<KIND>(d_tmem, ad + 2 * kk, bd + 2 * kk, idesc,  // K slice kk: +32 B
                           (k != kb || kk != 0) ? 1u : 0u);
          }
          // frees the smem slot (both CTAs' for a pair) when the MMAs land
          if constexpr (PAIR) tc_commit_pair(&empty[stage], 3);
          else tc_commit(&empty[stage]);
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
        // accumulator ready for the epilogue (both CTAs' for a pair)
        if constexpr (PAIR) tc_commit_pair(&tfull[acc], 3);
        else tc_commit(&tfull[acc]);
      }
    }
  } else if (warp >= 4) {
    // ------------------------------------------------- epilogue warps
    // Two groups of 4 warps; group g drains accumulator g, i.e. every
    // other tile, so two tiles' epilogues proceed concurrently. Warp w reads
    // TMEM lane quadrant (w % 4) = 32 output rows, all BN columns.
    const uint32_t q = warp & 3;
    const int grp = static_cast<int>(warp - 4) >> 2;
    const int gtid = static_cast<int>(threadIdx.x) - (kThreads - kEpiThreads) - grp * 128;
    uint8_t* stage = sStage + (warp - 4) * 4096;
    const bool coalesced =
        p.epi_mode == 0 &&
        ((KIND == MmaKind::kI8 || p.out_type != kBF16) ? (p.oc % 4) == 0 : (p.oc % 8) == 0);
    const epi::EpiProg prog = epi::make_prog(p.epi);
    const int fast = epi::classify_prog(p.epi);
    const bool tma_epi = p.tma_store && p.epi_mode == 0 && fast != epi::kProgGeneric &&
                         fast != epi::kProgBiasAddRelu;
    const uint32_t stage_u32 = smem_u32(stage);
    uint32_t box_cnt = 0;
    int local = 0;
    int staged_n_tile = -1;
    bool overflow = false;
    // hand the accumulator back: the peer of a pair arrives on the leader's
    const uint32_t tempty_l = PAIR ? mapa_u32(smem_u32(tempty), 0) : 0u;
    auto release_acc = [&](int a) {
      if constexpr (PAIR) {
        if (rank != 0) {
          mbar_arrive_cluster(tempty_l + 8 * a);
          return;
        }
      }
      mbar_arrive(&tempty[a]);
    };
    for (int u = t_first; u < t_count; u += t_step, ++local) {
      const int tile = tile_of(u);
      if ((local & 1) != grp) continue;
      const int acc = local & (nacc - 1);
      const uint32_t use = static_cast<uint32_t>(local >> acc_shift);
      const int mn = tile / splits;
      const int split = tile - mn * splits;
      const int m_tile = mn / p.n_tiles;
      const int n_tile = mn - m_tile * p.n_tiles;
      const int row0 = m_tile * kBM + static_cast<int>(q * 32);
      const int row = row0 + static_cast<int>(lane);
      const bool row_ok = row < p.m;
      // Per-tile bias copy in smem (one buffer per group).
      uint32_t* bias_s = sBias + grp * BN;
      // The group's bias buffer only changes with the output-channel tile
      // (a global load + two barriers on the per-tile critical path).
      if (n_tile != staged_n_tile) {
        epi::named_bar_sync(1 + grp, 128);  // previous tile's readers are done
        epi::stage_bias(bias_s, p.epi.bias, n_tile * BN, BN, p.oc, gtid, 128);
        epi::named_bar_sync(1 + grp, 128);
        staged_n_tile = n_tile;
      }
      const long long tw0 = p.dbg ? clock64() : 0;
      mbar_wait(&tfull[acc], use & 1);
      const long long tw1 = p.dbg ? clock64() : 0;
      if (p.dbg) dbg_wait[3] += tw1 - tw0;
      tc_fence_after();
      if (PAIR && m_tile >= p.m_tiles) {  // a pair's phantom tile: nothing to store
        tc_fence_before();
        release_acc(acc);
        continue;
      }
      if (splits > 1 && tma_epi) {
        // ---- split-K: publish this split's f32 partial tile, then the last
        // split of the tile (arrival counter) sums all partials IN SPLIT
        // ORDER (deterministic) and runs the fused epilogue.
        // Partial layout [item][warp q][chunk][column j][lane]: for a fixed
        // register j the 32 lanes write one contiguous 128-byte line.
        const uint32_t taddr = tmem_base + ((q * 32) << 16) + acc * BN;
        float* mine = p.ws + ((static_cast<size_t>(mn) * splits + split) * 4 + q) * 32 * BN + lane;
#pragma unroll 1
        for (int c0 = 0; c0 < BN; c0 += kChunk) {
          uint32_t v[kChunk];
          tmem_ld32(taddr + c0, v);
          tmem_ld_wait();
#pragma unroll
          for (int j = 0; j < kChunk; ++j) __stcg(mine + (c0 + j) * 32, __uint_as_float(v[j]));
        }
        tc_fence_before();
        release_acc(acc);  // TMEM free: the partial lives in ws now
        __threadfence();
        epi::named_bar_sync(1 + grp, 128);
        if (gtid == 0) s_last[grp] = atomicAdd(&p.tile_cnt[mn], 1) == splits - 1;
        epi::named_bar_sync(1 + grp, 128);
        if (s_last[grp]) {
          __threadfence();
          const float* part = p.ws + (static_cast<size_t>(mn) * splits * 4 + q) * 32 * BN + lane;
          const size_t pstride = static_cast<size_t>(4) * 32 * BN;  // one split's tile
          auto src = [&](int c0, uint32_t (&a)[epi::kChunk]) {
            float f[epi::kChunk];
#pragma unroll
            for (int j = 0; j < epi::kChunk; ++j) f[j] = __ldcg(part + (c0 + j) * 32);
#pragma unroll 1
            for (int sp = 1; sp < splits; ++sp) {
#pragma unroll
              for (int j = 0; j < epi::kChunk; ++j)
                f[j] = __fadd_rn(f[j], __ldcg(part + sp * pstride + (c0 + j) * 32));
            }
#pragma unroll
            for (int j = 0; j < epi::kChunk; ++j) a[j] = __float_as_uint(f[j]);
          };
          if constexpr (KIND != MmaKind::kI8) {
            auto run = [&](auto prog_c, auto es_c) {
              constexpr int kProg = decltype(prog_c)::value, kES = decltype(es_c)::value;
              epi::epi_rows_tma_src<kProg, kES, BN, false>(
                  src, static_cast<int>(lane), bias_s, stage_u32, p.oc - n_tile * BN, box_cnt,
                  &overflow, [&](uint32_t box, int c0) {
                    tma_store_2d(&tm_y, box, n_tile * BN + c0, row0);
                  });
            };
            using P0 = std::integral_constant<int, epi::kProgNone>;
            using P1 = std::integral_constant<int, epi::kProgBias>;
            using P2 = std::integral_constant<int, epi::kProgBiasRelu>;
            using E2 = std::integral_constant<int, 2>;
            using E4 = std::integral_constant<int, 4>;
            if (p.out_type == kBF16) {
              if (fast == epi::kProgNone) run(P0{}, E2{});
              else if (fast == epi::kProgBias) run(P1{}, E2{});
              else run(P2{}, E2{});
            } else {
              if (fast == epi::kProgNone) run(P0{}, E4{});
              else if (fast == epi::kProgBias) run(P1{}, E4{});
              else run(P2{}, E4{});
            }
          }
          if (gtid == 0) p.tile_cnt[mn] = 0;  // ready for the next launch
        }
        if (p.dbg) dbg_wait[4] += clock64() - tw1;
        continue;
      }
      {
        if (tma_epi) {
          // One 2-D box store per 32 columns; rows >= M are clipped.
          constexpr bool kInt = KIND == MmaKind::kI8;
          auto run = [&](auto prog_c, auto es_c) {
            constexpr int kProg = decltype(prog_c)::value, kES = decltype(es_c)::value;
            // the Q programs' i8 residual row (int8 graphs); NULL past M
            const uint8_t* rrow = nullptr;
            if constexpr (kProg == epi::kProgBiasAddReluQ)
              if (row_ok)
                rrow = static_cast<const uint8_t*>(p.epi.residual) +
                       static_cast<int64_t>(row) * p.oc + n_tile * BN;
            epi::QParams qp;
            qp.mult = p.epi.rq_mult;
            qp.shift = p.epi.rq_shift;
            qp.res_scale = p.epi.res_scale;
            epi::epi_rows_tma<kProg, kES, BN, kInt>(
                tmem_base + ((q * 32) << 16) + acc * BN, static_cast<int>(lane), bias_s,
                stage_u32, p.oc - n_tile * BN, box_cnt, &overflow, [&](uint32_t box, int c0) {
                  tma_store_2d(&tm_y, box, n_tile * BN + c0, row0);
                }, rrow, qp);
          };
          using P0 = std::integral_constant<int, epi::kProgNone>;
          using P1 = std::integral_constant<int, epi::kProgBias>;
          using P2 = std::integral_constant<int, epi::kProgBiasRelu>;
          using PQ = std::integral_constant<int, epi::kProgBiasReluQ>;
          using PAQ = std::integral_constant<int, epi::kProgBiasAddReluQ>;
          using PBQ = std::integral_constant<int, epi::kProgBiasQ>;
          using E1 = std::integral_constant<int, 1>;
          using E2 = std::integral_constant<int, 2>;
          using E4 = std::integral_constant<int, 4>;
          if constexpr (kInt) {
            if (fast == epi::kProgNone) run(P0{}, E4{});
            else if (fast == epi::kProgBias) run(P1{}, E4{});
            else if (fast == epi::kProgBiasReluQ) run(PQ{}, E1{});
            else if (fast == epi::kProgBiasAddReluQ) run(PAQ{}, E1{});
            else if (fast == epi::kProgBiasQ) run(PBQ{}, E1{});
            else run(P2{}, E4{});
          } else if (p.out_type == kBF16) {
            if (fast == epi::kProgNone) run(P0{}, E2{});
            else if (fast == epi::kProgBias) run(P1{}, E2{});
            else run(P2{}, E2{});
          } else {
            if (fast == epi::kProgNone) run(P0{}, E4{});
            else if (fast == epi::kProgBias) run(P1{}, E4{});
            else run(P2{}, E4{});
          }
          tc_fence_before();
          release_acc(acc);
          if (p.dbg) dbg_wait[4] += clock64() - tw1;
          continue;
        }
      }
      const int my_row = row_ok ? row : -1;
#pragma unroll 1
      for (int c0 = 0; c0 < BN && p.epi_mode != 2; c0 += kChunk) {  // 2: no epilogue (diagnostic)
        const uint32_t taddr = tmem_base + ((q * 32) << 16) + acc * BN + c0;
        const int col0 = n_tile * BN + c0;
        if (coalesced) {
          if (col0 < p.oc)
            epi::epi_block<KIND == MmaKind::kI8>(p, prog, fast, taddr, col0, lane, my_row,
                                                 bias_s + c0, stage, &overflow);
        } else {
          uint32_t v[kChunk];
          tmem_ld32(taddr, v);
          const bool active = row_ok && col0 < p.oc;
          const int ncols = min(kChunk, p.oc - col0);
          epi::epi_row_chunk<KIND == MmaKind::kI8>(p, prog, row, col0, ncols, active,
                                                   bias_s + c0, v, &overflow);
        }
      }
      // All of this thread's TMEM reads of the accumulator are complete
      // (each block waited on tcgen05.ld): hand it back to the MMA warp.
      tc_fence_before();
      release_acc(acc);
      if (p.dbg) dbg_wait[4] += clock64() - tw1;
    }
    if (lane == 0) bulk_wait_all();  // TMA stores done before smem goes away
    if (overflow && p.err) atomicOr(p.err, 1);
  }

  tc_fence_before();
  if constexpr (PAIR) cluster_sync();  // no DSMEM traffic may target an exited CTA
  else __syncthreads();
  tc_fence_after();
  if (warp == 2) {
    if constexpr (PAIR) tmem_dealloc_pair<Cfg::kTmemCols>(tmem_base);
    else tmem_dealloc<Cfg::kTmemCols>(tmem_base);
  }
  if (p.dbg) {
    // one representative thread per role: producer / MMA lane 0 of warps
    // 0 / 1, and epilogue thread 0 (its waits are typical of the group).
    const bool rep = (warp <= 1 && lane == 0) || threadIdx.x == kThreads - kEpiThreads;
    if (rep)
      for (int i = 0; i < 5; ++i)
        if (dbg_wait[i]) atomicAdd(&p.dbg[i], static_cast<unsigned long long>(dbg_wait[i]));
    if (threadIdx.x == 0) {
      atomicAdd(&p.dbg[5], static_cast<unsigned long long>(clock64() - t_start));
      atomicAdd(&p.dbg[6], static_cast<unsigned long long>((num_tiles - blockIdx.x + gridDim.x - 1) / gridDim.x));
    }
  }
}

}  // namespace

// Launch wrapper, instantiated for the supported (kind, BN, swizzle) set.
// Returns a cudaError_t.
// PAIR: grid even, launched in clusters of 2 (the CTA pairs).
template <MmaKind KIND, int BN, int STAGES, int SWZ, bool PAIR>
int launch_conv_fprop_tc(const CUtensorMap& tm_a, const CUtensorMap& tm_b,
                         const CUtensorMap& tm_y, const ConvGemmParams& p, int grid,
                         cudaStream_t stream) {
  using Cfg = ConvCfg<KIND, BN, STAGES, SWZ, PAIR>;
  auto kfn = conv_fprop_tc_kernel<KIND, BN, STAGES, SWZ, PAIR>;
  cudaError_t e = cudaFuncSetAttribute(
      kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::kSmemBytes);
  if (e != cudaSuccess) return e;
  if constexpr (PAIR)
    e = launch_pdl_cluster(kfn, dim3(grid), dim3(kThreads), Cfg::kSmemBytes, stream, 2, tm_a,
                           tm_b, tm_y, p);
  else
    e = launch_pdl(kfn, dim3(grid), dim3(kThreads), Cfg::kSmemBytes, stream, tm_a, tm_b, tm_y, p);
  if (e != cudaSuccess) return e;
  return cudaGetLastError();
}

#define TEC_INST(KIND, BN, ST, SWZ)                                         \
  template int launch_conv_fprop_tc<KIND, BN, ST, SWZ, false>(             \
      const CUtensorMap&, const CUtensorMap&, const CUtensorMap&,          \
      const ConvGemmParams&, int, cudaStream_t);
#define TEC_INST_PAIR(KIND, BN, ST, SWZ)                                    \
  template int launch_conv_fprop_tc<KIND, BN, ST, SWZ, true>(              \
      const CUtensorMap&, const CUtensorMap&, const CUtensorMap&,          \
      const ConvGemmParams&, int, cudaStream_t);

// bf16: 128 B channel blocks (64 ch) for Cp % 64 == 0, 32 B (16 ch) for
// the stem (C1, 3 -> 16 padded channels).
TEC_INST(MmaKind::kF16, 64, 8, 128)
TEC_INST(MmaKind::kF16, 128, 6, 128)
TEC_INST(MmaKind::kF16, 256, 3, 128)
TEC_INST(MmaKind::kF16, 64, 8, 32)
// int8: 128 B blocks (128 ch), 64 B (64 ch), 32 B (32 ch, the stem).
TEC_INST(MmaKind::kI8, 64, 8, 128)
TEC_INST(MmaKind::kI8, 128, 6, 128)
TEC_INST(MmaKind::kI8, 256, 3, 128)
TEC_INST(MmaKind::kI8, 64, 8, 64)
TEC_INST(MmaKind::kI8, 128, 6, 64)
TEC_INST(MmaKind::kI8, 64, 8, 32)
// CTA pairs (knob cluster_n = 2 on the im2col path)
// (the half-size weight stages buy deeper rings in the same shared memory)
TEC_INST_PAIR(MmaKind::kF16, 64, 9, 128)
TEC_INST_PAIR(MmaKind::kF16, 128, 8, 128)
TEC_INST_PAIR(MmaKind::kF16, 256, 5, 128)
TEC_INST_PAIR(MmaKind::kI8, 64, 9, 128)
TEC_INST_PAIR(MmaKind::kI8, 128, 8, 128)
TEC_INST_PAIR(MmaKind::kI8, 256, 5, 128)
TEC_INST_PAIR(MmaKind::kI8, 64, 9, 64)
TEC_INST_PAIR(MmaKind::kI8, 128, 8, 64)

#undef TEC_INST
#undef TEC_INST_PAIR

}  // namespace tec_sm100
