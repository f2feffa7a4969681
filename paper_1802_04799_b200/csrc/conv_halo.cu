// conv_halo.cu -- stride-1 fused conv2d as a shifted-window implicit GEMM.
//
// Why: the im2col kernel (conv_tc.cu) re-reads every input pixel R*S times
// from L2 (once per filter tap). For ResNet's 3x3 layers that is 9x the
// activation bytes per CTA tile and the kernel becomes L2->SM bandwidth
// bound (ncu: 347 MB of L2->SM traffic for the 25.7 MB C2 input). Here a
// CTA loads the input rows of its tile ONCE per channel block -- one tiled
// TMA box with the zero padding supplied by TMA out-of-bounds fill -- and
// every filter tap is a different start address into that halo:
//
//   halo pixel q = row * wp + col      (wp = W + 2*pw; 128 B per pixel)
//   output virtual row v = oh_local * wp + ow
//   tap (rh, rw) reads halo pixel v + rh * wp + rw
//
// The SWIZZLE_128B K-major UMMA descriptor accepts any 128-B-row start
// (the swizzle is a function of the absolute smem address; verified on
// B200 by tools/microbench/umma_shift_test.cu), so the shift is free. Virtual rows
// with ow >= OW are junk and never stored (wp/OW extra work: 3.6% on C2).
//
// Pipelines (the paper's virtual-thread latency hiding, as mbarriers):
//   halo ring (2 stages)   : TMA producer -> MMA, one stage per channel block
//   weight ring (WSTAGES)  : one (tap, channel block) B tile per stage
//   TMEM accumulators      : 2 x MS x BN columns, MMA <-> epilogue
// Weights per tap are reused by all MS*128 virtual rows of the tile.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <type_traits>

#include "conv_epilogue.cuh"
#include "conv_params.h"
#include "sm100_ptx.cuh"

namespace tec_sm100 {

namespace {

constexpr int kThreads = 384;     // 4 control warps + 8 epilogue warps
constexpr int kEpiThreads = 256;

template <int BN, int MS, int SWZ, int WSTAGES, bool kPair = false>
struct HaloCfg {
  static constexpr int kWBytes = BN * SWZ;
  // kPair: every sub-tile accumulator is [lo BN | hi BN] columns (see below)
  static constexpr uint32_t kAccCols = MS * BN * (kPair ? 2 : 1);
  // TMEM accumulator buffers (knob acc_bufs; the paper's virtual threads):
  // up to 4 when they fit, so the MMA can run ahead of a slow epilogue.
  static constexpr int kMaxAcc = 4 * kAccCols <= 512 ? 4 : 2;
  static constexpr uint32_t kTmemCols = kMaxAcc * kAccCols <= 32    ? 32
                                        : kMaxAcc * kAccCols <= 64  ? 64
                                        : kMaxAcc * kAccCols <= 128 ? 128
                                        : kMaxAcc * kAccCols <= 256 ? 256
                                                                    : 512;
  static_assert(2 * kAccCols <= 512, "TMEM holds at most 512 columns");
  static constexpr int kMmaPerTap = SWZ / 32;
};

__host__ __device__ inline int halo_bytes_aligned(int halo_px, int swz) {
  return (halo_px * swz + 1023) & ~1023;
}

// Paired taps (kPair, resident weights, BN = 64): the weight tiles of taps
// (rh, rw) and (rh, rw + 1) sit next to each other in shared memory, i.e.
// they ARE one 128-row B tile. One N=128 MMA at the A shift of (rh, rw)
// computes  lo = X[v + s] * W(rh, rw)      -> output row v     (columns 0..63)
//           hi = X[v + s] * W(rh, rw + 1)  -> output row v - 1 (columns 64..127)
// because tap (rh, rw + 1) of output v - 1 reads exactly X[v + s]. The same
// one-row offset holds for every pair, so one hi accumulator collects them
// all and the epilogue adds hi of row v + 1 to lo of row v (a lane shuffle;
// the last lane of each warp takes it from the next warp through shared
// memory). An odd last tap runs as a plain N=64 MMA into lo. N=128 MMAs cost
// 64 cycles vs 54 for N=64 (tools/microbench/RESULTS.md), so a 3x3 filter
// row drops from 3 x 54 to 64 + 54 cycles and a 4-tap row to 2 x 64.
template <MmaKind KIND, int BN, int MS, int SWZ, int WSTAGES, bool kPair = false>
__global__ void __launch_bounds__(kThreads, 1)
    conv_halo_kernel(const __grid_constant__ CUtensorMap tm_x,
                     const __grid_constant__ CUtensorMap tm_w,
                     const __grid_constant__ CUtensorMap tm_y,
                     const ConvHaloParams p) {
  using Cfg = HaloCfg<BN, MS, SWZ, WSTAGES, kPair>;
  static_assert(!kPair || (BN == 64 && KIND == MmaKind::kF16), "paired taps: bf16, BN = 64");
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int hbytes = halo_bytes_aligned(p.halo_px, SWZ);
  uint8_t* sH = smem;                       // 2 halo buffers
  uint8_t* sW = smem + 2 * hbytes;          // WSTAGES weight tiles
  uint8_t* sStage = sW + p.w_slots * Cfg::kWBytes;  // epilogue stage (>= 8 warps x 4 KB)
  uint64_t* hfull = reinterpret_cast<uint64_t*>(sStage + p.stage_bytes);
  uint64_t* hempty = hfull + 2;
  uint64_t* wfull = hempty + 2;
  uint64_t* wempty = wfull + WSTAGES;
  uint64_t* tfull = wempty + WSTAGES;
  uint64_t* tempty = tfull + 4;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 4);
  uint32_t* sBias = reinterpret_cast<uint32_t*>(
      reinterpret_cast<uint8_t*>(hfull) + 256);  // [2][BN] f32 / i32
  float* sXchg = reinterpret_cast<float*>(sBias + 2 * BN);  // kPair: [2 grp][MS][4 warps][64]

  const uint32_t warp = warp_id();
  const uint32_t lane = threadIdx.x & 31;
  // accumulator ring: tile `local` uses buffer local % nacc; epilogue group
  // local % 2 drains it (nacc even: a buffer always belongs to one group)
  const int nacc = p.nacc == 4 && Cfg::kMaxAcc == 4 ? 4 : 2;
  const int acc_shift = nacc == 4 ? 2 : 1;
  const int taps = p.r * p.s;
  const int num_tiles = p.n * p.bands * p.n_tiles;
  long long dbg_wait[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  const long long t_start = p.dbg ? clock64() : 0;
  constexpr int kCB =
      SWZ / (KIND == MmaKind::kF16 ? 2 : KIND == MmaKind::kTF32 ? 4 : 1);
  const uint32_t halo_tx = static_cast<uint32_t>((p.th + p.r - 1) * p.wp * SWZ);
  // Weight multicast (p.cl > 1, streamed weights): the cl CTAs of a cluster
  // work on the same output-channel tile at the same time; each loads 1/cl
  // of every weight tile and multicasts it to all, so weights cross L2->SM
  // once per cluster instead of once per CTA.
  const int cl = p.cl > 1 && !p.resident ? p.cl : 1;
  const int crank = cl > 1 ? static_cast<int>(cluster_ctarank()) : 0;
  const uint16_t cmask = static_cast<uint16_t>((1u << cl) - 1u);

  if (warp == 0 && elect_one()) {
    tma_prefetch_desc(&tm_x);
    tma_prefetch_desc(&tm_w);
    if (p.tma_store) tma_prefetch_desc(&tm_y);
    for (int i = 0; i < 2; ++i) {
      mbar_init(&hfull[i], 1);
      mbar_init(&hempty[i], 1);
    }
    for (int i = 0; i < 4; ++i) {
      mbar_init(&tfull[i], 1);
      mbar_init(&tempty[i], 128);  // the epilogue group of the accumulator
    }
    for (int i = 0; i < WSTAGES; ++i) {
      mbar_init(&wfull[i], 1);
      mbar_init(&wempty[i], cl);  // every CTA of the cluster releases the slot
    }
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc<Cfg::kTmemCols>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  // Weight multicast: peers write into this CTA's shared memory and arrive
  // on its barriers, so every CTA of the cluster must have initialised its
  // barriers before any of them issues a load (cluster-scope release/acquire).
  if (p.cl > 1 && !p.resident) cluster_sync();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  // Let the next layer launch. Only the producer waits for the previous one
  // (pdl_wait below), after issuing the resident weights (parameters): the
  // halo loads follow the wait, and every later step -- MMAs, epilogue reads
  // of the residual, output writes -- is ordered after them by mbarriers.
  pdl_launch_dependents();

  // Tile order. Streamed weights: tiles strided over the grid, N fastest.
  // Resident weights (p.resident): each CTA keeps ONE output-channel tile
  // (n_tile = blockIdx.x % n_tiles) and loads all of its weights once.
  const int spatial = p.n * p.bands;
  const int ctas_per_n = static_cast<int>(gridDim.x) / p.n_tiles;
  const int nclusters = static_cast<int>(gridDim.x) / cl;
  const int cunits = ((spatial + cl - 1) / cl) * p.n_tiles;
  // *dummy: a cluster's last spatial group may leave a CTA without a tile;
  // it still runs the shared weight pipeline, but loads and stores nothing.
  auto tile_at = [&](int i, int* n_tile, int* band, int* img, bool* dummy = nullptr) -> bool {
    int s;
    if (dummy) *dummy = false;
    if (cl > 1) {
      const int unit = static_cast<int>(blockIdx.x) / cl + i * nclusters;
      if (unit >= cunits) return false;
      *n_tile = unit % p.n_tiles;
      s = (unit / p.n_tiles) * cl + crank;
      if (s >= spatial) {
        if (dummy) *dummy = true;
        s = spatial - 1;
      }
    } else if (p.resident) {
      s = static_cast<int>(blockIdx.x) / p.n_tiles + i * ctas_per_n;
      if (s >= spatial || static_cast<int>(blockIdx.x) >= ctas_per_n * p.n_tiles) return false;
      *n_tile = static_cast<int>(blockIdx.x) % p.n_tiles;
    } else {
      const int tile = static_cast<int>(blockIdx.x) + i * static_cast<int>(gridDim.x);
      if (tile >= num_tiles) return false;
      *n_tile = tile % p.n_tiles;
      s = tile / p.n_tiles;
    }
    *band = s % p.bands;
    *img = s / p.bands;
    return true;
  };

  if (warp == 0) {
    // ------------------------------------------------ TMA producer
    if (elect_one()) {
      int hs = 0, ws = 0;
      uint32_t hph = 0, wph = 0;
      int n_tile, band, img;
      const int res_es = p.out_type == kBF16 ? 2 : 4;
      const bool res_prefetch = KIND != MmaKind::kI8 && SWZ == 128 && p.n_tiles == 1 &&
                                epi::classify_prog(p.epi) == epi::kProgBiasAddRelu &&
                                (p.th * p.ow * p.oc * res_es) % 16 == 0 &&
                                (p.ow * p.oc * res_es) % 16 == 0;
      if (p.resident && tile_at(0, &n_tile, &band, &img)) {
        // every (tap, channel block) weight tile of this CTA's N tile, once
        mbar_arrive_expect_tx(&wfull[0], static_cast<uint32_t>(taps * p.cblocks * Cfg::kWBytes));
        for (int cb = 0; cb < p.cblocks; ++cb)
          for (int t = 0; t < taps; ++t)
            tma_load_2d(sW + (cb * taps + t) * Cfg::kWBytes, &tm_w, &wfull[0],
                        t * p.cp + cb * kCB, n_tile * BN);
      }
      // streamed weights (no cluster): the first ring pass before the wait too
      int wpre = 0;
      if (!p.resident && cl == 1 && tile_at(0, &n_tile, &band, &img)) {
        for (int j = 0; j < taps * p.cblocks && wpre < WSTAGES; ++j, ++wpre) {
          const int cb = j / taps, t = j - cb * taps;
          mbar_arrive_expect_tx(&wfull[wpre], Cfg::kWBytes);
          tma_load_2d(sW + wpre * Cfg::kWBytes, &tm_w, &wfull[wpre], t * p.cp + cb * kCB,
                      n_tile * BN);
        }
      }
      pdl_wait();
      bool dummy = false;
      for (int i = 0; tile_at(i, &n_tile, &band, &img, &dummy); ++i) {
        const int ih0 = band * p.th - p.ph;
        for (int cb = 0; cb < p.cblocks; ++cb) {
          { const long long t0 = p.dbg ? clock64() : 0;
            mbar_wait(&hempty[hs], hph ^ 1);
            if (p.dbg) dbg_wait[0] += clock64() - t0; }
          if (dummy) {
            mbar_arrive(&hfull[hs]);  // nothing to load; the MMAs run on stale data
          } else {
            mbar_arrive_expect_tx(&hfull[hs], halo_tx);
            // box {CB, wp, th + r - 1, 1} at (c, -pw, ih0, img); TMA fills
            // the out-of-image pixels with zeros (the select(..., 0) pad).
            tma_load_4d(sH + hs * hbytes, &tm_x, &hfull[hs], cb * kCB, -p.pw, ih0, img);
            if (cb == 0 && res_prefetch) {
              // the tile's residual rows are one contiguous NHWC block when
              // the tile spans every output channel: into L2 two tiles ahead
              const int oh0 = band * p.th, rows = min(p.th, p.oh - oh0);
              bulk_prefetch_l2(static_cast<const uint8_t*>(p.epi.residual) +
                                   static_cast<int64_t>(img * p.oh + oh0) * p.ow * p.oc * res_es,
                               static_cast<uint32_t>(rows * p.ow * p.oc * res_es));
            }
          }
          if (++hs == 2) { hs = 0; hph ^= 1; }
          if (p.resident) continue;
          for (int t = 0; t < taps; ++t) {
            if (wpre > 0) {  // issued before the wait
              --wpre;
              if (++ws == WSTAGES) { ws = 0; wph ^= 1; }
              continue;
            }
            { const long long t0 = p.dbg ? clock64() : 0;
              mbar_wait(&wempty[ws], wph ^ 1);
              if (p.dbg) dbg_wait[0] += clock64() - t0; }
            mbar_arrive_expect_tx(&wfull[ws], Cfg::kWBytes);
            if (cl > 1) {  // this CTA's 1/cl row slice of the tile, to every CTA
              const int rows = BN / cl;
              tma_load_2d_mc(sW + ws * Cfg::kWBytes + crank * rows * SWZ, &tm_w, &wfull[ws],
                             t * p.cp + cb * kCB, n_tile * BN + crank * rows, cmask);
            } else {
              tma_load_2d(sW + ws * Cfg::kWBytes, &tm_w, &wfull[ws],
                          t * p.cp + cb * kCB, n_tile * BN);
            }
            if (++ws == WSTAGES) { ws = 0; wph ^= 1; }
          }
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------ single-thread MMA issuer
    if (elect_one()) {
      constexpr uint32_t idesc = make_idesc<KIND>(128, BN);
      int hs = 0, ws = 0;
      uint32_t hph = 0, wph = 0;
      int n_tile, band, img;
      if (p.resident) {
        const long long t0 = p.dbg ? clock64() : 0;
        mbar_wait(&wfull[0], 0);
        if (p.dbg) dbg_wait[1] += clock64() - t0;
      }
      // Descriptors are built once and advanced by adding (byte offset >> 4)
      // to the start-address field (smem addresses < 2^18, no carry-out).
      //
      // The issue loop is the MMA rate limiter when it is not lean: one
      // thread issues every MMA, and ncu showed the earlier version (tap
      // index division, per-tap parameter reloads) spending ~1000 cycles
      // per tap for 8 MMAs that execute in ~430. Taps are therefore walked
      // as (rh, rw) with incremental descriptor offsets, the resident /
      // streamed choice is a compile-time branch, and all per-MMA offsets
      // are immediates.
      const uint64_t wdesc0 = make_smem_desc<SWZ>(smem_u32(sW), 8 * SWZ);
      const bool dbg = p.dbg != nullptr;
      const int pr = p.r, ps = p.s, cblocks = p.cblocks;
      const uint32_t row_skip = static_cast<uint32_t>((p.wp - ps) * SWZ) >> 4;
      if constexpr (kPair) {
        // resident weights only (host guarantees); see the comment at the top
        constexpr uint32_t idesc2 = make_idesc<KIND>(128, 2 * BN);
        const int npair = ps >> 1;
        const uint32_t odd_skip = static_cast<uint32_t>(((ps & 1) ? 1 : 0) * SWZ) >> 4;
        for (int local = 0; tile_at(local, &n_tile, &band, &img); ++local) {
          const int acc = local & (nacc - 1);
          const uint32_t use = static_cast<uint32_t>(local >> acc_shift);
          { const long long t0 = dbg ? clock64() : 0;
            mbar_wait(&tempty[acc], (use & 1) ^ 1);
            if (dbg) dbg_wait[2] += clock64() - t0; }
          tc_fence_after();
          const uint32_t d0 = tmem_base + acc * Cfg::kAccCols;
          uint64_t bd = wdesc0;
          for (int cb = 0; cb < cblocks; ++cb) {
            { const long long t0 = dbg ? clock64() : 0;
              mbar_wait(&hfull[hs], hph);
              if (dbg) dbg_wait[1] += clock64() - t0; }
            tc_fence_after();
            uint64_t ad = make_smem_desc<SWZ>(smem_u32(sH + hs * hbytes), 8 * SWZ);
            uint32_t accum = cb == 0 ? 0u : 1u;
            for (int rh = 0; rh < pr; ++rh) {
              for (int pp = 0; pp < npair; ++pp) {
#pragma unroll
                for (int ms = 0; ms < MS; ++ms)
#pragma unroll
                  for (int kk = 0; kk < Cfg::kMmaPerTap; ++kk)
                    tc_mma<KIND>(d0 + ms * 2 * BN, ad + ((ms * 128 * SWZ + kk * 32) >> 4),
                                 bd + ((kk * 32) >> 4), idesc2, kk == 0 ? accum : 1u);
                accum = 1u;
                ad += (2 * SWZ) >> 4;
                bd += (2 * Cfg::kWBytes) >> 4;
              }
              if (ps & 1) {  // the row's last tap alone, into lo
#pragma unroll
                for (int ms = 0; ms < MS; ++ms)
#pragma unroll
                  for (int kk = 0; kk < Cfg::kMmaPerTap; ++kk)
                    tc_mma<KIND>(d0 + ms * 2 * BN, ad + ((ms * 128 * SWZ + kk * 32) >> 4),
                                 bd + ((kk * 32) >> 4), idesc, 1u);
                bd += Cfg::kWBytes >> 4;
              }
              ad += odd_skip + row_skip;
            }
            tc_commit(&hempty[hs]);
            if (++hs == 2) { hs = 0; hph ^= 1; }
          }
          tc_commit(&tfull[acc]);
        }
      } else {
      auto issue = [&](auto resident_c) {
        constexpr bool kRes = decltype(resident_c)::value;
        for (int local = 0; tile_at(local, &n_tile, &band, &img); ++local) {
          const int acc = local & (nacc - 1);
          const uint32_t use = static_cast<uint32_t>(local >> acc_shift);
          { const long long t0 = dbg ? clock64() : 0;
            mbar_wait(&tempty[acc], (use & 1) ^ 1);
            if (dbg) dbg_wait[2] += clock64() - t0; }
          tc_fence_after();
          const uint32_t d0 = tmem_base + acc * Cfg::kAccCols;
          uint64_t bd = wdesc0;  // resident: walks all (cb, tap) tiles in order
          for (int cb = 0; cb < cblocks; ++cb) {
            { const long long t0 = dbg ? clock64() : 0;
              mbar_wait(&hfull[hs], hph);
              if (dbg) dbg_wait[1] += clock64() - t0; }
            tc_fence_after();
            uint64_t ad = make_smem_desc<SWZ>(smem_u32(sH + hs * hbytes), 8 * SWZ);
            uint32_t accum = cb == 0 ? 0u : 1u;
            for (int rh = 0; rh < pr; ++rh) {
              for (int rw = 0; rw < ps; ++rw) {
                if constexpr (!kRes) {
                  const long long t0 = dbg ? clock64() : 0;
                  mbar_wait(&wfull[ws], wph);
                  if (dbg) dbg_wait[1] += clock64() - t0;
                  tc_fence_after();
                  bd = wdesc0 + static_cast<uint32_t>((ws * Cfg::kWBytes) >> 4);
                }
#pragma unroll
                for (int ms = 0; ms < MS; ++ms) {
#pragma unroll
                  for (int kk = 0; kk < Cfg::kMmaPerTap; ++kk) {
                    tc_mma<KIND>(d0 + ms * BN, ad + ((ms * 128 * SWZ + kk * 32) >> 4),
                                 bd + ((kk * 32) >> 4), idesc, kk == 0 ? accum : 1u);
                  }
                }
                accum = 1u;
                ad += SWZ >> 4;
                if constexpr (kRes) {
                  bd += Cfg::kWBytes >> 4;
                } else {
                  if (cl > 1) tc_commit_mc(&wempty[ws], cmask);  // release in every CTA
                  else tc_commit(&wempty[ws]);
                  if (++ws == WSTAGES) { ws = 0; wph ^= 1; }
                }
              }
              ad += row_skip;
            }
            tc_commit(&hempty[hs]);
            if (++hs == 2) { hs = 0; hph ^= 1; }
          }
          tc_commit(&tfull[acc]);
        }
      };
      if (p.resident)
        issue(std::true_type{});
      else
        issue(std::false_type{});
      }  // !kPair
    }
  } else if (warp >= 4) {
    // ------------------------------------------------- epilogue warps
    // Two groups of 4 warps; group g drains accumulator g (every other
    // tile). Warp w reads TMEM lane quadrant (w % 4): 32 virtual rows of
    // each sub-tile, all BN columns.
    const uint32_t q = warp & 3;
    const int grp = static_cast<int>(warp - 4) >> 2;
    const int gtid = static_cast<int>(threadIdx.x) - (kThreads - kEpiThreads) - grp * 128;
    uint8_t* stage = sStage + (warp - 4) * 4096;
    const bool coalesced =
        p.epi_mode == 0 &&
        ((KIND == MmaKind::kI8 || p.out_type != kBF16) ? (p.oc % 4) == 0 : (p.oc % 8) == 0);
    const epi::EpiProg prog = epi::make_prog(p.epi);
    const int fast = epi::classify_prog(p.epi);
    // Residual programs compile into the 128-B-block float instances only
    // (the stems / SW32 instances never carry a shortcut; keeping the extra
    // path out of them keeps their register allocation unchanged).
    constexpr bool kResTma = KIND != MmaKind::kI8 && SWZ == 128;
    // bias + residual add + relu (the ResNet block) too, on the float kinds
    // (residual read per row; oc % 32 == 0 keeps 32-column reads in the row)
    const bool tma_epi =
        p.tma_store && p.epi_mode == 0 && fast != epi::kProgGeneric &&
        (fast != epi::kProgBiasAddRelu || (kResTma && p.oc % 32 == 0));
    uint32_t chunk_cnt = 0;
    int local = 0;
    int staged_n_tile = -1;
    bool overflow = false;
    int n_tile, band, img;
    bool dummy = false;
    for (; tile_at(local, &n_tile, &band, &img, &dummy); ++local) {
      if ((local & 1) != grp) continue;
      const int acc = local & (nacc - 1);
      const uint32_t use = static_cast<uint32_t>(local >> acc_shift);
      uint32_t* bias_s = sBias + grp * BN;
      // The group's bias buffer only changes with the output-channel tile
      // (a global load + two barriers on the per-tile critical path).
      if (n_tile != staged_n_tile) {
        epi::named_bar_sync(1 + grp, 128);  // previous tile's readers are done
        epi::stage_bias(bias_s, p.epi.bias, n_tile * BN, BN, p.oc, gtid, 128);
        epi::named_bar_sync(1 + grp, 128);
        staged_n_tile = n_tile;
      }
      if (tma_epi && !dummy &&
          ((kResTma && fast == epi::kProgBiasAddRelu) || fast == epi::kProgBiasAddReluQ)) {
        // The residual rows are read right after the accumulator lands: pull
        // this lane's lines into L2 while the MMAs still run.
        const int es = fast == epi::kProgBiasAddReluQ ? 1 : p.out_type == kBF16 ? 2 : 4;
        for (int ms = 0; ms < MS; ++ms) {
          const int v = ms * 128 + static_cast<int>(q * 32 + lane);
          const int ohl = v / p.wp, ow = v - ohl * p.wp, oh = band * p.th + ohl;
          if (ohl < p.th && oh < p.oh && ow < p.ow) {
            const uint8_t* r = static_cast<const uint8_t*>(p.epi.residual) +
                               ((static_cast<int64_t>(img * p.oh + oh) * p.ow + ow) * p.oc +
                                n_tile * BN) * es;
            for (int b = 0; b < BN * es && n_tile * BN + b / es < p.oc; b += 128)
              prefetch_l2(r + b);
          }
        }
      }
      const long long tw0 = p.dbg ? clock64() : 0;
      mbar_wait(&tfull[acc], use & 1);
      const long long tw1 = p.dbg ? clock64() : 0;
      if (p.dbg) dbg_wait[3] += tw1 - tw0;
      tc_fence_after();
      if (dummy) {  // no tile for this CTA in its cluster's last group
        tc_fence_before();
        mbar_arrive(&tempty[acc]);
        continue;
      }
      if (kPair && !tma_epi) __trap();  // host guarantees the TMA-store program for kPair
      {
        if (tma_epi) {
          constexpr bool kInt = KIND == MmaKind::kI8;
          // The GROUP stages the whole tile's virtual rows for one 32-column
          // chunk (MS*128 rows, the row-per-lane writes of its 4 warps), then
          // one thread stores every output row of the band as a 4-D box
          // {32 ch, OW px} read from smem row ohl*wp: junk virtual rows are
          // simply never read, rows past OH are clipped by the map. (A store
          // per warp would need negative box coordinates for rows that
          // straddle an output-row boundary; TMA stores reject those.)
          // Host guarantees: MS*128 rows x 32*ES bytes <= 16 KB and
          // wp*32*ES a multiple of 128 B (TMA source alignment); the
          // swizzle is absolute-address based, so any such row start works.
          epi::QParams qp;  // the Q programs (int8 graphs)
          qp.mult = p.epi.rq_mult;
          qp.shift = p.epi.rq_shift;
          qp.res_scale = p.epi.res_scale;
          auto run = [&](auto prog_c, auto es_c) {
            constexpr int kProg = decltype(prog_c)::value, kES = decltype(es_c)::value;
            constexpr uint32_t kRowB = 32 * kES;
            const uint32_t gbytes = static_cast<uint32_t>(p.stage_bytes) / 2;
            const uint32_t cbytes = MS * 128 * kRowB;
            const uint32_t gbase = smem_u32(sStage) + static_cast<uint32_t>(grp) * gbytes;
            const bool two = gbytes >= 2 * cbytes;  // chunk ring of 2: write one while one drains
            const bool issuer = q == 0 && lane == 0;
            const int valid = p.oc - n_tile * BN;
#pragma unroll 1
            for (int c0 = 0; c0 < BN && c0 < valid; c0 += epi::kChunk) {
              const uint32_t gbuf = gbase + (two ? (chunk_cnt & 1) * cbytes : 0);
              ++chunk_cnt;
              if (issuer) {  // the slot's previous stores have finished reading it
                if (two) bulk_wait_read<1>(); else bulk_wait_read<0>();
              }
              epi::named_bar_sync(1 + grp, 128);
#pragma unroll 1
              for (int ms = 0; ms < MS; ++ms) {
                const uint8_t* rrow = nullptr;
                if constexpr (kProg == epi::kProgBiasAddRelu || kProg == epi::kProgBiasAddReluQ) {
                  // virtual row -> output pixel (junk rows: no residual, not stored)
                  const int v = ms * 128 + static_cast<int>(q * 32 + lane);
                  const int ohl = v / p.wp, ow = v - ohl * p.wp, oh = band * p.th + ohl;
                  if (ohl < p.th && oh < p.oh && ow < p.ow)
                    rrow = static_cast<const uint8_t*>(p.epi.residual) +
                           ((static_cast<int64_t>(img * p.oh + oh) * p.ow + ow) * p.oc +
                            n_tile * BN + c0) * kES;
                }
                const uint32_t box =
                    gbuf + static_cast<uint32_t>(ms * 128 + static_cast<int>(q) * 32) * kRowB;
                if constexpr (kPair) {
                  // output row v = lo(v) + hi(v + 1): hi of the next lane by
                  // shuffle; lane 31's row needs the next warp's lane 0 and is
                  // finished after the barrier below from the exchange slots.
                  const uint32_t ta =
                      tmem_base + ((q * 32) << 16) + acc * Cfg::kAccCols + ms * 2 * BN + c0;
                  uint32_t lo[epi::kChunk], hi[epi::kChunk];
                  tmem_ld32(ta, lo);
                  tmem_ld32(ta + BN, hi);
                  tmem_ld_wait();
                  float* xs = sXchg + ((grp * MS + ms) * 4 + q) * 64;  // [hi of lane 0 | lo of lane 31]
                  if (lane == 0 || lane == 31) {
                    float4* x4 = reinterpret_cast<float4*>(xs + (lane == 0 ? 0 : 32));
                    const uint32_t* src = lane == 0 ? hi : lo;
#pragma unroll
                    for (int j = 0; j < epi::kChunk / 4; ++j)
                      x4[j] = make_float4(__uint_as_float(src[4 * j]), __uint_as_float(src[4 * j + 1]),
                                          __uint_as_float(src[4 * j + 2]),
                                          __uint_as_float(src[4 * j + 3]));
                  }
#pragma unroll
                  for (int j = 0; j < epi::kChunk; ++j) {
                    const float hn = __shfl_down_sync(0xffffffffu, __uint_as_float(hi[j]), 1);
                    lo[j] = __float_as_uint(__fadd_rn(__uint_as_float(lo[j]), hn));
                  }
                  epi::epi_acc_to_box<kProg, kES, kInt>(lo, static_cast<int>(lane), bias_s + c0,
                                                        box, &overflow, rrow);
                } else {
                  epi::epi_block_box<kProg, kES, kInt>(
                      tmem_base + ((q * 32) << 16) + acc * Cfg::kAccCols + ms * BN + c0,
                      static_cast<int>(lane), bias_s + c0, box, &overflow, rrow, qp);
                }
              }
              if constexpr (kPair) {
                epi::named_bar_sync(1 + grp, 128);  // exchange slots written
                // the warp's last row, one column per lane
#pragma unroll 1
                for (int ms = 0; ms < MS; ++ms) {
                  const float* mine = sXchg + ((grp * MS + ms) * 4 + q) * 64 + 32;
                  const float* nx = q < 3 ? sXchg + ((grp * MS + ms) * 4 + q + 1) * 64
                                    : ms + 1 < MS ? sXchg + ((grp * MS + ms + 1) * 4) * 64
                                                  : nullptr;  // past the tile: a junk row
                  const uint8_t* rrow = nullptr;
                  if constexpr (kProg == epi::kProgBiasAddRelu) {
                    const int v = ms * 128 + static_cast<int>(q * 32 + 31);
                    const int ohl = v / p.wp, ow = v - ohl * p.wp, oh = band * p.th + ohl;
                    if (ohl < p.th && oh < p.oh && ow < p.ow)
                      rrow = static_cast<const uint8_t*>(p.epi.residual) +
                             ((static_cast<int64_t>(img * p.oh + oh) * p.ow + ow) * p.oc +
                              n_tile * BN + c0) * kES;
                  }
                  epi::row_col_to_box<kProg, kES>(
                      mine, nx, bias_s + c0, rrow,
                      gbuf + static_cast<uint32_t>(ms * 128 + static_cast<int>(q) * 32) * kRowB,
                      31, static_cast<int>(lane));
                }
              }
              fence_proxy_async_smem();
              epi::named_bar_sync(1 + grp, 128);
              if (issuer) {
                for (int ohl = 0; ohl < p.th && band * p.th + ohl < p.oh; ++ohl)
                  tma_store_4d(&tm_y, gbuf + static_cast<uint32_t>(ohl * p.wp) * kRowB,
                               n_tile * BN + c0, 0, band * p.th + ohl, img);
                bulk_commit();
              }
            }
          };
          using P0 = std::integral_constant<int, epi::kProgNone>;
          using P1 = std::integral_constant<int, epi::kProgBias>;
          using P2 = std::integral_constant<int, epi::kProgBiasRelu>;
          using P3 = std::integral_constant<int, epi::kProgBiasAddRelu>;
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
            else if (fast == epi::kProgBiasRelu || !kResTma) run(P2{}, E2{});
            else if constexpr (kResTma) run(P3{}, E2{});
          } else {
            if (fast == epi::kProgNone) run(P0{}, E4{});
            else if (fast == epi::kProgBias) run(P1{}, E4{});
            else if (fast == epi::kProgBiasRelu || !kResTma) run(P2{}, E4{});
            else if constexpr (kResTma) run(P3{}, E4{});
          }
          tc_fence_before();
          mbar_arrive(&tempty[acc]);
          if (p.dbg) dbg_wait[4] += clock64() - tw1;
          continue;
        }
      }
#pragma unroll 1
      for (int ms = 0; ms < MS; ++ms) {
        const int vbase = ms * 128 + static_cast<int>(q * 32);
        // Virtual row -> output row (or -1 for the junk columns ow >= OW
        // and rows past the band).
        int my_row = -1;  // this lane's output row, -1 for junk virtual rows
        {
          const int v = vbase + static_cast<int>(lane);
          const int ohl = v / p.wp;
          const int ow = v - ohl * p.wp;
          const int oh = band * p.th + ohl;
          if (ohl < p.th && oh < p.oh && ow < p.ow) my_row = (img * p.oh + oh) * p.ow + ow;
        }
#pragma unroll 1
        for (int c0 = 0; c0 < BN && p.epi_mode != 2; c0 += epi::kChunk) {  // 2: diagnostic
          const uint32_t taddr =
              tmem_base + ((q * 32) << 16) + acc * Cfg::kAccCols + ms * BN + c0;
          const int col0 = n_tile * BN + c0;
          if (coalesced) {
            if (col0 < p.oc)
              epi::epi_block<KIND == MmaKind::kI8>(p, prog, fast, taddr, col0, lane, my_row,
                                                   bias_s + c0, stage, &overflow);
          } else {
            uint32_t vv[epi::kChunk];
            tmem_ld32(taddr, vv);
            const bool active = my_row >= 0 && col0 < p.oc;
            const int ncols = min(epi::kChunk, p.oc - col0);
            epi::epi_row_chunk<KIND == MmaKind::kI8>(p, prog, my_row, col0, ncols, active,
                                                     bias_s + c0, vv, &overflow);
          }
        }
      }
      tc_fence_before();
      mbar_arrive(&tempty[acc]);
      if (p.dbg) dbg_wait[4] += clock64() - tw1;
    }
    if (lane == 0) bulk_wait_all();  // TMA stores done before smem goes away
    if (overflow && p.err) atomicOr(p.err, 1);
  }

  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  // Peers multicast into this CTA's smem and arrive on its barriers until
  // they finish: nobody leaves before the whole cluster is done.
  if (cl > 1) cluster_sync();
  if (warp == 2) tmem_dealloc<Cfg::kTmemCols>(tmem_base);
  if (p.dbg) {
    const bool rep = (warp <= 1 && lane == 0) || threadIdx.x == kThreads - kEpiThreads;
    if (rep)
      for (int i = 0; i < 8; ++i)
        if (dbg_wait[i])
          atomicAdd(&p.dbg[i < 5 ? i : i + 3], static_cast<unsigned long long>(dbg_wait[i]));
    if (threadIdx.x == 0) {
      atomicAdd(&p.dbg[5], static_cast<unsigned long long>(clock64() - t_start));
      atomicAdd(&p.dbg[6], static_cast<unsigned long long>((num_tiles - blockIdx.x + gridDim.x - 1) / gridDim.x));
    }
  }
}

}  // namespace

template <MmaKind KIND, int BN, int MS, int SWZ, int WSTAGES, bool kPair>
int launch_conv_halo(const CUtensorMap& tm_x, const CUtensorMap& tm_w,
                     const CUtensorMap& tm_y, const ConvHaloParams& p, int grid,
                     cudaStream_t stream) {
  using Cfg = HaloCfg<BN, MS, SWZ, WSTAGES, kPair>;
  const int smem = 1024 + 2 * halo_bytes_aligned(p.halo_px, SWZ) +
                   p.w_slots * Cfg::kWBytes + p.stage_bytes + 256 + 2 * BN * 4 +
                   (kPair ? 2 * MS * 4 * 64 * 4 : 0);
  if (kPair && (!p.resident || p.s < 2 || !p.tma_store)) return cudaErrorInvalidValue;
  if (p.stage_bytes < 8 * 4096 || p.stage_bytes % 2048) return cudaErrorInvalidValue;
  if (!p.resident && p.w_slots != WSTAGES) return cudaErrorInvalidValue;
  if (smem > 227 * 1024) return cudaErrorInvalidConfiguration;
  auto kfn = conv_halo_kernel<KIND, BN, MS, SWZ, WSTAGES, kPair>;
  cudaError_t e = cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) return e;
  e = launch_pdl_cluster(kfn, dim3(grid), dim3(kThreads), smem, stream,
                         p.cl > 1 && !p.resident ? p.cl : 1, tm_x, tm_w, tm_y, p);
  if (e != cudaSuccess) return e;
  return cudaGetLastError();
}

// Returns the dynamic smem a configuration needs (host-side planning).
int conv_halo_smem_bytes(int bn, int swz, int w_slots, int halo_px, int stage_bytes, int ms,
                         bool pair) {
  return 1024 + 2 * halo_bytes_aligned(halo_px, swz) + w_slots * bn * swz + stage_bytes + 256 +
         2 * bn * 4 + (pair ? 2 * ms * 4 * 64 * 4 : 0);
}

#define TEC_HALO(KIND, BN, MS, SWZ, WS)                                        \
  template int launch_conv_halo<KIND, BN, MS, SWZ, WS, false>(                \
      const CUtensorMap&, const CUtensorMap&, const CUtensorMap&,           \
      const ConvHaloParams&, int, cudaStream_t);
#define TEC_HALO_PAIR(KIND, BN, MS, SWZ, WS)                                   \
  template int launch_conv_halo<KIND, BN, MS, SWZ, WS, true>(                 \
      const CUtensorMap&, const CUtensorMap&, const CUtensorMap&,           \
      const ConvHaloParams&, int, cudaStream_t);

TEC_HALO(MmaKind::kF16, 64, 1, 128, 6)
TEC_HALO(MmaKind::kF16, 64, 2, 128, 6)
TEC_HALO(MmaKind::kF16, 64, 4, 128, 4)
TEC_HALO(MmaKind::kF16, 128, 1, 128, 6)
TEC_HALO(MmaKind::kF16, 128, 2, 128, 4)
TEC_HALO(MmaKind::kF16, 256, 1, 128, 4)
TEC_HALO(MmaKind::kF16, 64, 2, 32, 8)
TEC_HALO(MmaKind::kF16, 64, 4, 32, 8)
TEC_HALO(MmaKind::kI8, 64, 1, 128, 6)
TEC_HALO(MmaKind::kI8, 128, 1, 128, 6)
TEC_HALO(MmaKind::kI8, 64, 1, 32, 8)
TEC_HALO(MmaKind::kI8, 64, 1, 64, 6)
TEC_HALO(MmaKind::kI8, 64, 2, 128, 6)
TEC_HALO(MmaKind::kI8, 64, 4, 128, 4)
TEC_HALO(MmaKind::kI8, 128, 2, 128, 4)
TEC_HALO(MmaKind::kI8, 256, 1, 128, 4)
TEC_HALO(MmaKind::kI8, 64, 2, 32, 8)
TEC_HALO(MmaKind::kI8, 64, 4, 32, 8)
TEC_HALO(MmaKind::kI8, 64, 2, 64, 6)
TEC_HALO(MmaKind::kI8, 64, 4, 64, 6)

TEC_HALO_PAIR(MmaKind::kF16, 64, 1, 128, 6)
TEC_HALO_PAIR(MmaKind::kF16, 64, 2, 128, 6)
TEC_HALO_PAIR(MmaKind::kF16, 64, 1, 32, 8)
TEC_HALO_PAIR(MmaKind::kF16, 64, 2, 32, 8)

#undef TEC_HALO
#undef TEC_HALO_PAIR

}  // namespace tec_sm100
