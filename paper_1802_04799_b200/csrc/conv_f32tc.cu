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
constexpr int kMaxRows = 8;    // row-ring slots (ConvGemmParams::rows)

template <int BN, int SWZ, int STAGES, bool INTER, bool RES = false, bool HALO = false,
          bool PAIR = false>
struct F32tcCfg {
  static constexpr int kAPlanes = INTER ? 1 : 3;  // A boxes per k-iteration
  static constexpr int kA = kBM * SWZ;            // one A box
  // B: three boxes of BN rows (one per plane), or -- interleaved -- one 3-D
  // box [plane][BN rows][16 ch] with the 32-B swizzle. Either way the planes
  // are consecutive row blocks: [B_h; B_m; B_l] is one N-concatenated operand.
  static constexpr int kBSW = INTER ? 32 : SWZ;      // B row bytes / swizzle
  // bytes per B plane (a CTA of a pair holds half of the tile's rows)
  static constexpr int kBPlane = (PAIR ? BN / 2 : BN) * kBSW;
  static constexpr int kBBoxes = INTER ? 1 : 3;
  static constexpr int kBBox = INTER ? 3 * kBPlane : kBPlane;
  static constexpr int kBStage = 3 * kBPlane;       // B bytes per k-iteration
  // RES: every k-iteration's B tile of the CTA's output-channel tile stays
  // in shared memory (loaded once per CTA, p.res_bytes); the ring carries A only
  // HALO: A lives in the halo buffers (runtime-sized), the ring carries B
  static constexpr int kStage = (HALO ? 0 : kAPlanes * kA) + (RES ? 0 : kBStage);
  static constexpr int kKSteps = INTER ? 1 : SWZ / 32;  // K16 steps per plane per stage
  // GRP (BN = 64): the products sharing an operand run as ONE MMA on the
  // N-concatenated planes -- A_h x [B_h|B_m|B_l] (N=192) into the chunk
  // accumulator X = [hh | hm | hl]; A_m x [B_h|B_m] (N=128) into X[64:192]
  // (mh onto hm, mm onto hl: all cross terms) and A_l x B_h (N=64) into
  // X[64:128] -- 3 MMAs instead of 6 N=64 ones, whose rate is bound by
  // re-reading A from shared memory (54 vs 32 cycles each,
  // tools/microbench/RESULTS.md). Everything folds per chunk, so there is no
  // tile accumulator and no tile-boundary wait for the epilogue: TMEM = X
  // ring 2 x 192. (Measured before: with the cross terms of A_m / A_l in a
  // single-buffered tile accumulator the MMA waited for the epilogue at every
  // tile start -- 17 % of C1; a 4-MMA form with a double-buffered one was
  // slower still, C1 197 vs 169 us.)
  // Otherwise (BN = 128): six N=128 MMAs; chunk ring S 2 x BN (hh) + tile
  // accumulators T 2 x BN (cross terms over the whole tile).
  static constexpr bool kGrp = BN == 64;
  static constexpr bool kHasY = !kGrp;
  static constexpr int kXCols = kGrp ? 3 * BN : BN;     // chunk accumulator width
  static constexpr int kYCols = kGrp ? 0 : BN;          // tile accumulator width
  static constexpr int kYBufs = kGrp ? 1 : 2;
  static constexpr int kYBase = 2 * kXCols;
  static constexpr uint32_t kTmemCols = 2 * kXCols + kYBufs * kYCols <= 256 ? 256 : 512;
  // + res_bytes (RES) + hbuf x kAPlanes x halo_bytes (HALO)
  static constexpr int kSmem = 1024 + STAGES * kStage + 8 * 4096 + 512 + BN * 4;
  static_assert(kSmem <= 227 * 1024, "shared memory budget");
  static_assert(2 * kXCols + kYBufs * kYCols <= 512, "TMEM budget");
  static_assert(!INTER || SWZ == 128, "interleaved planes live in one 128-B row");
  static_assert(!PAIR || (BN == 128 && !INTER && !RES && !HALO), "CTA pairs: the im2col BN=128 path");
};

// The work items of one CTA: (output tile mn, k-iterations [kb, ke), its
// segment index seg of nseg). Modes: items strided over the grid (split-K
// splits of kps k-iterations, splits = 1 without), one contiguous range of
// items (the row ring), or stream-K ranges of the flattened (tile, k) space.
struct WorkIter {
  int mode;  // 0 strided, 1 contiguous, 2 stream-K
  int item, hi, step, splits, kps, k_iters, G, c;
  long long pos, end, W;
  // the CTA owning work position x: max c with floor(c W / G) <= x
  __device__ __forceinline__ int owner(long long x) const {
    return static_cast<int>(((x + 1) * G + W - 1) / W) - 1;
  }
  __device__ __forceinline__ bool next(int& it, int& mn, int& kb, int& ke, int& seg, int& nseg) {
    if (mode < 2) {
      if (item >= hi) return false;
      it = item;
      mn = item / splits;
      seg = item - mn * splits;
      nseg = splits;
      kb = seg * kps;
      ke = min(k_iters, kb + kps);
      item += step;
      return true;
    }
    if (pos >= end) return false;
    mn = static_cast<int>(pos / k_iters);
    const long long t0 = static_cast<long long>(mn) * k_iters;
    const long long se = min(end, t0 + k_iters);
    kb = static_cast<int>(pos - t0);
    ke = static_cast<int>(se - t0);
    const int o0 = owner(t0);
    seg = c - o0;
    nseg = owner(t0 + k_iters - 1) - o0 + 1;
    it = mn;
    pos = se;
    return true;
  }
};

// mbar_wait that adds its waiting cycles to *acc when profiling (p.dbg)
__device__ __forceinline__ void twait(uint64_t* bar, uint32_t parity, bool prof, long long* acc) {
  if (!prof) {
    mbar_wait(bar, parity);
    return;
  }
  const long long t0 = clock64();
  mbar_wait(bar, parity);
  *acc += clock64() - t0;
}

template <int BN, int SWZ, int STAGES, bool INTER, bool RES, bool HALO, int PROG, bool PAIR>
__global__ void __launch_bounds__(kThreads, 1)
    conv_f32tc_kernel(const __grid_constant__ CUtensorMap tm_a,
                      const __grid_constant__ CUtensorMap tm_b,
                      const __grid_constant__ CUtensorMap tm_y, const ConvGemmParams p) {
  using Cfg = F32tcCfg<BN, SWZ, STAGES, INTER, RES, HALO, PAIR>;
  constexpr int kCB = SWZ / 2;  // bf16 channels per box row
  constexpr int HB = BN / 2;    // columns per epilogue warp
  constexpr int kBSW = Cfg::kBSW;
  // byte offset of A plane q inside a stage: its own box, or its K16 slice
  // of the interleaved row
  constexpr int kPlaneA = INTER ? 32 : Cfg::kA;
  constexpr int kPlaneB = Cfg::kBPlane;
  // shared-memory descriptors without their start address (make_smem_desc)
  constexpr uint64_t kADescHi = (1ull << 16) | (static_cast<uint64_t>((8 * SWZ) >> 4) << 32) |
                                (1ull << 46) | (static_cast<uint64_t>(SWZ == 128 ? 2 : SWZ == 64 ? 4 : 6) << 61);
  constexpr uint64_t kBDescHi = (1ull << 16) | (static_cast<uint64_t>((8 * kBSW) >> 4) << 32) |
                                (1ull << 46) | (static_cast<uint64_t>(kBSW == 128 ? 2 : kBSW == 64 ? 4 : 6) << 61);
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sHalo = smem;  // HALO: hbuf x kAPlanes halo buffers of halo_bytes
  uint8_t* sRing = sHalo + (HALO ? p.hbuf * Cfg::kAPlanes * p.halo_bytes : 0);
  uint8_t* sRes = sRing + STAGES * Cfg::kStage;  // RES: resident B, k_iters x kBStage
  uint8_t* sStage = sRes + (RES ? p.res_bytes : 0);  // 8 warps x 4 KB
  uint64_t* full = reinterpret_cast<uint64_t*>(sStage + 8 * 4096);
  uint64_t* empty = full + STAGES;
  uint64_t* sfull = empty + STAGES;
  uint64_t* sempty = sfull + 2;
  uint64_t* tfull = sempty + 2;
  uint64_t* tempty = tfull + 2;
  uint64_t* wfull = tempty + 2;  // RES: the resident B tiles landed
  uint64_t* hfull = wfull + 1;   // HALO: halo buffer (row ring: row slot) landed / free
  uint64_t* hempty = hfull + kMaxRows;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(hempty + kMaxRows);
  int* s_last = reinterpret_cast<int*>(tmem_slot + 1);
  uint32_t* sBias = reinterpret_cast<uint32_t*>(reinterpret_cast<uint8_t*>(full) + 512);

  const uint32_t warp = warp_id();
  const uint32_t lane = threadIdx.x & 31;
  const int splits = p.splits > 1 ? p.splits : 1;
  // CTA pair (PAIR, cluster of 2, cta_group::2 -- as conv_tc.cu): the pair
  // runs one MMA stream (the leader's) over a 256-row M tile, each CTA
  // loading its own A rows and half of the weight rows; work units are
  // (M-tile pair, N tile) and own_mn() maps a unit to this CTA's tile
  const uint32_t rank = PAIR ? cluster_ctarank() : 0u;
  const int m_units = PAIR ? (p.m_tiles + 1) / 2 : p.m_tiles;
  auto own_mn = [&](int mnu) -> int {
    if constexpr (!PAIR) return mnu;
    const int mp = mnu / p.n_tiles;
    return (2 * mp + static_cast<int>(rank)) * p.n_tiles + (mnu - mp * p.n_tiles);
  };
  const int num_items = m_units * p.n_tiles * splits;
  // TEC_SM100_PROFILE: per-role waiting cycles, summed over CTAs into p.dbg --
  // [0] producer A (halo/ring) free, [1] producer B ring free, [2] MMA
  // tile accumulator free, [3] MMA chunk accumulator free, [4] MMA operands
  // landed, [5] epilogue chunk ready, [6] epilogue tile ready, [7] epilogue
  // busy, [8] CTA cycles, [9] items
  const bool prof = p.dbg != nullptr;
  long long dw[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  const long long t_start = prof ? clock64() : 0;
  const int k_iters = p.r * p.s * p.cblocks;
  const int kps = splits > 1 ? p.kps : k_iters;  // k-iterations per split
  const int chunk = p.chunk_iters;               // k-iterations per hh chunk
  const int cpp = p.cp;                          // channels per plane
  const int pix = INTER ? 64 : 3 * cpp;          // packed channels per pixel
  // work items of this CTA: strided over the grid, or (row ring) one
  // contiguous range, so consecutive items are consecutive output rows
  const bool ring = HALO && p.rows > 0;
  const int cta = PAIR ? static_cast<int>(blockIdx.x >> 1) : static_cast<int>(blockIdx.x);
  const int ctas = PAIR ? static_cast<int>(gridDim.x >> 1) : static_cast<int>(gridDim.x);
  const int it_lo = ring ? static_cast<int>(static_cast<int64_t>(num_items) * blockIdx.x / gridDim.x)
                         : cta;
  const int it_hi = ring ? static_cast<int>(static_cast<int64_t>(num_items) * (blockIdx.x + 1) / gridDim.x)
                         : num_items;
  const int it_step = ring ? 1 : ctas;
  const bool sk = !HALO && p.stream_k;
  auto make_iter = [&]() {
    WorkIter w;
    w.mode = sk ? 2 : (ring ? 1 : 0);
    w.item = it_lo;
    w.hi = it_hi;
    w.step = it_step;
    w.splits = sk ? 1 : splits;
    w.kps = kps;
    w.k_iters = k_iters;
    w.G = ctas;
    w.c = cta;
    w.W = static_cast<long long>(m_units) * p.n_tiles * k_iters;
    w.pos = w.W * w.c / w.G;
    w.end = w.W * (w.c + 1) / w.G;
    return w;
  };

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
      mbar_init(&sempty[i], PAIR ? 512 : 256);  // a pair: both CTAs' epilogues
      mbar_init(&tfull[i], 1);
      mbar_init(&tempty[i], PAIR ? 512 : 256);
    }
    mbar_init(wfull, 1);
    for (int i = 0; i < kMaxRows; ++i) {
      mbar_init(&hfull[i], 1);
      mbar_init(&hempty[i], 1);
    }
    fence_barrier_init();
  }
  if (warp == 2) {
    if constexpr (PAIR) tmem_alloc_pair<Cfg::kTmemCols>(tmem_slot);
    else tmem_alloc<Cfg::kTmemCols>(tmem_slot);
  }
  tc_fence_before();
  if constexpr (PAIR) cluster_sync();  // both CTAs' barriers initialised
  else __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  pdl_launch_dependents();

  if (warp == 0 || (warp == 3 && p.producers == 2)) {
    // ------------------------------------------------ TMA producers
    // warp 0 issues the activation boxes (and arms the stage's transaction
    // count); with two producers warp 3 issues the weight boxes of the same
    // stage, so the two TMA streams are not serialised behind one thread
    const bool issue_a = warp == 0;
    const bool issue_b = warp == 3 || p.producers != 2;
    if (elect_one()) {
      const int sc = p.s * p.cblocks;
      if (RES && issue_b && static_cast<int>(blockIdx.x) < num_items) {
        // the CTA's output-channel tile is fixed (grid % n_tiles == 0, no
        // split): its B tiles for all k-iterations, once -- parameters, so
        // before the wait on the previous layer
        const int n_tile = static_cast<int>(blockIdx.x) % p.n_tiles;
        mbar_arrive_expect_tx(wfull, static_cast<uint32_t>(k_iters * Cfg::kBStage));
        int r = 0, s = 0, cb = 0;
        for (int k = 0; k < k_iters; ++k) {
          uint8_t* bb = sRes + k * Cfg::kBStage;
          if constexpr (INTER) {
            tma_load_3d(bb, &tm_b, wfull, 0, n_tile * BN, 3 * (r * p.s + s));
          } else {
            const int wcol = (r * p.s + s) * pix + cb * kCB;
#pragma unroll
            for (int pl = 0; pl < 3; ++pl)
              tma_load_2d(bb + pl * kPlaneB, &tm_b, wfull, wcol + pl * cpp, n_tile * BN);
          }
          if (++cb == p.cblocks) {
            cb = 0;
            if (++s == p.s) { s = 0; ++r; }
          }
        }
      }
      pdl_wait();
      int stage = 0;
      uint32_t phase = 0;
      const int ohw = p.oh * p.ow;
      if constexpr (HALO) {
        // per tile and channel block: ONE halo box per plane (the A thread),
        // then one weight stage per filter tap (the B thread)
        int hb = 0;
        uint32_t hphase = 0;
        // row ring: next input row (as v = ih + ph) to load, per-slot fill
        // parity / ever-filled bits
        int ring_img = -1, ring_v = 0;
        uint32_t fillpar = 0, filled = 0;
        for (int item = it_lo; item < it_hi; item += it_step) {
          const int m_tile = item / p.n_tiles;
          const int n_tile = item - m_tile * p.n_tiles;
          const int img = m_tile / p.bands;
          const int oh0 = (m_tile - img * p.bands) * p.th;
          if (ring && issue_a) {
            if (img != ring_img) {
              ring_img = img;
              ring_v = oh0;
            }
            for (; ring_v < oh0 + p.r; ++ring_v) {
              const int slot = ring_v % p.rows;
              const uint32_t bit = 1u << slot;
              if (filled & bit)  // the MMAs of the last reader of this slot have landed
                twait(&hempty[slot], ((fillpar & bit) ? 0u : 1u), prof, &dw[0]);
              filled |= bit;
              fillpar ^= bit;
              mbar_arrive_expect_tx(&hfull[slot], static_cast<uint32_t>(p.halo_box_bytes));
              tma_load_4d(sHalo + slot * p.halo_bytes, &tm_a, &hfull[slot], 0, -p.pw,
                          ring_v - p.ph, img);
            }
          }
          for (int cb = 0; cb < p.cblocks; ++cb) {
            if (issue_a && !ring) {
              twait(&hempty[hb], hphase ^ 1, prof, &dw[0]);
              mbar_arrive_expect_tx(&hfull[hb],
                                    static_cast<uint32_t>(Cfg::kAPlanes * p.halo_box_bytes));
#pragma unroll
              for (int pl = 0; pl < Cfg::kAPlanes; ++pl)
                tma_load_4d(sHalo + (hb * Cfg::kAPlanes + pl) * p.halo_bytes, &tm_a, &hfull[hb],
                            pl * cpp + cb * kCB, -p.pw, oh0 - p.ph, img);
              if (++hb == p.hbuf) {
                hb = 0;
                hphase ^= 1;
              }
            }
            if (issue_b && !RES) {
              for (int r = 0; r < p.r; ++r)
                for (int s = 0; s < p.s; ++s) {
                  twait(&empty[stage], phase ^ 1, prof, &dw[1]);
                  mbar_arrive_expect_tx(&full[stage], Cfg::kStage);
                  uint8_t* bbase = sRing + stage * Cfg::kStage;
                  if constexpr (INTER) {
                    tma_load_3d(bbase, &tm_b, &full[stage], 0, n_tile * BN, 3 * (r * p.s + s));
                  } else {
                    const int wcol = (r * p.s + s) * pix + cb * kCB;
#pragma unroll
                    for (int pl = 0; pl < 3; ++pl)
                      tma_load_2d(bbase + pl * kPlaneB, &tm_b, &full[stage], wcol + pl * cpp,
                                  n_tile * BN);
                  }
                  if (++stage == STAGES) {
                    stage = 0;
                    phase ^= 1;
                  }
                }
            }
          }
        }
      } else {
      WorkIter wi = make_iter();
      int item, mnu, kb, ke, seg, nseg;
      // a pair's loads complete on the leader's full barrier
      const uint32_t full_l = PAIR ? mapa_u32(smem_u32(full), 0) : 0u;
      while (wi.next(item, mnu, kb, ke, seg, nseg)) {
        const int mn = own_mn(mnu);
        const int m_tile = mn / p.n_tiles;
        const int n_tile = mn - m_tile * p.n_tiles;
        // a pair's phantom tile (odd M-tile count) reads its partner's rows
        const int m0 = (PAIR ? min(m_tile, p.m_tiles - 1) : m_tile) * kBM;
        const int img = m0 / ohw;
        const int rem = m0 - img * ohw;
        const int oh = rem / p.ow;
        const int ow = rem - oh * p.ow;
        const int w0 = ow * p.sw - p.pw;
        const int h0 = oh * p.sh - p.ph;
        int r = kb / sc, rem_k = kb - r * sc;
        int s = rem_k / p.cblocks, cb = rem_k - s * p.cblocks;
        for (int k = kb; k < ke; ++k) {
          twait(&empty[stage], phase ^ 1, prof, &dw[0]);
          if (issue_a && (!PAIR || rank == 0))
            mbar_arrive_expect_tx(&full[stage], PAIR ? 2 * Cfg::kStage : Cfg::kStage);
          uint8_t* base = sRing + stage * Cfg::kStage;
          uint8_t* bbase = base + Cfg::kAPlanes * Cfg::kA;
#pragma unroll
          for (int pl = 0; pl < Cfg::kAPlanes; ++pl)
            if (issue_a) {
              if constexpr (PAIR)
                tma_load_im2col_4d_pair(base + pl * Cfg::kA, &tm_a, full_l + 8 * stage,
                                        pl * cpp + cb * kCB, w0, h0, img,
                                        static_cast<uint16_t>(s), static_cast<uint16_t>(r));
              else
                tma_load_im2col_4d(base + pl * Cfg::kA, &tm_a, &full[stage], pl * cpp + cb * kCB,
                                   w0, h0, img, static_cast<uint16_t>(s), static_cast<uint16_t>(r));
            }
          if (issue_b && !RES) {
            if constexpr (INTER) {
              tma_load_3d(bbase, &tm_b, &full[stage], 0, n_tile * BN, 3 * (r * p.s + s));
            } else {
              const int wcol = (r * p.s + s) * pix + cb * kCB;
#pragma unroll
              for (int pl = 0; pl < 3; ++pl) {
                if constexpr (PAIR)  // this CTA's half of the tile's weight rows
                  tma_load_2d_pair(bbase + pl * kPlaneB, &tm_b, full_l + 8 * stage, wcol + pl * cpp,
                                   n_tile * BN + static_cast<int>(rank) * (BN / 2));
                else
                  tma_load_2d(bbase + pl * kPlaneB, &tm_b, &full[stage], wcol + pl * cpp,
                              n_tile * BN);
              }
            }
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
    }
  } else if (warp == 1 && (!PAIR || rank == 0)) {
    // ------------------------------------------ single-thread MMA issuer
    if (elect_one()) {
      constexpr uint32_t idesc = make_idesc<MmaKind::kF16>(PAIR ? 2 * kBM : kBM, BN);
      constexpr uint32_t idesc3 = make_idesc<MmaKind::kF16>(kBM, 3 * BN);
      constexpr uint32_t idesc2 = make_idesc<MmaKind::kF16>(kBM, 2 * BN);
      int stage = 0;
      uint32_t phase = 0;
      int g = 0;  // hh chunks issued so far (S ring position)
      int local = 0;
      if (RES) {
        mbar_wait(wfull, 0);
        tc_fence_after();
      }
      int hb = 0;
      uint32_t hphase = 0;
      int ring_img = -1, ring_v = 0;
      uint32_t fillpar = 0;
      // the fast ring path (C1: interleaved planes, resident weights, GRP):
      // parameters in registers (the asm "memory" clobbers would otherwise
      // reload them from the constant bank every tap) and descriptors
      // advanced by adding to their 16-byte address field
      constexpr bool kFast = HALO && RES && INTER && Cfg::kGrp;
      const int R = p.r, S = p.s, nrows = p.rows > 0 ? p.rows : 1, hbytes = p.halo_bytes;
      const int ntl = p.n_tiles, bands = p.bands;
      const uint64_t adesc0 = make_smem_desc<SWZ>(smem_u32(sHalo), 8 * SWZ);
      const uint64_t hstep = static_cast<uint64_t>(hbytes >> 4);  // one row slot, in 16-B units
      int f_img = 0, f_oh = 0, f_s0 = 0, ring_slot = 0;
      // the fast path's tile-end commits (chunk ready, ring row free), issued
      // after the NEXT tile's first tap so the tensor pipe never runs dry at
      // a tile boundary (only within an image: the next tile's rows are then
      // already resident)
      int pend_sb = -1, pend_s0 = 0;
      bool f_prepared = false;  // the next tile's waits already done
      const uint64_t bdesc0 = make_smem_desc<kBSW>(smem_u32(sRes), 8 * kBSW);
      WorkIter wi = make_iter();
      int item, w_mn, w_kb, w_ke, w_seg, w_nseg;
      for (; wi.next(item, w_mn, w_kb, w_ke, w_seg, w_nseg); ++local) {
        const int tb = local % Cfg::kYBufs;
        const int tuse = local / Cfg::kYBufs;
        if (Cfg::kHasY) {
          twait(&tempty[tb], (tuse & 1) ^ 1, prof, &dw[2]);
          tc_fence_after();
        }
        const uint32_t t_tmem = tmem_base + Cfg::kYBase + tb * Cfg::kYCols;
        uint32_t s_tmem = tmem_base;
        int in_chunk = 0;
        bool first = true;
        // one k-step: the 3 (GRP) or 6 products of every K16 slice of the
        // stage; A planes `a_plane` bytes apart (boxes, or K16 slices)
        auto step = [&](uint32_t abase, uint32_t bbase, uint32_t a_plane, bool last_of_tile) {
          if (in_chunk == 0) {
            const int sb = g & 1;
            twait(&sempty[sb], ((g >> 1) & 1) ^ 1, prof, &dw[3]);
            tc_fence_after();
            s_tmem = tmem_base + sb * Cfg::kXCols;
          }
          // descriptors by adding to the 16-byte address field (shared
          // addresses < 256 KB: no carry out of its 14 bits) -- the issuing
          // thread's scalar work between MMA batches is tensor-pipe idle time
          const uint64_t ad = kADescHi | (abase >> 4), bd = kBDescHi | (bbase >> 4);
          const uint32_t ap = a_plane >> 4;
#pragma unroll
          for (int kk = 0; kk < Cfg::kKSteps; ++kk) {
            const uint64_t ah = ad + 2 * kk;  // K16 slice kk: +32 B
            const uint64_t am = ah + ap;
            const uint64_t al = ah + 2 * ap;
            const uint64_t bh = bd + 2 * kk;
            const uint32_t t_acc = (first && kk == 0) ? 0u : 1u;
            const uint32_t s_acc = (in_chunk | kk) != 0 ? 1u : 0u;
            if constexpr (Cfg::kGrp) {
              // X[0:192] += A_h x [B_h|B_m|B_l]; X[64:192] += A_m x [B_h|B_m];
              // X[64:128] += A_l x B_h
              tc_mma<MmaKind::kF16>(s_tmem, ah, bh, idesc3, s_acc);
              tc_mma<MmaKind::kF16>(s_tmem + BN, am, bh, idesc2, 1u);
              tc_mma<MmaKind::kF16>(s_tmem + BN, al, bh, idesc, 1u);
            } else {
              const uint64_t bm = bh + (kPlaneB >> 4);
              const uint64_t bl = bh + 2 * (kPlaneB >> 4);
              if constexpr (PAIR) {
                tc_mma_pair<MmaKind::kF16>(s_tmem, ah, bh, idesc, s_acc);
                tc_mma_pair<MmaKind::kF16>(t_tmem, ah, bm, idesc, t_acc);
                tc_mma_pair<MmaKind::kF16>(t_tmem, am, bh, idesc, 1u);
                tc_mma_pair<MmaKind::kF16>(t_tmem, ah, bl, idesc, 1u);
                tc_mma_pair<MmaKind::kF16>(t_tmem, al, bh, idesc, 1u);
                tc_mma_pair<MmaKind::kF16>(t_tmem, am, bm, idesc, 1u);
              } else {
                tc_mma<MmaKind::kF16>(s_tmem, ah, bh, idesc, s_acc);
                tc_mma<MmaKind::kF16>(t_tmem, ah, bm, idesc, t_acc);
                tc_mma<MmaKind::kF16>(t_tmem, am, bh, idesc, 1u);
                tc_mma<MmaKind::kF16>(t_tmem, ah, bl, idesc, 1u);
                tc_mma<MmaKind::kF16>(t_tmem, al, bh, idesc, 1u);
                tc_mma<MmaKind::kF16>(t_tmem, am, bm, idesc, 1u);
              }
            }
          }
          first = false;
          if (++in_chunk == chunk || last_of_tile) {
            if constexpr (PAIR) tc_commit_pair(&sfull[g & 1], 3);  // both CTAs' epilogues
            else tc_commit(&sfull[g & 1]);  // chunk ready to fold
            ++g;
            in_chunk = 0;
          }
        };
        if (ring && kFast && p.chunk_iters >= R * S) {
          // the row ring with the issue loop reduced to descriptor adds and
          // incrementally stepped row / slot counters. The tensor pipe queues
          // only about one tap of MMAs, so every wait or scalar step between
          // two tiles is pipe idle time: the next tile's waits (its new row,
          // its chunk buffer) run DURING this tile's last taps when the next
          // tile is the next row of the same image (at an image change the
          // new image's rows may need this tile's slots, released at its end)
          if (!f_prepared) {
            if (item == it_lo) {
              f_img = item / bands;  // n_tiles == 1 in ring mode
              f_oh = item - f_img * bands;
              f_s0 = f_oh % nrows;
              ring_v = f_oh;
              ring_slot = f_s0;
            } else {  // the next image
              ++f_img;
              f_oh = 0;
              f_s0 = 0;
              ring_v = 0;
              ring_slot = 0;
            }
            for (; ring_v < f_oh + R; ++ring_v) {
              twait(&hfull[ring_slot], (fillpar >> ring_slot) & 1u, prof, &dw[4]);
              fillpar ^= 1u << ring_slot;
              ring_slot = ring_slot + 1 == nrows ? 0 : ring_slot + 1;
            }
            twait(&sempty[g & 1], ((g >> 1) & 1) ^ 1, prof, &dw[3]);
            tc_fence_after();
          }
          const int cur_oh = f_oh, cur_s0 = f_s0;
          const bool next_same = item + 1 < it_hi && cur_oh + 1 < bands;
          f_prepared = false;
          const int sb = g & 1;
          const uint32_t x = tmem_base + sb * Cfg::kXCols;
          const int prep_at = R * S > 3 ? R * S - 3 : 0;
          uint64_t bh = bdesc0;
          int slot = cur_s0;
          auto prep_next = [&]() {  // the next tile's new row and chunk buffer
            ++f_oh;
            f_s0 = f_s0 + 1 == nrows ? 0 : f_s0 + 1;
            for (; ring_v < f_oh + R; ++ring_v) {
              twait(&hfull[ring_slot], (fillpar >> ring_slot) & 1u, prof, &dw[4]);
              fillpar ^= 1u << ring_slot;
              ring_slot = ring_slot + 1 == nrows ? 0 : ring_slot + 1;
            }
            twait(&sempty[(g + 1) & 1], (((g + 1) >> 1) & 1) ^ 1, prof, &dw[3]);
            tc_fence_after();
            f_prepared = true;
          };
          auto tap3 = [&](uint64_t ah, uint32_t acc) {
            tc_mma<MmaKind::kF16>(x, ah, bh, idesc3, acc);
            tc_mma<MmaKind::kF16>(x + BN, ah + 2, bh, idesc2, 1u);  // A_m: +32 B
            tc_mma<MmaKind::kF16>(x + BN, ah + 4, bh, idesc, 1u);   // A_l: +64 B
            bh += Cfg::kBStage >> 4;
          };
          if (R == 4 && S == 4) {
            // the space-to-depth stem (4 x 4 taps): fully unrolled, so the
            // issuing thread only adds descriptors between MMAs
#pragma unroll
            for (int r = 0; r < 4; ++r) {
              uint64_t ah = adesc0 + static_cast<uint64_t>(slot) * hstep;
              slot = slot + 1 == nrows ? 0 : slot + 1;
#pragma unroll
              for (int s = 0; s < 4; ++s) {
                tap3(ah, (r | s) != 0 ? 1u : 0u);
                ah += SWZ >> 4;
                if (r == 0 && s == 0 && pend_sb >= 0) {
                  tc_commit(&sfull[pend_sb]);
                  tc_commit(&hempty[pend_s0]);
                  pend_sb = -1;
                }
                if (r * 4 + s == 13 && next_same) prep_next();
              }
            }
          } else {
            int tap = 0;
            for (int r = 0; r < R; ++r) {
              uint64_t ah = adesc0 + static_cast<uint64_t>(slot) * hstep;
              slot = slot + 1 == nrows ? 0 : slot + 1;
              for (int s = 0; s < S; ++s, ++tap) {
                tap3(ah, (r | s) != 0 ? 1u : 0u);
                ah += SWZ >> 4;
                if (tap == prep_at && next_same) prep_next();
              }
            }
          }
          if (next_same && R == 4 && S == 4) {  // committed after the next tile's first tap
            pend_sb = sb;
            pend_s0 = cur_s0;
            ++g;
            continue;
          }
          tc_commit(&sfull[sb]);
          ++g;
          // the next item is the next row of the same image: only row cur_oh
          // is done; otherwise all r rows are
          if (next_same) {
            tc_commit(&hempty[cur_s0]);
          } else {
            int sl = cur_s0;
            for (int r = 0; r < R; ++r) {
              tc_commit(&hempty[sl]);
              sl = sl + 1 == nrows ? 0 : sl + 1;
            }
          }
        } else if (ring) {
          // one output row: taps (r, s) read row slot (oh0 + r) % rows from
          // pixel s on; rows land once, in order, and are released when the
          // last of their r readers is issued
          const int m_tile = item / p.n_tiles;
          const int img = m_tile / p.bands;
          const int oh0 = (m_tile - img * p.bands) * p.th;
          if (img != ring_img) {
            ring_img = img;
            ring_v = oh0;
          }
          for (; ring_v < oh0 + p.r; ++ring_v) {
            const int slot = ring_v % p.rows;
            twait(&hfull[slot], (fillpar >> slot) & 1u, prof, &dw[4]);
            fillpar ^= 1u << slot;
          }
          tc_fence_after();
          const uint32_t a_plane = INTER ? 32u : static_cast<uint32_t>(p.halo_bytes);
          for (int r = 0; r < p.r; ++r) {
            const uint32_t row = smem_u32(sHalo + ((oh0 + r) % p.rows) * p.halo_bytes);
            for (int s = 0; s < p.s; ++s) {
              const int k = r * p.s + s;
              uint32_t bbase;
              if (RES) {
                bbase = smem_u32(sRes) + k * Cfg::kBStage;
              } else {
                twait(&full[stage], phase, prof, &dw[4]);
                tc_fence_after();
                bbase = smem_u32(sRing + stage * Cfg::kStage);
              }
              step(row + s * SWZ, bbase, a_plane, r + 1 == p.r && s + 1 == p.s);
              if (!RES) {
                tc_commit(&empty[stage]);
                if (++stage == STAGES) {
                  stage = 0;
                  phase ^= 1;
                }
              }
            }
          }
          // the next item is the next row of the same image: only row oh0
          // is done; otherwise all r rows are (and any prefetched beyond)
          bool next_row = false;
          if (item + 1 < it_hi) {
            const int nm = (item + 1) / p.n_tiles;
            const int nimg = nm / p.bands;
            next_row = nimg == img && (nm - nimg * p.bands) * p.th == oh0 + 1;
          }
          if (next_row) {
            tc_commit(&hempty[oh0 % p.rows]);
          } else {
            for (int v = oh0; v < oh0 + p.r; ++v) tc_commit(&hempty[v % p.rows]);
          }
        } else if constexpr (HALO) {
          const uint32_t a_plane = INTER ? 32u : static_cast<uint32_t>(p.halo_bytes);
          for (int cb = 0; cb < p.cblocks; ++cb) {
            twait(&hfull[hb], hphase, prof, &dw[4]);
            tc_fence_after();
            const uint32_t halo = smem_u32(sHalo + hb * Cfg::kAPlanes * p.halo_bytes);
            for (int r = 0; r < p.r; ++r)
              for (int s = 0; s < p.s; ++s) {
                const int k = (r * p.s + s) * p.cblocks + cb;
                uint32_t bbase;
                if (RES) {
                  bbase = smem_u32(sRes) + k * Cfg::kBStage;
                } else {
                  twait(&full[stage], phase, prof, &dw[4]);
                  tc_fence_after();
                  bbase = smem_u32(sRing + stage * Cfg::kStage);
                }
                // tap (r, s) of output virtual row v reads halo row v + r*wp + s
                step(halo + (r * p.wp + s) * SWZ, bbase, a_plane,
                     cb + 1 == p.cblocks && r + 1 == p.r && s + 1 == p.s);
                if (!RES) {
                  tc_commit(&empty[stage]);
                  if (++stage == STAGES) {
                    stage = 0;
                    phase ^= 1;
                  }
                }
              }
            tc_commit(&hempty[hb]);  // halo free once these MMAs land
            if (++hb == p.hbuf) {
              hb = 0;
              hphase ^= 1;
            }
          }
        } else {
          const int kb = w_kb, ke = w_ke;
          for (int k = kb; k < ke; ++k) {
            twait(&full[stage], phase, prof, &dw[4]);
            tc_fence_after();
            const uint32_t base = smem_u32(sRing + stage * Cfg::kStage);
            step(base, RES ? smem_u32(sRes) + k * Cfg::kBStage : base + Cfg::kAPlanes * Cfg::kA,
                 kPlaneA, k + 1 == ke);
            // frees the smem slot (a pair: both CTAs') when the MMAs land
            if constexpr (PAIR) tc_commit_pair(&empty[stage], 3);
            else tc_commit(&empty[stage]);
            if (++stage == STAGES) {
              stage = 0;
              phase ^= 1;
            }
          }
        }
        if (Cfg::kHasY) {
          if constexpr (PAIR) tc_commit_pair(&tfull[tb], 3);
          else tc_commit(&tfull[tb]);
        }
      }
      if (pend_sb >= 0) {  // (the last tile never defers; kept for safety)
        tc_commit(&sfull[pend_sb]);
        tc_commit(&hempty[pend_s0]);
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
    WorkIter wi = make_iter();
    int item, mnu, kb, ke, split, nseg;
    // accumulator hand-back: a pair's peer arrives on the leader's barriers
    const uint32_t sempty_l = PAIR ? mapa_u32(smem_u32(sempty), 0) : 0u;
    const uint32_t tempty_l = PAIR ? mapa_u32(smem_u32(tempty), 0) : 0u;
    auto release = [&](uint64_t* bar, uint32_t bar_l) {
      if constexpr (PAIR) {
        if (rank != 0) {
          mbar_arrive_cluster(bar_l);
          return;
        }
      }
      mbar_arrive(bar);
    };
    for (; wi.next(item, mnu, kb, ke, split, nseg); ++local) {
      const int mn = own_mn(mnu);
      const int m_tile = mn / p.n_tiles;
      const int n_tile = mn - m_tile * p.n_tiles;
      const int row0 = m_tile * kBM + static_cast<int>(q * 32);
      // this lane's output row (NHWC row index), or -1: past M, or (HALO) a
      // junk virtual row of the shifted window
      int orow;
      int img = 0, oh0 = 0;
      if constexpr (HALO) {
        img = m_tile / p.bands;
        oh0 = (m_tile - img * p.bands) * p.th;
        const int v = static_cast<int>(q * 32 + lane);
        const int ohl = v / p.wp, ow = v - ohl * p.wp;
        orow = ow < p.ow && ohl < p.th && oh0 + ohl < p.oh ? (img * p.oh + oh0 + ohl) * p.ow + ow
                                                          : -1;
      } else {
        const int row = row0 + static_cast<int>(lane);
        orow = row < p.m ? row : -1;
      }
      const int nch = (ke - kb + chunk - 1) / chunk;
      float sum[HB];
      float cross[Cfg::kGrp ? HB : 1];  // GRP: the cross terms of the X chunks
#pragma unroll
      for (int j = 0; j < HB; ++j) sum[j] = 0.0f;
#pragma unroll
      for (int j = 0; j < (Cfg::kGrp ? HB : 1); ++j) cross[j] = 0.0f;
      auto fold = [&](float* acc, uint32_t taddr) {
#pragma unroll
        for (int c0 = 0; c0 < HB; c0 += 32) {
          uint32_t v[32];
          tmem_ld32(taddr + c0, v);
          tmem_ld_wait();
#pragma unroll
          for (int j = 0; j < 32; ++j) acc[c0 + j] = __fadd_rn(acc[c0 + j], __uint_as_float(v[j]));
        }
      };
      // hh chunks, folded in K order with round-to-nearest adds (GRP: the
      // chunk also carries hm | hl, folded into the cross-term registers)
#pragma unroll 1
      for (int c = 0; c < nch; ++c, ++g) {
        const int sb = g & 1;
        twait(&sfull[sb], (g >> 1) & 1, prof, &dw[5]);
        tc_fence_after();
        const uint32_t xb = lane_base + sb * Cfg::kXCols;
        fold(sum, xb);
        if constexpr (Cfg::kGrp) {
          fold(cross, xb + BN);
          fold(cross, xb + 2 * BN);
        }
        tc_fence_before();
        // GRP (no tile accumulator): the fault test drops a chunk arrive
        if (!(Cfg::kGrp && p.fault == 1 && local == 0 && c == 0)) release(&sempty[sb], sempty_l + 8 * sb);
      }
      if constexpr (Cfg::kHasY) {
        // + the tile's cross-term accumulator
        const int tb = local % Cfg::kYBufs;
        twait(&tfull[tb], (local / Cfg::kYBufs) & 1, prof, &dw[6]);
        tc_fence_after();
        fold(sum, lane_base + Cfg::kYBase + tb * Cfg::kYCols);
        tc_fence_before();
        // p.fault == 1 (tests only): lose one arrive -- the MMA warp then
        // waits for this accumulator forever and the mbarrier watchdog must trap
        if (!(p.fault == 1 && local == 0)) release(&tempty[tb], tempty_l + 8 * tb);
      }
      if constexpr (Cfg::kGrp) {
#pragma unroll
        for (int j = 0; j < HB; ++j) sum[j] = __fadd_rn(sum[j], cross[j]);
      }
      if (PAIR && m_tile >= p.m_tiles) continue;  // a pair's phantom tile: nothing to store
      if (nseg > 1) {
        // publish this split's partial ([item][warp][column][lane]: one
        // 128-B line per column); the last split of the tile sums them all
        // in split order
        float* mine = p.ws + ((static_cast<size_t>(mn) * splits + split) * 8 + ew) * HB * 32 + lane;
#pragma unroll
        for (int j = 0; j < HB; ++j) __stcg(mine + j * 32, sum[j]);
        __threadfence();
        epi::named_bar_sync(1, 256);
        if (etid == 0) *s_last = atomicAdd(&p.tile_cnt[mn], 1) == nseg - 1;
        epi::named_bar_sync(1, 256);
        if (!*s_last) continue;
        __threadfence();
        const float* part = p.ws + (static_cast<size_t>(mn) * splits * 8 + ew) * HB * 32 + lane;
#pragma unroll
        for (int j = 0; j < HB; ++j) sum[j] = __ldcg(part + j * 32);
#pragma unroll 1
        for (int sp = 1; sp < nseg; ++sp) {
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
          if (orow < 0 || col >= p.oc) continue;
          const int64_t o = static_cast<int64_t>(orow) * p.oc + col;
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
      if (PROG == epi::kProgBiasAddRelu && orow >= 0)
        rrow = static_cast<const uint8_t*>(p.epi.residual) +
               (static_cast<int64_t>(orow) * p.oc + n_tile * BN + hf * HB) * 4;
      // shifted window with th > 1: a warp's 32 virtual rows can straddle
      // two output rows, so the half's 4 warps stage all 128 rows (their 4
      // KB stages are consecutive) and one thread stores each output row of
      // the tile as a {32 ch, OW px} box from staged row ohl * wp
      const bool group = HALO && p.th > 1;
#pragma unroll
      for (int c0 = 0; c0 < HB; c0 += 32) {
        if (n_tile * BN + hf * HB + c0 < p.oc) {
          uint32_t acc[32];
#pragma unroll
          for (int j = 0; j < 32; ++j) acc[j] = __float_as_uint(sum[c0 + j]);
          if (group) {
            if (q == 0 && lane == 0) bulk_wait_read<0>();  // the half's previous stores have read it
            epi::named_bar_sync(3 + hf, 128);
            epi::epi_acc_to_box<PROG, 4>(acc, static_cast<int>(lane), sBias + hf * HB + c0,
                                         stage_u32, &overflow, rrow ? rrow + c0 * 4 : nullptr);
            fence_proxy_async_smem();
            epi::named_bar_sync(3 + hf, 128);
            if (q == 0 && lane == 0) {
              const uint32_t half = smem_u32(sStage + hf * 4 * 4096);
              for (int ohl = 0; ohl < p.th && oh0 + ohl < p.oh; ++ohl)
                tma_store_3d(&tm_y, half + static_cast<uint32_t>(ohl * p.wp) * 128,
                             n_tile * BN + hf * HB + c0, 0, img * p.oh + oh0 + ohl);
              bulk_commit();
            }
            continue;
          }
          if (lane == 0) bulk_wait_read<0>();  // the box's previous store has read it
          __syncwarp();
          epi::epi_acc_to_box<PROG, 4>(acc, static_cast<int>(lane), sBias + hf * HB + c0,
                                       stage_u32, &overflow, rrow ? rrow + c0 * 4 : nullptr);
          fence_proxy_async_smem();
          __syncwarp();
          if (lane == 0) {
            if constexpr (HALO)  // one output row per tile: (OC, OW, N*OH) map
              tma_store_3d(&tm_y, stage_u32, n_tile * BN + hf * HB + c0, static_cast<int>(q * 32),
                           img * p.oh + oh0);
            else
              tma_store_2d(&tm_y, stage_u32, n_tile * BN + hf * HB + c0, row0);
            bulk_commit();
          }
        }
      }
    }
    if (lane == 0) bulk_wait_all();  // TMA stores done before smem goes away
    if (prof) dw[7] = clock64() - t_start - dw[5] - dw[6];
  }

  tc_fence_before();
  if constexpr (PAIR) cluster_sync();  // no DSMEM traffic may target an exited CTA
  else __syncthreads();
  tc_fence_after();
  if (warp == 2) {
    if constexpr (PAIR) tmem_dealloc_pair<Cfg::kTmemCols>(tmem_base);
    else tmem_dealloc<Cfg::kTmemCols>(tmem_base);
  }
  if (prof) {
    // one representative thread per role: producer warps 0 / 3, MMA warp 1,
    // the first epilogue thread
    const bool rep = ((warp == 0 || warp == 1 || warp == 3) && lane == 0) || threadIdx.x == 128;
    if (rep)
      for (int i = 0; i < 8; ++i)
        if (dw[i]) atomicAdd(&p.dbg[i], static_cast<unsigned long long>(dw[i]));
    if (threadIdx.x == 0) {
      atomicAdd(&p.dbg[8], static_cast<unsigned long long>(clock64() - t_start));
      atomicAdd(&p.dbg[9], static_cast<unsigned long long>((it_hi - it_lo + it_step - 1) / it_step));
    }
  }
}

template <int BN, int SWZ, int STAGES, bool INTER, bool RES, bool HALO, int PROG, bool PAIR>
int launch_f32tc_inst(const CUtensorMap& tm_a, const CUtensorMap& tm_b, const CUtensorMap& tm_y,
                      const ConvGemmParams& p, int grid, cudaStream_t stream) {
  using Cfg = F32tcCfg<BN, SWZ, STAGES, INTER, RES, HALO, PAIR>;
  auto kfn = conv_f32tc_kernel<BN, SWZ, STAGES, INTER, RES, HALO, PROG, PAIR>;
  const int smem = Cfg::kSmem + (RES ? p.res_bytes : 0) +
                   (HALO ? p.hbuf * Cfg::kAPlanes * p.halo_bytes : 0);
  if (smem > 227 * 1024) return -1;
  cudaError_t e = cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) return e;
  if constexpr (PAIR)
    e = launch_pdl_cluster(kfn, dim3(grid), dim3(kThreads), smem, stream, 2, tm_a, tm_b, tm_y, p);
  else
    e = launch_pdl(kfn, dim3(grid), dim3(kThreads), smem, stream, tm_a, tm_b, tm_y, p);
  if (e != cudaSuccess) return e;
  return cudaGetLastError();
}

template <int BN, int SWZ, int STAGES, bool INTER, bool RES, bool HALO, bool PAIR = false>
int launch_f32tc_prog(const CUtensorMap& tm_a, const CUtensorMap& tm_b, const CUtensorMap& tm_y,
                      const ConvGemmParams& p, int prog, int grid, cudaStream_t st) {
  switch (prog) {
    case epi::kProgNone: return launch_f32tc_inst<BN, SWZ, STAGES, INTER, RES, HALO, epi::kProgNone, PAIR>(tm_a, tm_b, tm_y, p, grid, st);
    case epi::kProgBias: return launch_f32tc_inst<BN, SWZ, STAGES, INTER, RES, HALO, epi::kProgBias, PAIR>(tm_a, tm_b, tm_y, p, grid, st);
    case epi::kProgBiasRelu: return launch_f32tc_inst<BN, SWZ, STAGES, INTER, RES, HALO, epi::kProgBiasRelu, PAIR>(tm_a, tm_b, tm_y, p, grid, st);
    case epi::kProgBiasAddRelu: return launch_f32tc_inst<BN, SWZ, STAGES, INTER, RES, HALO, epi::kProgBiasAddRelu, PAIR>(tm_a, tm_b, tm_y, p, grid, st);
    default: return -1;
  }
}

// The instantiated (BN, block, stages, interleaved, resident weights, halo)
// set. Halo instances: the ring carries weights only (STAGES = its depth,
// 0 with resident weights).
#define TEC_F32TC_INSTANCES(X)         \
  X(64, 128, 2, false, false, false)   \
  X(128, 128, 2, false, false, false)  \
  X(64, 32, 8, false, false, false)    \
  X(128, 32, 6, false, false, false)   \
  X(64, 128, 6, true, false, false)    \
  X(128, 128, 5, true, false, false)   \
  X(64, 128, 3, false, true, false)    \
  X(128, 128, 2, false, true, false)   \
  X(64, 128, 6, true, true, false)     \
  X(128, 128, 4, true, true, false)    \
  X(64, 128, 1, true, true, true)      \
  X(64, 128, 3, false, false, true)    \
  X(128, 128, 2, false, false, true)

}  // namespace

// Fixed shared memory of an instance (resident weights come on top), its
// ring depth, and B bytes per k-iteration; -1 when not instantiated.
int conv_f32tc_smem_bytes(int bn, int swz, bool inter, bool res, bool halo) {
#define TEC_X(BN, SW, ST, IN, RS, HA)                                     \
  if (bn == BN && swz == SW && inter == IN && res == RS && halo == HA) \
    return F32tcCfg<BN, SW, ST, IN, RS, HA>::kSmem;
  TEC_F32TC_INSTANCES(TEC_X)
#undef TEC_X
  return -1;
}

int conv_f32tc_stages(int bn, int swz, bool inter, bool res, bool halo) {
#define TEC_X(BN, SW, ST, IN, RS, HA) \
  if (bn == BN && swz == SW && inter == IN && res == RS && halo == HA) return ST;
  TEC_F32TC_INSTANCES(TEC_X)
#undef TEC_X
  return -1;
}

int conv_f32tc_b_stage_bytes(int bn, int swz, bool inter) {
  return 3 * bn * (inter ? 32 : swz);
}

// The CTA-pair instance (im2col, BN = 128, 128-B channel blocks): its
// shared memory per CTA, or -1 for another configuration.
int conv_f32tc_pair_smem_bytes(int bn, int swz, bool inter, bool res, bool halo) {
  if (bn != 128 || swz != 128 || inter || res || halo) return -1;
  return F32tcCfg<128, 128, 2, false, false, false, true>::kSmem;
}

// Returns a cudaError_t, or -1 for an unsupported (bn, swz, program).
int launch_conv_f32tc(const CUtensorMap& tm_a, const CUtensorMap& tm_b, const CUtensorMap& tm_y,
                      const ConvGemmParams& p, int bn, int swz, bool inter, bool res, bool halo,
                      int prog, int grid, cudaStream_t st, bool pair) {
  if (pair) {
    if (conv_f32tc_pair_smem_bytes(bn, swz, inter, res, halo) < 0) return -1;
    return launch_f32tc_prog<128, 128, 2, false, false, false, true>(tm_a, tm_b, tm_y, p, prog,
                                                                    grid, st);
  }
#define TEC_X(BN, SW, ST, IN, RS, HA)                                     \
  if (bn == BN && swz == SW && inter == IN && res == RS && halo == HA) \
    return launch_f32tc_prog<BN, SW, ST, IN, RS, HA>(tm_a, tm_b, tm_y, p, prog, grid, st);
  TEC_F32TC_INSTANCES(TEC_X)
#undef TEC_X
  return -1;
}

}  // namespace tec_sm100
