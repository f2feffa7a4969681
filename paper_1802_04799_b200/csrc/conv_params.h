// conv_params.h -- plain-old-data shared by the host launchers (C++) and
// the sm_100a kernels (CUDA). No torch or CUDA-runtime types.
#pragma once
#include <cstdint>

namespace tec_sm100 {

// Epilogue member ops, in fused-node member order (R/src/graph.cpp:209-222).
enum EpiOp : int32_t {
  kEpiNone = 0,
  kEpiScale = 1,  // x * c            R/src/ops.cpp:260-281
  kEpiBias = 2,   // x + b[oc]        R/src/ops.cpp:282-305
  kEpiAdd = 3,    // x + r (same shape) R/src/ops.cpp:216-223
  kEpiMul = 4,    // x * r (same shape) R/src/ops.cpp:224-231
  kEpiRelu = 5,   // max(x, 0)        R/src/ops.cpp:250-259
  kEpiRequant = 6,  // i32 -> i8 clamp((x*m + 2^(s-1)) >> s) (int8 graphs; last member)
};

enum ElemType : int32_t { kF32 = 0, kI32 = 1, kI8 = 2, kBF16 = 3 };

constexpr int kMaxEpi = 8;

struct EpilogueParams {
  int32_t n_ops;
  int32_t ops[kMaxEpi];
  float fscale[kMaxEpi];    // float-rounded scale factors (cstf)
  int64_t iscale[kMaxEpi];  // integral scale factors (cst)
  const void* bias;         // [OC], accumulator dtype (f32 / i32)
  const void* residual;     // NHWC [M][OC], output dtype (res_i8: i8)
  const void* mul_operand;  // NHWC [M][OC], output dtype
  // int8 graphs: the requantize member's parameters, and an
  // i8 residual entering as scale(cast(r, i32), res_scale) -- the identity
  // shortcut side chain fused into the add's operand read.
  int64_t rq_mult;
  int32_t rq_shift;
  int32_t res_i8;
  int64_t res_scale;
};

// Implicit-GEMM convolution: GEMM M = N*OH*OW output pixels (NHWC order),
// GEMM N = OC, GEMM K = R*S*Cp in (r, s, c) order.
struct ConvGemmParams {
  int32_t n, h, w, cp;  // input NHWC, cp = stored (padded) channels
  int32_t oh, ow, oc;
  int32_t r, s, sh, sw, ph, pw;
  int32_t m;            // n*oh*ow
  int32_t m_tiles, n_tiles;
  int32_t cblocks;      // cp / channels-per-block
  int32_t out_type;     // ElemType of y
  void* y;              // NHWC [M][OC]
  int32_t* err;         // set to 1 on i32 range overflow (may be null)
  EpilogueParams epi;
  // Optional pipeline profile (null in production): cycles summed over
  // CTAs -- [0] producer waiting for free slots, [1] MMA waiting for data,
  // [2] MMA waiting for a free accumulator, [3] epilogue waiting for an
  // accumulator, [4] epilogue busy, [5] CTA lifetime, [6] tiles.
  unsigned long long* dbg;
  int32_t epi_mode;     // 0: warp-coalesced epilogue, 1: per-thread rows
  int32_t tma_store;    // 1: y has a TMA store map (fast programs use it)
  // Split-K (splits > 1): work item = (output tile, split); split s runs
  // k-iterations [s*kps, min((s+1)*kps, k_iters)), writes its f32 partial
  // tile to ws, and the last split to arrive (tile_cnt) sums the partials in
  // split order and runs the epilogue. Requires the TMA-store fast path.
  int32_t splits, kps;
  int32_t nacc;         // TMEM accumulator buffers: 2 or 4 (when 4 fit in 512 columns)
  float* ws;            // [m_tiles*n_tiles][splits][128][BN]
  int32_t* tile_cnt;    // [m_tiles*n_tiles], zero between launches
  int32_t chunk_iters;  // f32tc: k-iterations per hh promotion chunk
  int32_t fault;        // test-only fault injection (TEC_SM100_FAULT): 1 = the
                        // epilogue drops its first accumulator-free arrive
  int32_t producers;    // f32tc: TMA issuing threads (1, or 2: A and B split)
  int32_t res_bytes;    // f32tc resident weights: shared-memory bytes of all B tiles
  // f32tc shifted-window mode (stride 1): a tile is th output rows of one
  // image; its (th + r - 1) x wp input rows are loaded ONCE per channel
  // block (tiled TMA, zero padding by OOB fill) and every filter tap is a
  // row shift of that halo (see conv_halo.cu); m_tiles = n * bands.
  int32_t th, wp, bands;
  int32_t halo_bytes;      // smem bytes per halo plane buffer (1024-aligned)
  int32_t halo_box_bytes;  // bytes one halo box lands (th + r - 1) * wp * 128
  int32_t hbuf;            // halo buffers (1 or 2), or the row ring's size
  // f32tc row ring (rows > 0; th == 1, one channel block, one N tile): each
  // CTA walks a CONTIGUOUS range of output rows, and the `rows` halo
  // buffers hold single input rows -- a row is loaded once and serves the
  // r consecutive output rows that read it (a per-tile halo box re-reads
  // r - 1 of its r rows). halo_bytes / halo_box_bytes are then per row.
  int32_t rows;
  // f32tc stream-K (stream_k = 1, im2col): CTA c of the grid owns work
  // positions [c*W/G, (c+1)*W/G) of W = tiles x k-iterations, so every CTA
  // does the same number of k-iterations; a tile cut by CTA boundaries is
  // finished by its last segment (partials summed in segment order; splits
  // = the most segments any tile has)
  int32_t stream_k;
};

// Shifted-window ("halo") implicit GEMM for stride-1 convolutions. A CTA
// tile is `th` output rows of one image (x BN output channels). The input
// rows it needs, padded left/right, are loaded ONCE per channel block as a
// (th + r - 1) x wp pixel halo (wp = w + 2*pw); output pixel (oh, ow) of the
// tile is "virtual row" v = oh_local * wp + ow, and filter tap (rh, rw)
// reads halo pixel v + rh * wp + rw -- a plain shift of the MMA operand's
// start address. Virtual rows with ow >= OW are computed and discarded.
struct ConvHaloParams {
  int32_t n, h, w, cp;  // input NHWC, cp = stored channels
  int32_t oh, ow, oc;
  int32_t r, s, ph, pw;
  int32_t th, wp;       // rows per tile, padded halo width
  int32_t bands;        // ceil(oh / th)
  int32_t n_tiles;      // ceil(oc / BN)
  int32_t cblocks;      // cp / channels-per-block
  int32_t halo_px;      // pixels per halo buffer (>= MS*128 + (r-1)*wp + s)
  int32_t resident;     // 1: all weights of the CTA's N tile stay in smem
  int32_t w_slots;      // weight tiles in smem (ring stages, or taps*cblocks)
  int32_t out_type;
  void* y;              // NHWC [N*OH*OW][OC]
  int32_t* err;
  EpilogueParams epi;
  unsigned long long* dbg;  // optional pipeline profile, as ConvGemmParams
  int32_t epi_mode;         // 0: warp-coalesced epilogue, 1: per-thread rows
  int32_t tma_store;        // 1: y has a TMA store map (fast programs use it)
  int32_t stage_bytes;      // epilogue stage (>= 32 KB); two halves, one per group
  int32_t cl;               // streamed weights: CTAs per cluster sharing them by multicast
  int32_t nacc;             // TMEM accumulator buffers: 2 or 4 (when 4 fit in 512 columns)
};

struct DepthwiseParams {
  int32_t n, h, w, c;   // NHWC
  int32_t oh, ow;
  int32_t r, s, sh, sw, ph, pw;
  int32_t in_type, out_type;
  const void* x;
  const void* wt;       // [R][S][C] (tap-major, channel fastest)
  void* y;
  int32_t* err;
  EpilogueParams epi;
};

// Tile shape of the TMA depthwise kernel (depthwise_tma.cu).
struct DwTmaShape {
  int32_t th;         // output rows per tile
  int32_t cb;         // channels per tile (block)
  int32_t rows_in;    // (th-1)*sw + 3
  int32_t cols_in;    // (ow-1)*sw + 3
  int32_t bands;      // ceil(oh / th)
  int32_t cblocks;    // c / cb
  int32_t buf_bytes;  // ni * rows_in * cols_in * cb * elem, rounded to 128
  int32_t ni;         // images per tile (TMA box N extent)
  float neg_zero;     // -0.0f, set by the host: the packed f32 products' addend
};

// max_pool2d / global_avg_pool on NHWC activations (pool.cu).
struct PoolParams {
  int32_t n, h, w, c, oh, ow, r, s, sh, sw, ph, pw;
  float scale;  // global_avg_pool factor, float-rounded 1/(H*W)
  int32_t type, out_type;  // ElemType
  const void* x;
  void* y;
};

// Unary member program of an elementwise graph node (elementwise.cu):
// cast / scale / relu / requantize in member order.
enum ElemOp : int32_t { kElemCast = 1, kElemScale = 2, kElemRelu = 3, kElemRequant = 4 };
constexpr int kMaxElemOps = 4;

struct ElemProg {
  int32_t n_ops;
  int32_t kind[kMaxElemOps];
  int32_t shift[kMaxElemOps];      // REQUANTIZE
  int32_t cast_to_f[kMaxElemOps];  // CAST: 1 = to f32 (else to an integer type)
  int64_t mult[kMaxElemOps];       // REQUANTIZE multiplier / integral SCALE factor
  float fscale[kMaxElemOps];       // float-rounded SCALE factor (f32 data)
  int32_t in_type, out_type;       // ElemType
  int32_t out_f;                   // final value is in the float domain
  int64_t count;                   // elements
};

}  // namespace tec_sm100
