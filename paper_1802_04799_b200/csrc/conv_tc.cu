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
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "conv_params.h"
#include "sm100_ptx.cuh"

namespace tec_sm100 {

namespace {

constexpr int kBM = 128;
constexpr int kThreads = 256;  // 4 control warps + 4 epilogue warps
constexpr int kChunk = 32;     // epilogue columns per tcgen05.ld

// 32 consecutive elements of an output-shaped operand, as floats.
__device__ __forceinline__ void load32_f(const void* base, int64_t off,
                                         int type, bool vec, int ncols,
                                         float (&r)[kChunk]) {
  if (type == kBF16) {
    const __nv_bfloat16* p = static_cast<const __nv_bfloat16*>(base) + off;
    if (vec) {
      uint4 u[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) u[i] = __ldg(reinterpret_cast<const uint4*>(p) + i);
      const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(u);
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        const float2 f = __bfloat1622float2(h[i]);
        r[2 * i] = f.x;
        r[2 * i + 1] = f.y;
      }
    } else {
#pragma unroll
      for (int j = 0; j < kChunk; ++j) r[j] = j < ncols ? __bfloat162float(p[j]) : 0.f;
    }
  } else {
    const float* p = static_cast<const float*>(base) + off;
    if (vec) {
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const float4 f = __ldg(reinterpret_cast<const float4*>(p) + i);
        r[4 * i] = f.x; r[4 * i + 1] = f.y; r[4 * i + 2] = f.z; r[4 * i + 3] = f.w;
      }
    } else {
#pragma unroll
      for (int j = 0; j < kChunk; ++j) r[j] = j < ncols ? p[j] : 0.f;
    }
  }
}

__device__ __forceinline__ void load32_i(const int32_t* p, bool vec, int ncols,
                                         int32_t (&r)[kChunk]) {
  if (vec) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int4 f = __ldg(reinterpret_cast<const int4*>(p) + i);
      r[4 * i] = f.x; r[4 * i + 1] = f.y; r[4 * i + 2] = f.z; r[4 * i + 3] = f.w;
    }
  } else {
#pragma unroll
    for (int j = 0; j < kChunk; ++j) r[j] = j < ncols ? p[j] : 0;
  }
}

// Float epilogue chain over one 32-column chunk of one output row. Each
// member rounds to float separately (the reference materialises every
// member, R/src/graph.cpp:215-219); __f*_rn forbids FMA contraction.
__device__ __forceinline__ void epi_chunk_float(const ConvGemmParams& p, int row,
                                                int col0, int ncols,
                                                const uint32_t (&acc)[kChunk]) {
  const EpilogueParams& e = p.epi;
  const int64_t base = static_cast<int64_t>(row) * p.oc + col0;
  const bool vec = ncols == kChunk && (p.oc % 8) == 0;
  float v[kChunk];
#pragma unroll
  for (int j = 0; j < kChunk; ++j) v[j] = __uint_as_float(acc[j]);
#pragma unroll 1
  for (int i = 0; i < e.n_ops; ++i) {
    const int op = e.ops[i];
    if (op == kEpiScale) {
      const float s = e.fscale[i];
#pragma unroll
      for (int j = 0; j < kChunk; ++j) v[j] = __fmul_rn(v[j], s);
    } else if (op == kEpiBias) {
      float b[kChunk];
      load32_f(e.bias, col0, kF32, ncols == kChunk, ncols, b);
#pragma unroll
      for (int j = 0; j < kChunk; ++j) v[j] = __fadd_rn(v[j], b[j]);
    } else if (op == kEpiAdd) {
      float r[kChunk];
      load32_f(e.residual, base, p.out_type, vec, ncols, r);
#pragma unroll
      for (int j = 0; j < kChunk; ++j) v[j] = __fadd_rn(v[j], r[j]);
    } else if (op == kEpiMul) {
      float r[kChunk];
      load32_f(e.mul_operand, base, p.out_type, vec, ncols, r);
#pragma unroll
      for (int j = 0; j < kChunk; ++j) v[j] = __fmul_rn(v[j], r[j]);
    } else if (op == kEpiRelu) {
#pragma unroll
      for (int j = 0; j < kChunk; ++j) v[j] = (v[j] < 0.0f) ? 0.0f : v[j];  // std::max(x, 0)
    }
  }
  if (p.out_type == kBF16) {
    __nv_bfloat16* yp = static_cast<__nv_bfloat16*>(p.y) + base;
    if (vec) {
      __nv_bfloat162 h[16];
#pragma unroll
      for (int j = 0; j < 16; ++j) h[j] = __floats2bfloat162_rn(v[2 * j], v[2 * j + 1]);
      uint4* dst = reinterpret_cast<uint4*>(yp);
      const uint4* src = reinterpret_cast<const uint4*>(h);
#pragma unroll
      for (int j = 0; j < 4; ++j) dst[j] = src[j];
    } else {
#pragma unroll
      for (int j = 0; j < kChunk; ++j)
        if (j < ncols) yp[j] = __float2bfloat16_rn(v[j]);
    }
  } else {
    float* yp = static_cast<float*>(p.y) + base;
    if (vec) {
      float4* dst = reinterpret_cast<float4*>(yp);
#pragma unroll
      for (int j = 0; j < 8; ++j)
        dst[j] = make_float4(v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]);
    } else {
#pragma unroll
      for (int j = 0; j < kChunk; ++j)
        if (j < ncols) yp[j] = v[j];
    }
  }
}

// Integer epilogue: int64 arithmetic, i32 range check after every member
// (DenseTensor::set_i, R/include/tec/tensor.hpp:63-69).
__device__ __forceinline__ void epi_chunk_int(const ConvGemmParams& p, int row,
                                              int col0, int ncols,
                                              const uint32_t (&acc)[kChunk],
                                              bool* overflow) {
  const EpilogueParams& e = p.epi;
  const int64_t base = static_cast<int64_t>(row) * p.oc + col0;
  const bool vec = ncols == kChunk && (p.oc % 4) == 0;
  int64_t v[kChunk];
#pragma unroll
  for (int j = 0; j < kChunk; ++j) v[j] = static_cast<int32_t>(acc[j]);
  bool ovf = false;
#pragma unroll 1
  for (int i = 0; i < e.n_ops; ++i) {
    const int op = e.ops[i];
    if (op == kEpiScale) {
      const int64_t s = e.iscale[i];
#pragma unroll
      for (int j = 0; j < kChunk; ++j) v[j] *= s;
    } else if (op == kEpiBias) {
      int32_t b[kChunk];
      load32_i(static_cast<const int32_t*>(e.bias) + col0, ncols == kChunk, ncols, b);
#pragma unroll
      for (int j = 0; j < kChunk; ++j) v[j] += b[j];
    } else if (op == kEpiAdd || op == kEpiMul) {
      int32_t r[kChunk];
      load32_i(static_cast<const int32_t*>(op == kEpiAdd ? e.residual : e.mul_operand) + base,
               vec, ncols, r);
      if (op == kEpiAdd) {
#pragma unroll
        for (int j = 0; j < kChunk; ++j) v[j] += r[j];
      } else {
#pragma unroll
        for (int j = 0; j < kChunk; ++j) v[j] *= r[j];
      }
    } else if (op == kEpiRelu) {
#pragma unroll
      for (int j = 0; j < kChunk; ++j) v[j] = v[j] < 0 ? 0 : v[j];
    }
#pragma unroll
    for (int j = 0; j < kChunk; ++j)
      ovf |= (j < ncols) && (v[j] < INT32_MIN || v[j] > INT32_MAX);
  }
  if (ovf) *overflow = true;
  int32_t* yp = static_cast<int32_t*>(p.y) + base;
  if (vec) {
    int4* dst = reinterpret_cast<int4*>(yp);
#pragma unroll
    for (int j = 0; j < 8; ++j)
      dst[j] = make_int4(static_cast<int32_t>(v[4 * j]), static_cast<int32_t>(v[4 * j + 1]),
                         static_cast<int32_t>(v[4 * j + 2]), static_cast<int32_t>(v[4 * j + 3]));
  } else {
#pragma unroll
    for (int j = 0; j < kChunk; ++j)
      if (j < ncols) yp[j] = static_cast<int32_t>(v[j]);
  }
}

template <MmaKind KIND, int BN, int STAGES, int SWZ>
struct ConvCfg {
  static constexpr int kABytes = kBM * SWZ;  // one stage of A
  static constexpr int kBBytes = BN * SWZ;   // one stage of B
  static constexpr int kStageBytes = kABytes + kBBytes;
  static constexpr int kMmaPerStage = SWZ / 32;  // each MMA eats 32 B of K
  static constexpr uint32_t kTmemCols = 2 * BN <= 32    ? 32
                                        : 2 * BN <= 64  ? 64
                                        : 2 * BN <= 128 ? 128
                                        : 2 * BN <= 256 ? 256
                                                        : 512;
  static constexpr int kSmemBytes =
      1024 /*align slack*/ + STAGES * kStageBytes + 256 /*barriers*/;
};

template <MmaKind KIND, int BN, int STAGES, int SWZ>
__global__ void __launch_bounds__(kThreads, 1)
    conv_fprop_tc_kernel(const __grid_constant__ CUtensorMap tm_a,
                         const __grid_constant__ CUtensorMap tm_b,
                         const ConvGemmParams p) {
  using Cfg = ConvCfg<KIND, BN, STAGES, SWZ>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + STAGES * Cfg::kABytes;
  uint64_t* full = reinterpret_cast<uint64_t*>(sB + STAGES * Cfg::kBBytes);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const uint32_t warp = warp_id();
  const uint32_t lane = threadIdx.x & 31;
  const int num_tiles = p.m_tiles * p.n_tiles;
  const int k_iters = p.r * p.s * p.cblocks;
  constexpr int kCB =
      SWZ / (KIND == MmaKind::kF16 ? 2 : KIND == MmaKind::kTF32 ? 4 : 1);

  if (warp == 0 && elect_one()) {
    tma_prefetch_desc(&tm_a);
    tma_prefetch_desc(&tm_b);
    for (int i = 0; i < STAGES; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&tfull[i], 1);
      mbar_init(&tempty[i], 128);
    }
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc<Cfg::kTmemCols>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    // ------------------------------------------------ TMA producer warp
    if (elect_one()) {
      int stage = 0;
      uint32_t phase = 0;
      const int ohw = p.oh * p.ow;
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
        for (int r = 0; r < p.r; ++r) {
          for (int s = 0; s < p.s; ++s) {
            const int kbase = (r * p.s + s) * p.cp;
            for (int cb = 0; cb < p.cblocks; ++cb) {
              mbar_wait(&empty[stage], phase ^ 1);
              mbar_arrive_expect_tx(&full[stage], Cfg::kStageBytes);
              tma_load_im2col_4d(sA + stage * Cfg::kABytes, &tm_a,
                                 &full[stage], cb * kCB, w0, h0, img,
                                 static_cast<uint16_t>(s),
                                 static_cast<uint16_t>(r));
              tma_load_2d(sB + stage * Cfg::kBBytes, &tm_b, &full[stage],
                          kbase + cb * kCB, n_tile * BN);
              if (++stage == STAGES) {
                stage = 0;
                phase ^= 1;
              }
            }
          }
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------ single-thread MMA issuer
    if (elect_one()) {
      constexpr uint32_t idesc = make_idesc<KIND>(kBM, BN);
      int stage = 0;
      uint32_t phase = 0;
      int local = 0;
      for (int tile = blockIdx.x; tile < num_tiles;
           tile += gridDim.x, ++local) {
        const int acc = local & 1;
        const uint32_t use = static_cast<uint32_t>(local >> 1);
        mbar_wait(&tempty[acc], (use & 1) ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * BN;
        for (int k = 0; k < k_iters; ++k) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          const uint32_t a_base = smem_u32(sA + stage * Cfg::kABytes);
          const uint32_t b_base = smem_u32(sB + stage * Cfg::kBBytes);
#pragma unroll
          for (int kk = 0; kk < Cfg::kMmaPerStage; ++kk) {
            const uint64_t ad = make_smem_desc<SWZ>(a_base + kk * 32, 8 * SWZ);
            const uint64_t bd = make_smem_desc<SWZ>(b_base + kk * 32, 8 * SWZ);
            tc_mma<KIND>(d_tmem, ad, bd, idesc, (k | kk) != 0 ? 1u : 0u);
          }
          tc_commit(&empty[stage]);  // frees the smem slot when MMAs land
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
        tc_commit(&tfull[acc]);  // accumulator ready for the epilogue
      }
    }
  } else if (warp >= 4) {
    // ------------------------------------------------- epilogue warps
    const uint32_t q = warp - 4;  // TMEM lane quadrant owned by this warp
    int local = 0;
    bool overflow = false;
    for (int tile = blockIdx.x; tile < num_tiles;
         tile += gridDim.x, ++local) {
      const int acc = local & 1;
      const uint32_t use = static_cast<uint32_t>(local >> 1);
      const int m_tile = tile / p.n_tiles;
      const int n_tile = tile - m_tile * p.n_tiles;
      const int row = m_tile * kBM + static_cast<int>(q * 32 + lane);
      const bool row_ok = row < p.m;
      mbar_wait(&tfull[acc], use & 1);
      tc_fence_after();
#pragma unroll 1
      for (int c0 = 0; c0 < BN; c0 += kChunk) {
        uint32_t v[kChunk];
        tmem_ld32(tmem_base + ((q * 32) << 16) + acc * BN + c0, v);
        tmem_ld_wait();
        if (c0 + kChunk >= BN) {
          // Every TMEM read of this accumulator is done: hand it back to
          // the MMA warp before the global stores of the last chunk.
          tc_fence_before();
          mbar_arrive(&tempty[acc]);
        }
        const int col0 = n_tile * BN + c0;
        if (!row_ok || col0 >= p.oc) continue;
        const int ncols = min(kChunk, p.oc - col0);
        if constexpr (KIND == MmaKind::kI8)
          epi_chunk_int(p, row, col0, ncols, v, &overflow);
        else
          epi_chunk_float(p, row, col0, ncols, v);
      }
    }
    if (overflow && p.err) atomicOr(p.err, 1);
  }

  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 2) tmem_dealloc<ConvCfg<KIND, BN, STAGES, SWZ>::kTmemCols>(tmem_base);
}

}  // namespace

// Launch wrapper, instantiated for the supported (kind, BN, swizzle) set.
// Returns a cudaError_t.
template <MmaKind KIND, int BN, int STAGES, int SWZ>
int launch_conv_fprop_tc(const CUtensorMap& tm_a, const CUtensorMap& tm_b,
                         const ConvGemmParams& p, int grid,
                         cudaStream_t stream) {
  using Cfg = ConvCfg<KIND, BN, STAGES, SWZ>;
  auto kfn = conv_fprop_tc_kernel<KIND, BN, STAGES, SWZ>;
  cudaError_t e = cudaFuncSetAttribute(
      kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::kSmemBytes);
  if (e != cudaSuccess) return e;
  kfn<<<grid, kThreads, Cfg::kSmemBytes, stream>>>(tm_a, tm_b, p);
  return cudaGetLastError();
}

#define TEC_INST(KIND, BN, ST, SWZ)                                         \
  template int launch_conv_fprop_tc<KIND, BN, ST, SWZ>(                    \
      const CUtensorMap&, const CUtensorMap&, const ConvGemmParams&, int, \
      cudaStream_t);

// bf16: 128 B channel blocks (64 ch) for Cp % 64 == 0, 32 B (16 ch) for
// the stem (C1, 3 -> 16 padded channels).
TEC_INST(MmaKind::kF16, 64, 8, 128)
TEC_INST(MmaKind::kF16, 128, 6, 128)
TEC_INST(MmaKind::kF16, 256, 4, 128)
TEC_INST(MmaKind::kF16, 64, 8, 32)
// int8: 128 B blocks (128 ch), 64 B (64 ch), 32 B (32 ch, the stem).
TEC_INST(MmaKind::kI8, 64, 8, 128)
TEC_INST(MmaKind::kI8, 128, 6, 128)
TEC_INST(MmaKind::kI8, 256, 4, 128)
TEC_INST(MmaKind::kI8, 64, 8, 64)
TEC_INST(MmaKind::kI8, 128, 6, 64)
TEC_INST(MmaKind::kI8, 64, 8, 32)
// tf32 (approximate-f32 3xTF32 path, K = [hi|hi|lo] x [hi|lo|hi]): 128 B
// blocks (32 ch), 64 B (16 ch, the stem: 3*3 -> 16 padded channels).
TEC_INST(MmaKind::kTF32, 64, 8, 128)
TEC_INST(MmaKind::kTF32, 128, 6, 128)
TEC_INST(MmaKind::kTF32, 256, 4, 128)
TEC_INST(MmaKind::kTF32, 64, 8, 64)

#undef TEC_INST

}  // namespace tec_sm100
