// conv_epilogue.cuh -- fused-epilogue helpers shared by the tensor-core conv
// kernels: accumulator columns straight from TMEM, through the fused members
// (scale / bias_add / add / mul / relu, R/src/ops.cpp:216-305) in member
// order, to global memory.
//
// Two forms:
//  * epi_warp_block (default): a warp owns 32 TMEM lanes (= 32 output rows)
//    and one 32-column block; rows are transposed through a 4 KB swizzled
//    shared-memory stage so global loads/stores move whole 32-byte sectors.
//  * epi_chunk_* (fallback for channel counts that are not a multiple of
//    one 16-byte vector): one thread, one row, 32 columns.
// Both round every member to float separately (the reference materialises
// every member, R/src/graph.cpp:215-219; __f*_rn forbids FMA contraction)
// and range-check every integer member (DenseTensor::set_i,
// R/include/tec/tensor.hpp:63-69).
#pragma once
#include <cuda_bf16.h>

#include <cstdint>

#include "conv_params.h"
#include "sm100_ptx.cuh"

namespace tec_sm100 {
namespace epi {

constexpr int kChunk = 32;  // epilogue columns per tcgen05.ld

// The fused-member program, decoded ONCE per thread into registers (op
// codes packed 4 bits each; scale factors as f32 and i64), so the per-block
// loops never index kernel-parameter space dynamically.
// (Scale factors stay in parameter space: the member loops are fully
// unrolled, so e.fscale[i] / e.iscale[i] are static-offset constant loads.)
struct EpiProg {
  uint32_t ops = 0;
  int n = 0;
  __device__ __forceinline__ int op(int i) const { return (ops >> (4 * i)) & 15; }
};

__device__ __forceinline__ EpiProg make_prog(const EpilogueParams& e) {
  EpiProg g;
#pragma unroll
  for (int i = 0; i < kMaxEpi; ++i)
    g.ops |= static_cast<uint32_t>(i < e.n_ops ? e.ops[i] : 0) << (4 * i);
  g.n = e.n_ops;
  return g;
}

// requantize (int8 graphs, elementwise.cu states the semantics): int64
// product (|t| < 2^31, m < 2^31: exact), round half up, clamp to i8.
__device__ __forceinline__ int64_t requant(int64_t t, int64_t m, int s) {
  t *= m;
  if (s > 0) t = (t + (int64_t(1) << (s - 1))) >> s;
  return t < -128 ? -128 : (t > 127 ? 127 : t);
}

// 32 elements as raw 32-bit words: bf16 pairs packed (16 words) or f32/i32.
__device__ __forceinline__ float bf16_lo(uint32_t w) { return __uint_as_float(w << 16); }
__device__ __forceinline__ float bf16_hi(uint32_t w) { return __uint_as_float(w & 0xFFFF0000u); }
__device__ __forceinline__ float word_elem_f(const uint32_t (&w)[kChunk], bool bf, int j) {
  if (bf) return (j & 1) ? bf16_hi(w[j >> 1]) : bf16_lo(w[j >> 1]);
  return __uint_as_float(w[j]);
}
__device__ __forceinline__ uint32_t pack_bf16x2(float a, float b) {
  const __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<const uint32_t*>(&h);
}

// Explicit shared-space accesses (the stage pointers are carved out of the
// dynamic smem block; generic addressing would cost an extra conversion).
__device__ __forceinline__ void sts128(uint32_t addr, uint4 v) {
  asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "r"(v.x), "r"(v.y),
               "r"(v.z), "r"(v.w)
               : "memory");
}
__device__ __forceinline__ uint4 lds128(uint32_t addr) {
  uint4 v;
  asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "r"(addr)
               : "memory");
  return v;
}
// 32 bias words from shared memory (broadcast reads).
__device__ __forceinline__ void load_bias32(const uint32_t* bias_s, uint32_t (&b)[kChunk]) {
  const uint32_t a = smem_u32(bias_s);
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const uint4 v = lds128(a + 16 * i);
    b[4 * i] = v.x; b[4 * i + 1] = v.y; b[4 * i + 2] = v.z; b[4 * i + 3] = v.w;
  }
}

// Float member chain on 32 values (v) of one row. opnd_fn(op) must leave
// the same-shape operand of `op` (add / mul) in `opnd`.
template <typename OpndFn>
__device__ __forceinline__ void apply_float(const EpiProg& g, const EpilogueParams& e,
                                            float (&v)[kChunk],
                                            const uint32_t* bias_s, bool bf,
                                            uint32_t (&opnd)[kChunk], OpndFn opnd_fn) {
#pragma unroll 1
  for (int i = 0; i < g.n; ++i) {
    const int op = g.op(i);
    if (op == kEpiScale) {
      const float s = e.fscale[i];
#pragma unroll
      for (int j = 0; j < kChunk; ++j) v[j] = __fmul_rn(v[j], s);
    } else if (op == kEpiBias) {
      uint32_t b[kChunk];
      load_bias32(bias_s, b);
#pragma unroll
      for (int j = 0; j < kChunk; ++j) v[j] = __fadd_rn(v[j], __uint_as_float(b[j]));
    } else if (op == kEpiAdd) {
      opnd_fn(kEpiAdd);
#pragma unroll
      for (int j = 0; j < kChunk; ++j) v[j] = __fadd_rn(v[j], word_elem_f(opnd, bf, j));
    } else if (op == kEpiMul) {
      opnd_fn(kEpiMul);
#pragma unroll
      for (int j = 0; j < kChunk; ++j) v[j] = __fmul_rn(v[j], word_elem_f(opnd, bf, j));
    } else if (op == kEpiRelu) {
#pragma unroll
      for (int j = 0; j < kChunk; ++j) v[j] = (v[j] < 0.0f) ? 0.0f : v[j];  // std::max(x, 0)
    }
  }
}

// Integer member chain: every member in int64, range-checked, stored back as
// i32 (after an overflow the kernel reports FoldOverflow -- the reference
// throws -- so the wrapped value is never consumed).
template <typename OpndFn>
__device__ __forceinline__ bool apply_int(const EpiProg& g, const EpilogueParams& e,
                                          uint32_t (&acc)[kChunk],
                                          const uint32_t* bias_s, int ncols, bool live,
                                          uint32_t (&opnd)[kChunk], OpndFn opnd_fn) {
  bool ovf = false;
#pragma unroll 1
  for (int i = 0; i < g.n; ++i) {
    const int op = g.op(i);
    if (op == kEpiAdd || op == kEpiMul) opnd_fn(op);
    uint32_t b[kChunk];
    if (op == kEpiBias) load_bias32(bias_s, b);
    const int64_t s = op == kEpiScale ? e.iscale[i] : 1;
    // i8 residual (res_i8): 4 packed bytes per operand word, entering as
    // scale(cast(r, i32), res_scale) -- |res_scale| <= 2^24, no overflow
    const bool r8 = op == kEpiAdd && e.res_i8;
    if (op == kEpiBias || op == kEpiAdd) {
      // 32-bit adds with an explicit signed-overflow bit ((a^s) & (b^s) < 0)
      const int32_t rs = static_cast<int32_t>(e.res_scale);  // |rs| <= 2^24
      uint32_t bits = 0u;
#pragma unroll
      for (int j = 0; j < kChunk; ++j) {
        const int32_t a = static_cast<int32_t>(acc[j]);
        const int32_t o = op == kEpiBias ? static_cast<int32_t>(b[j])
                          : r8 ? static_cast<int32_t>(static_cast<int8_t>(opnd[j >> 2] >> (8 * (j & 3)))) * rs
                               : static_cast<int32_t>(opnd[j]);
        const uint32_t x = static_cast<uint32_t>(a) + static_cast<uint32_t>(o);
        if (j < ncols) bits |= (static_cast<uint32_t>(a) ^ x) & (static_cast<uint32_t>(o) ^ x);
        acc[j] = x;
      }
      ovf |= live && (bits >> 31);
      continue;
    }
    if (op == kEpiRelu) {
#pragma unroll
      for (int j = 0; j < kChunk; ++j) {
        const int32_t a = static_cast<int32_t>(acc[j]);
        acc[j] = static_cast<uint32_t>(a < 0 ? 0 : a);
      }
      continue;
    }
#pragma unroll
    for (int j = 0; j < kChunk; ++j) {
      int64_t t = static_cast<int32_t>(acc[j]);
      if (op == kEpiScale) t *= s;
      else if (op == kEpiMul) t *= static_cast<int32_t>(opnd[j]);
      else if (op == kEpiRequant) t = requant(t, e.rq_mult, e.rq_shift);
      ovf |= live && (j < ncols) && (t < INT32_MIN || t > INT32_MAX);
      acc[j] = static_cast<uint32_t>(static_cast<int32_t>(t));
    }
  }
  return ovf;
}

// 32 i8 results (values already in [-128, 127]) packed 4 per word.
__device__ __forceinline__ void pack_i8x32(const uint32_t (&v)[kChunk], uint32_t (&w)[kChunk]) {
#pragma unroll
  for (int k = 0; k < kChunk / 4; ++k)
    w[k] = (v[4 * k] & 0xFFu) | ((v[4 * k + 1] & 0xFFu) << 8) | ((v[4 * k + 2] & 0xFFu) << 16) |
           ((v[4 * k + 3] & 0xFFu) << 24);
#pragma unroll
  for (int k = kChunk / 4; k < kChunk; ++k) w[k] = 0u;
}

// ------------------------------------------------- per-thread fallback
__device__ __forceinline__ void fetch_row32(const void* base, int64_t off, int es, int ncols,
                                            uint32_t (&w)[kChunk]) {
  if (es == 2) {
    const uint16_t* h = static_cast<const uint16_t*>(base) + off;
#pragma unroll
    for (int j = 0; j < kChunk / 2; ++j) {
      const uint32_t lo = 2 * j < ncols ? h[2 * j] : 0u;
      const uint32_t hi = 2 * j + 1 < ncols ? h[2 * j + 1] : 0u;
      w[j] = lo | (hi << 16);
    }
  } else {
    const uint32_t* s = static_cast<const uint32_t*>(base) + off;
#pragma unroll
    for (int j = 0; j < kChunk; ++j) w[j] = j < ncols ? s[j] : 0u;
  }
}

// One row, 32 columns (any channel count). Waits on the pending TMEM load.
template <bool kInt, typename P>
__device__ __forceinline__ void epi_row_chunk(const P& p, const EpiProg& g, int64_t row,
                                              int col0, int ncols, bool active,
                                              const uint32_t* bias_s, uint32_t (&acc)[kChunk],
                                              bool* overflow) {
  tmem_ld_wait();
  if (!active) return;
  const EpilogueParams& e = p.epi;
  const int64_t base = row * p.oc + col0;
  const bool bf = !kInt && p.out_type == kBF16;
  const int es = bf ? 2 : 4;
  uint32_t opnd[kChunk];
  auto opnd_fn = [&](int op) {
    fetch_row32(op == kEpiAdd ? e.residual : e.mul_operand, base, es, ncols, opnd);
  };
  if constexpr (kInt) {
    if (apply_int(g, e, acc, bias_s, ncols, true, opnd, opnd_fn)) *overflow = true;
    int32_t* yp = static_cast<int32_t*>(p.y) + base;
#pragma unroll
    for (int j = 0; j < kChunk; ++j)
      if (j < ncols) yp[j] = static_cast<int32_t>(acc[j]);
  } else {
    float v[kChunk];
#pragma unroll
    for (int j = 0; j < kChunk; ++j) v[j] = __uint_as_float(acc[j]);
    apply_float(g, e, v, bias_s, bf, opnd, opnd_fn);
    if (bf) {
      __nv_bfloat16* yp = static_cast<__nv_bfloat16*>(p.y) + base;
#pragma unroll
      for (int j = 0; j < kChunk; ++j)
        if (j < ncols) yp[j] = __float2bfloat16_rn(v[j]);
    } else {
      float* yp = static_cast<float*>(p.y) + base;
#pragma unroll
      for (int j = 0; j < kChunk; ++j)
        if (j < ncols) yp[j] = v[j];
    }
  }
}

// ------------------------------------------- warp-cooperative, coalesced
// Stage layout: row r of the 32 x (32 * es) block at r * rowbytes, 16-byte
// chunks XOR-swizzled by their 128-byte line index (conflict-free for both
// the row-per-thread writes and the line-per-lanes reads). Rows are given
// per lane (my_row = global output row of this lane, -1 = junk/padding)
// and exchanged with shuffles.
__device__ __forceinline__ uint32_t stage_off(int row, int chunk, int rowbytes) {
  const uint32_t lin = static_cast<uint32_t>(row * rowbytes + chunk * 16);
  return lin ^ (((lin >> 7) & 7u) << 4);
}

__device__ __forceinline__ void coalesced_load_block(const void* src, int es, int64_t oc,
                                                     int col0, int ncols, int lane, int my_row,
                                                     uint8_t* stage, uint32_t (&w)[kChunk]) {
  const int rowbytes = 32 * es, cpr = rowbytes / 16, rpi = 32 / cpr;
  const uint32_t sbase = smem_u32(stage);
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    if (i >= cpr) break;
    const int r = i * rpi + lane / cpr;
    const int c = lane % cpr;
    const int g = __shfl_sync(0xffffffffu, my_row, r);
    uint4 v = make_uint4(0, 0, 0, 0);
    const int cc = c * (16 / es);
    if (g >= 0 && cc < ncols)
      v = __ldg(reinterpret_cast<const uint4*>(static_cast<const uint8_t*>(src) +
                                               (static_cast<int64_t>(g) * oc + col0 + cc) * es));
    sts128(sbase + stage_off(r, c, rowbytes), v);
  }
  __syncwarp();
#pragma unroll
  for (int c = 0; c < 8; ++c) {
    if (c < cpr) {
      const uint4 v = lds128(sbase + stage_off(lane, c, rowbytes));
      w[4 * c] = v.x; w[4 * c + 1] = v.y; w[4 * c + 2] = v.z; w[4 * c + 3] = v.w;
    }
  }
  __syncwarp();
}

__device__ __forceinline__ void coalesced_store_block(void* dst, int es, int64_t oc, int col0,
                                                      int ncols, int lane, int my_row,
                                                      uint8_t* stage, const uint32_t (&w)[kChunk]) {
  const int rowbytes = 32 * es, cpr = rowbytes / 16, rpi = 32 / cpr;
  const uint32_t sbase = smem_u32(stage);
#pragma unroll
  for (int c = 0; c < 8; ++c)
    if (c < cpr)
      sts128(sbase + stage_off(lane, c, rowbytes),
             make_uint4(w[4 * c], w[4 * c + 1], w[4 * c + 2], w[4 * c + 3]));
  __syncwarp();
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    if (i >= cpr) break;
    const int r = i * rpi + lane / cpr;
    const int c = lane % cpr;
    const int g = __shfl_sync(0xffffffffu, my_row, r);
    const int cc = c * (16 / es);
    const uint4 v = lds128(sbase + stage_off(r, c, rowbytes));
    if (g >= 0 && cc < ncols)
      *reinterpret_cast<uint4*>(static_cast<uint8_t*>(dst) +
                                (static_cast<int64_t>(g) * oc + col0 + cc) * es) = v;
  }
  __syncwarp();
}

// One 32-column block of one warp. taddr: TMEM address of this warp's lane
// quadrant at the block's first accumulator column; col0: global column;
// bias_s: the block's 32 bias values (raw f32/i32 bits) in shared memory.
// Requires oc % (16 / out_bytes) == 0 (whole 16-byte chunks per row).
template <bool kInt, typename P>
__device__ __forceinline__ void epi_warp_block(const P& p, const EpiProg& g, uint32_t taddr,
                                               int col0, int lane, int my_row,
                                               const uint32_t* bias_s, uint8_t* stage,
                                               bool* overflow, long long* prof = nullptr) {
  const long long t0 = prof ? clock64() : 0;
  const EpilogueParams& e = p.epi;
  const bool bf = !kInt && p.out_type == kBF16;
  const bool i8_out = kInt && p.out_type == kI8;  // requantize member (host-checked)
  const int es = bf ? 2 : (i8_out ? 1 : 4);
  const int ncols = min(kChunk, p.oc - col0);
  // operand element bytes: the output's, or 1 for an i8 residual (res_i8)
  auto opnd_es = [&](int op) { return kInt && op == kEpiAdd && e.res_i8 ? 1 : (kInt ? 4 : es); };
  // One operand buffer: the first same-shape operand in member order is
  // fetched before waiting on TMEM; any later one is fetched on demand.
  uint32_t opnd[kChunk];
  int have = 0;
  const int first =
      e.residual && !e.mul_operand ? kEpiAdd : (!e.residual && e.mul_operand ? kEpiMul : 0);
  uint32_t acc[kChunk];
  tmem_ld32(taddr, acc);
  if (first) {
    coalesced_load_block(first == kEpiAdd ? e.residual : e.mul_operand, opnd_es(first), p.oc,
                         col0, ncols, lane, my_row, stage, opnd);
    have = first;
  }
  auto opnd_fn = [&](int op) {
    if (have != op) {
      coalesced_load_block(op == kEpiAdd ? e.residual : e.mul_operand, opnd_es(op), p.oc, col0,
                           ncols, lane, my_row, stage, opnd);
      have = op;
    }
  };
  tmem_ld_wait();
  const long long t1 = prof ? clock64() : 0;
  uint32_t out[kChunk];
  if constexpr (kInt) {
    if (apply_int(g, e, acc, bias_s, ncols, my_row >= 0, opnd, opnd_fn)) *overflow = true;
    if (i8_out) {
      pack_i8x32(acc, out);
    } else {
#pragma unroll
      for (int j = 0; j < kChunk; ++j) out[j] = acc[j];
    }
  } else {
    float v[kChunk];
#pragma unroll
    for (int j = 0; j < kChunk; ++j) v[j] = __uint_as_float(acc[j]);
    apply_float(g, e, v, bias_s, bf, opnd, opnd_fn);
    if (bf) {
#pragma unroll
      for (int j = 0; j < kChunk / 2; ++j) out[j] = pack_bf16x2(v[2 * j], v[2 * j + 1]);
#pragma unroll
      for (int j = kChunk / 2; j < kChunk; ++j) out[j] = 0u;
    } else {
#pragma unroll
      for (int j = 0; j < kChunk; ++j) out[j] = __float_as_uint(v[j]);
    }
  }
  const long long t2 = prof ? clock64() : 0;
  coalesced_store_block(p.y, es, p.oc, col0, ncols, lane, my_row, stage, out);
  if (prof) {
    prof[0] += t1 - t0;          // operand prefetch + TMEM load
    prof[1] += t2 - t1;          // member ops
    prof[2] += clock64() - t2;   // transpose + global stores
  }
}

// ------------------------------------------- specialised fast path
// The member programs fuse_pass produces for the benchmark networks, fixed
// at compile time so a block is ~100 instructions: no op decoding, no
// partial-block predicates (full 32-column block, oc % 8 == 0).
// The int8-graph programs end in requantize and store i8 (ES = 1):
// kProgBiasReluQ [bias, relu, requantize], kProgBiasAddReluQ [bias,
// add(i8 residual, scaled), relu, requantize], kProgBiasQ [bias,
// requantize] (the downsample branch).
enum FastProg : int { kProgGeneric = 0, kProgNone = 1, kProgBias = 2, kProgBiasRelu = 3,
                      kProgBiasAddRelu = 4, kProgBiasReluQ = 5, kProgBiasAddReluQ = 6,
                      kProgBiasQ = 7 };

__device__ __forceinline__ int classify_prog(const EpilogueParams& e) {
  if (e.n_ops == 0) return kProgNone;
  if (e.n_ops == 1 && e.ops[0] == kEpiBias) return kProgBias;
  if (e.n_ops == 2 && e.ops[0] == kEpiBias && e.ops[1] == kEpiRelu) return kProgBiasRelu;
  if (e.n_ops == 3 && e.ops[0] == kEpiBias && e.ops[1] == kEpiAdd && e.ops[2] == kEpiRelu &&
      !e.res_i8)
    return kProgBiasAddRelu;
  if (e.n_ops == 3 && e.ops[0] == kEpiBias && e.ops[1] == kEpiRelu && e.ops[2] == kEpiRequant)
    return kProgBiasReluQ;
  if (e.n_ops == 2 && e.ops[0] == kEpiBias && e.ops[1] == kEpiRequant) return kProgBiasQ;
  if (e.n_ops == 4 && e.ops[0] == kEpiBias && e.ops[1] == kEpiAdd && e.ops[2] == kEpiRelu &&
      e.ops[3] == kEpiRequant && e.res_i8)
    return kProgBiasAddReluQ;
  return kProgGeneric;
}

// Fast float block. es = 2 (bf16) or 4 (f32) output bytes; `oc_es` = row
// pitch in bytes; `ybase` = output base + col0 * es.
template <int PROG, int ES>
__device__ __forceinline__ void epi_block_fast(uint8_t* ybase, const uint8_t* rbase,
                                               int64_t oc_es, uint32_t taddr, int lane,
                                               int my_row, const uint32_t* bias_s,
                                               uint32_t sbase) {
  constexpr int kRowBytes = 32 * ES, kCpr = kRowBytes / 16, kRpi = 32 / kCpr;
  uint32_t acc[kChunk];
  tmem_ld32(taddr, acc);
  uint32_t res[kChunk];
  if constexpr (PROG == kProgBiasAddRelu) {
    // coalesced residual read through the stage (same transposition)
#pragma unroll
    for (int i = 0; i < kCpr; ++i) {
      const int r = i * kRpi + lane / kCpr, c = lane % kCpr;
      const int g = __shfl_sync(0xffffffffu, my_row, r);
      uint4 v = make_uint4(0, 0, 0, 0);
      if (g >= 0) v = __ldg(reinterpret_cast<const uint4*>(rbase + g * oc_es + c * 16));
      sts128(sbase + stage_off(r, c, kRowBytes), v);
    }
    __syncwarp();
#pragma unroll
    for (int c = 0; c < kCpr; ++c) {
      const uint4 v = lds128(sbase + stage_off(lane, c, kRowBytes));
      res[4 * c] = v.x; res[4 * c + 1] = v.y; res[4 * c + 2] = v.z; res[4 * c + 3] = v.w;
    }
    __syncwarp();
  }
  uint32_t b[kChunk];
  if constexpr (PROG != kProgNone) load_bias32(bias_s, b);
  tmem_ld_wait();
  float v[kChunk];
#pragma unroll
  for (int j = 0; j < kChunk; ++j) {
    float x = __uint_as_float(acc[j]);
    if constexpr (PROG != kProgNone) x = __fadd_rn(x, __uint_as_float(b[j]));
    if constexpr (PROG == kProgBiasAddRelu)
      x = __fadd_rn(x, ES == 2 ? ((j & 1) ? bf16_hi(res[j >> 1]) : bf16_lo(res[j >> 1]))
                               : __uint_as_float(res[j]));
    if constexpr (PROG == kProgBiasRelu || PROG == kProgBiasAddRelu) x = (x < 0.0f) ? 0.0f : x;
    v[j] = x;
  }
  uint32_t out[kChunk];
  if constexpr (ES == 2) {
#pragma unroll
    for (int j = 0; j < kChunk / 2; ++j) out[j] = pack_bf16x2(v[2 * j], v[2 * j + 1]);
  } else {
#pragma unroll
    for (int j = 0; j < kChunk; ++j) out[j] = __float_as_uint(v[j]);
  }
#pragma unroll
  for (int c = 0; c < kCpr; ++c)
    sts128(sbase + stage_off(lane, c, kRowBytes),
           make_uint4(out[4 * c], out[4 * c + 1], out[4 * c + 2], out[4 * c + 3]));
  __syncwarp();
#pragma unroll
  for (int i = 0; i < kCpr; ++i) {
    const int r = i * kRpi + lane / kCpr, c = lane % kCpr;
    const int g = __shfl_sync(0xffffffffu, my_row, r);
    const uint4 val = lds128(sbase + stage_off(r, c, kRowBytes));
    if (g >= 0) *reinterpret_cast<uint4*>(ybase + g * oc_es + c * 16) = val;
  }
  __syncwarp();
}

// Dispatch one 32-column block: fast path when possible, generic otherwise.
template <bool kInt, typename P>
__device__ __forceinline__ void epi_block(const P& p, const EpiProg& g, int prog, uint32_t taddr,
                                          int col0, int lane, int my_row,
                                          const uint32_t* bias_s, uint8_t* stage,
                                          bool* overflow) {
  const bool full = col0 + kChunk <= p.oc;
  if (!kInt && full && prog != kProgGeneric) {
    const uint32_t sbase = smem_u32(stage);
    const int es = p.out_type == kBF16 ? 2 : 4;
    uint8_t* yb = static_cast<uint8_t*>(p.y) + static_cast<int64_t>(col0) * es;
    const uint8_t* rb = static_cast<const uint8_t*>(p.epi.residual) + static_cast<int64_t>(col0) * es;
    const int64_t oc_es = static_cast<int64_t>(p.oc) * es;
    if (es == 2) {
      switch (prog) {
        case kProgNone: epi_block_fast<kProgNone, 2>(yb, rb, oc_es, taddr, lane, my_row, bias_s, sbase); return;
        case kProgBias: epi_block_fast<kProgBias, 2>(yb, rb, oc_es, taddr, lane, my_row, bias_s, sbase); return;
        case kProgBiasRelu: epi_block_fast<kProgBiasRelu, 2>(yb, rb, oc_es, taddr, lane, my_row, bias_s, sbase); return;
        default: epi_block_fast<kProgBiasAddRelu, 2>(yb, rb, oc_es, taddr, lane, my_row, bias_s, sbase); return;
      }
    } else {
      switch (prog) {
        case kProgNone: epi_block_fast<kProgNone, 4>(yb, rb, oc_es, taddr, lane, my_row, bias_s, sbase); return;
        case kProgBias: epi_block_fast<kProgBias, 4>(yb, rb, oc_es, taddr, lane, my_row, bias_s, sbase); return;
        case kProgBiasRelu: epi_block_fast<kProgBiasRelu, 4>(yb, rb, oc_es, taddr, lane, my_row, bias_s, sbase); return;
        default: epi_block_fast<kProgBiasAddRelu, 4>(yb, rb, oc_es, taddr, lane, my_row, bias_s, sbase); return;
      }
    }
  }
  epi_warp_block<kInt>(p, g, taddr, col0, lane, my_row, bias_s, stage, overflow);
}

// ---------------------------------------------------- TMA-store epilogue
// For the fast programs (none / bias / bias+relu) the block goes TMEM ->
// registers -> output dtype -> a swizzled 32-row x 32-column shared-memory
// box, and ONE lane stores the box with cp.async.bulk.tensor: no address
// math, shuffles or predicated global stores per element, and the tensor
// map clips rows/columns outside the output (M tail, OC tail, the halo
// kernel's junk virtual rows) for free.
//
// Box rows are 32 * ES bytes; 16-byte chunks are placed exactly as the
// tensor map's swizzle expects: bf16 SWIZZLE_64B (chunk c of row r at
// c ^ ((r >> 1) & 3)), f32 SWIZZLE_128B (c ^ (r & 7)). Both are
// bank-conflict free for the one-row-per-lane writes.
template <int ES>
__device__ __forceinline__ uint32_t box_off(int row, int chunk) {
  if constexpr (ES == 1)  // i8 rows of 32 B, SWIZZLE_32B: chunk ^ address bit 7
    return static_cast<uint32_t>(row * 32 + ((chunk ^ ((row >> 2) & 1)) << 4));
  else if constexpr (ES == 2)
    return static_cast<uint32_t>(row * 64 + ((chunk ^ ((row >> 1) & 3)) << 4));
  else
    return static_cast<uint32_t>(row * 128 + ((chunk ^ (row & 7)) << 4));
}

// kInt: the int8 path -- s32 accumulator + i32 bias in int64 with the
// reference's i32 range check per member (DenseTensor::set_i,
// R/include/tec/tensor.hpp:63-69); sets *ovf, stores i32 (ES == 4).
// acc: this lane's row, 32 accumulator columns (raw f32 / s32 bits).
// Residual operand of kProgBiasAddRelu (float kinds): the warp's 32 rows x
// 32 columns of the output-shaped NHWC operand, read COALESCED (each load
// instruction covers kRpi whole 32-column row segments) into this block's
// output box -- the same swizzled slots the results go to -- and handed to
// each lane as its own row. rrow = this lane's row (already offset to the
// block's first column) or NULL for a row that is not stored (zeros).
template <int ES>
__device__ __forceinline__ void load_res_box(const uint8_t* rrow, int lane, uint32_t box,
                                             uint32_t (&res)[kChunk]) {
  constexpr int kCpr = 32 * ES / 16, kRpi = 32 / kCpr;
#pragma unroll
  for (int i = 0; i < kCpr; ++i) {
    const int r = i * kRpi + lane / kCpr, c = lane % kCpr;
    const uint8_t* src = reinterpret_cast<const uint8_t*>(__shfl_sync(
        0xffffffffu, reinterpret_cast<unsigned long long>(rrow), r));
    uint4 v = make_uint4(0, 0, 0, 0);
    if (src) v = __ldg(reinterpret_cast<const uint4*>(src) + c);
    sts128(box + box_off<ES>(r, c), v);
  }
  __syncwarp();
#pragma unroll
  for (int c = 0; c < kCpr; ++c) {
    const uint4 v = lds128(box + box_off<ES>(lane, c));
    res[4 * c] = v.x; res[4 * c + 1] = v.y; res[4 * c + 2] = v.z; res[4 * c + 3] = v.w;
  }
}

// Requantize parameters of the Q programs (EpilogueParams fields).
struct QParams {
  int64_t mult = 1;
  int32_t shift = 0;
  int64_t res_scale = 1;
};

template <int PROG, int ES, bool kInt = false>
__device__ __forceinline__ void epi_acc_to_box(uint32_t (&acc)[kChunk], int lane,
                                               const uint32_t* bias_s, uint32_t box,
                                               bool* ovf = nullptr,
                                               const uint8_t* rrow = nullptr,
                                               const QParams& qp = QParams{}) {
  static_assert(!(kInt && PROG == kProgBiasAddRelu), "int residual programs use the SIMT path");
  if constexpr (PROG == kProgBiasReluQ || PROG == kProgBiasAddReluQ || PROG == kProgBiasQ) {
    // int8 graphs: bias -> (+ i8 residual * res_scale) -> relu -> requantize,
    // each integer member range-checked (as apply_int does in int64); 32 i8
    // results = this lane's 32-byte box row.
    static_assert(kInt && ES == 1, "the Q programs store i8");
    uint32_t res[kChunk];
    if constexpr (PROG == kProgBiasAddReluQ) load_res_box<1>(rrow, lane, box, res);
    uint32_t b[kChunk];
    load_bias32(bias_s, b);
    // 32-bit arithmetic with explicit overflow bits (the int64 form of
    // apply_int costs ~3x the instructions, and the epilogue is issue-bound
    // at i8 output): signed a + b overflows iff (a ^ s) & (b ^ s) < 0.
    uint32_t ovf_bits = 0u;
    const uint32_t m = static_cast<uint32_t>(qp.mult);  // 1 <= m < 2^31 (host-checked)
    const int sh = qp.shift;
    const uint64_t half = sh > 0 ? (uint64_t(1) << (sh - 1)) : 0u;
    // requantize of x >= 0 as one 32 x 32 high product when m < 2^sh <= 2^32:
    // (x*m + 2^(sh-1)) >> sh == hi32(x * m' + 2^31) with m' = m << (32 - sh),
    // exact (x < 2^31, m' < 2^32); the carry of the low half adds the rounding
    const bool hi_form = sh >= 1 && sh <= 32 && (static_cast<uint64_t>(m) >> sh) == 0;
    const uint32_t mp = hi_form ? static_cast<uint32_t>(static_cast<uint64_t>(m) << (32 - sh)) : 0u;
    const int32_t rs = static_cast<int32_t>(qp.res_scale);  // |rs| <= 2^24: r * rs fits i32
    uint32_t w[kChunk / 4];
#pragma unroll
    for (int k = 0; k < kChunk / 4; ++k) w[k] = 0u;
#pragma unroll
    for (int j = 0; j < kChunk; ++j) {
      const int32_t a = static_cast<int32_t>(acc[j]), bj = static_cast<int32_t>(b[j]);
      int32_t x = static_cast<int32_t>(static_cast<uint32_t>(a) + static_cast<uint32_t>(bj));
      ovf_bits |= static_cast<uint32_t>((a ^ x) & (bj ^ x));
      if constexpr (PROG == kProgBiasAddReluQ) {
        const int32_t r = static_cast<int32_t>(static_cast<int8_t>(res[j >> 2] >> (8 * (j & 3)))) * rs;
        const int32_t x2 = static_cast<int32_t>(static_cast<uint32_t>(x) + static_cast<uint32_t>(r));
        ovf_bits |= static_cast<uint32_t>((x ^ x2) & (r ^ x2));
        x = x2;
      }
      uint32_t q;
      if constexpr (PROG != kProgBiasQ) {
        // after relu x >= 0
        const uint32_t xu = static_cast<uint32_t>(x < 0 ? 0 : x);
        if (hi_form) {
          const uint32_t lo = xu * mp;
          const uint32_t v = __umulhi(xu, mp) + (lo >> 31);
          q = v > 127u ? 127u : v;
        } else {  // an unsigned 32 x 32 -> 64 product
          const uint64_t t = static_cast<uint64_t>(xu) * m + half;
          const uint64_t v = t >> sh;
          q = v > 127u ? 127u : static_cast<uint32_t>(v);
        }
      } else {
        const int64_t t = static_cast<int64_t>(x) * static_cast<int64_t>(static_cast<int32_t>(m)) +
                          static_cast<int64_t>(half);
        const int64_t v = t >> sh;  // arithmetic: floor
        q = static_cast<uint32_t>(static_cast<int32_t>(v < -128 ? -128 : (v > 127 ? 127 : v)));
      }
      w[j >> 2] |= (q & 0xFFu) << (8 * (j & 3));
    }
    if ((ovf_bits >> 31) && ovf) *ovf = true;
    sts128(box + box_off<1>(lane, 0), make_uint4(w[0], w[1], w[2], w[3]));
    sts128(box + box_off<1>(lane, 1), make_uint4(w[4], w[5], w[6], w[7]));
    return;
  }
  uint32_t res[kChunk];
  if constexpr (PROG == kProgBiasAddRelu) load_res_box<ES>(rrow, lane, box, res);
  uint32_t b[kChunk];
  if constexpr (PROG != kProgNone) load_bias32(bias_s, b);
  if constexpr (kInt) {
    static_assert(ES == 4 || PROG == kProgBiasReluQ || PROG == kProgBiasAddReluQ || PROG == kProgBiasQ,
                  "int8 conv stores i32 (i8 only through the Q programs above)");
    // 32-bit adds with an explicit signed-overflow bit, (a ^ s) & (b ^ s) < 0
    // (the int64 form costs ~2x the instructions in an issue-bound epilogue)
    uint32_t bits = 0u;
#pragma unroll
    for (int j = 0; j < kChunk; ++j) {
      uint32_t x = acc[j];
      if constexpr (PROG != kProgNone) {
        const uint32_t a = acc[j];
        x = a + b[j];
        bits |= (a ^ x) & (b[j] ^ x);
      }
      if constexpr (PROG == kProgBiasRelu) {
        const int32_t xi = static_cast<int32_t>(x);
        x = static_cast<uint32_t>(xi < 0 ? 0 : xi);
      }
      acc[j] = x;
    }
    if ((bits >> 31) && ovf) *ovf = true;
#pragma unroll
    for (int c = 0; c < 8; ++c)
      sts128(box + box_off<4>(lane, c),
             make_uint4(acc[4 * c], acc[4 * c + 1], acc[4 * c + 2], acc[4 * c + 3]));
    return;
  }
  float v[kChunk];
#pragma unroll
  for (int j = 0; j < kChunk; ++j) {
    float x = __uint_as_float(acc[j]);
    if constexpr (PROG != kProgNone) x = __fadd_rn(x, __uint_as_float(b[j]));
    if constexpr (PROG == kProgBiasAddRelu)  // R/src/ops.cpp:216-223, member order
      x = __fadd_rn(x, ES == 2 ? ((j & 1) ? bf16_hi(res[j >> 1]) : bf16_lo(res[j >> 1]))
                               : __uint_as_float(res[j]));
    if constexpr (PROG == kProgBiasRelu || PROG == kProgBiasAddRelu) x = (x < 0.0f) ? 0.0f : x;
    v[j] = x;
  }
  constexpr int kCpr = 32 * ES / 16;
  if constexpr (ES == 2) {
#pragma unroll
    for (int c = 0; c < kCpr; ++c)
      sts128(box + box_off<2>(lane, c),
             make_uint4(pack_bf16x2(v[8 * c], v[8 * c + 1]), pack_bf16x2(v[8 * c + 2], v[8 * c + 3]),
                        pack_bf16x2(v[8 * c + 4], v[8 * c + 5]),
                        pack_bf16x2(v[8 * c + 6], v[8 * c + 7])));
  } else {
#pragma unroll
    for (int c = 0; c < kCpr; ++c)
      sts128(box + box_off<4>(lane, c),
             make_uint4(__float_as_uint(v[4 * c]), __float_as_uint(v[4 * c + 1]),
                        __float_as_uint(v[4 * c + 2]), __float_as_uint(v[4 * c + 3])));
  }
}

// One row of a box (the paired-tap halo kernel's last row per warp), one
// column per lane (j = lane): v = lo + hi_next (f32, NULL hi = 0), then the
// program (bias, residual from global, relu) into row `row` of `box`.
template <int PROG, int ES>
__device__ __forceinline__ void row_col_to_box(const float* lo, const float* hi_next,
                                               const uint32_t* bias_s, const uint8_t* rrow,
                                               uint32_t box, int row, int j) {
  float x = __fadd_rn(lo[j], hi_next ? hi_next[j] : 0.0f);
  if constexpr (PROG != kProgNone) x = __fadd_rn(x, __uint_as_float(bias_s[j]));
  if constexpr (PROG == kProgBiasAddRelu) {
    float r = 0.0f;
    if (rrow) {
      if constexpr (ES == 2)
        r = __bfloat162float(reinterpret_cast<const __nv_bfloat16*>(rrow)[j]);
      else
        r = reinterpret_cast<const float*>(rrow)[j];
    }
    x = __fadd_rn(x, r);
  }
  if constexpr (PROG == kProgBiasRelu || PROG == kProgBiasAddRelu) x = (x < 0.0f) ? 0.0f : x;
  const uint32_t a = box + box_off<ES>(row, (j * ES) >> 4) + ((j * ES) & 15);
  if constexpr (ES == 2) {
    const unsigned short h = __bfloat16_as_ushort(__float2bfloat16_rn(x));
    asm volatile("st.shared.u16 [%0], %1;" ::"r"(a), "h"(h) : "memory");
  } else {
    asm volatile("st.shared.f32 [%0], %1;" ::"r"(a), "f"(x) : "memory");
  }
}

template <int PROG, int ES, bool kInt = false>
__device__ __forceinline__ void epi_block_box(uint32_t taddr, int lane, const uint32_t* bias_s,
                                              uint32_t box, bool* ovf = nullptr,
                                              const uint8_t* rrow = nullptr,
                                              const QParams& qp = QParams{}) {
  uint32_t acc[kChunk];
  tmem_ld32(taddr, acc);
  tmem_ld_wait();
  epi_acc_to_box<PROG, ES, kInt>(acc, lane, bias_s, box, ovf, rrow, qp);
}

// One warp's 32 accumulator rows x BN columns through the TMA-store path.
// `stage` = this warp's 4 KB (2 bf16 boxes / 1 f32 box, used as a ring;
// `cnt` counts boxes across calls). `store(box, c0)` runs on lane 0 and
// issues the TMA store(s) of the box holding columns [c0, c0 + 32).
// `src(c0, acc)` fills this lane's 32 accumulator columns starting at c0
// (TMEM, or the split-K partial sums).
template <int PROG, int ES, int BN, bool kInt, typename SrcFn, typename StoreFn>
__device__ __forceinline__ void epi_rows_tma_src(SrcFn&& src, int lane, const uint32_t* bias_s,
                                                 uint32_t stage, int valid_cols, uint32_t& cnt,
                                                 bool* ovf, StoreFn&& store,
                                                 const uint8_t* rrow = nullptr,
                                                 const QParams& qp = QParams{}) {
  constexpr uint32_t kBox = 32 * 32 * ES;
  constexpr uint32_t kSlots = 4096 / kBox;
#pragma unroll 1
  for (int c0 = 0; c0 < BN && c0 < valid_cols; c0 += kChunk) {
    const uint32_t box = stage + (cnt % kSlots) * kBox;
    uint32_t acc[kChunk];
    src(c0, acc);
    if (lane == 0) bulk_wait_read<kSlots - 1>();  // the box's previous store has read it
    __syncwarp();
    epi_acc_to_box<PROG, ES, kInt>(acc, lane, bias_s + c0, box, ovf,
                                   rrow ? rrow + c0 * ES : nullptr, qp);
    fence_proxy_async_smem();
    __syncwarp();
    if (lane == 0) {
      store(box, c0);
      bulk_commit();
    }
    ++cnt;
  }
}

template <int PROG, int ES, int BN, bool kInt, typename StoreFn>
__device__ __forceinline__ void epi_rows_tma(uint32_t taddr0, int lane, const uint32_t* bias_s,
                                             uint32_t stage, int valid_cols, uint32_t& cnt,
                                             bool* ovf, StoreFn&& store,
                                             const uint8_t* rrow = nullptr,
                                             const QParams& qp = QParams{}) {
  epi_rows_tma_src<PROG, ES, BN, kInt>(
      [&](int c0, uint32_t (&acc)[kChunk]) {
        tmem_ld32(taddr0 + c0, acc);
        tmem_ld_wait();
      },
      lane, bias_s, stage, valid_cols, cnt, ovf, store, rrow, qp);
}

// Cooperative per-tile bias staging: `nthreads` epilogue threads copy the
// tile's BN bias values into shared memory (zero past OC).
template <typename T>
__device__ __forceinline__ void stage_bias(T* dst, const void* bias, int col0, int bn,
                                           int oc, int tid, int nthreads) {
  for (int i = tid; i < bn; i += nthreads)
    dst[i] = (bias && col0 + i < oc) ? static_cast<const T*>(bias)[col0 + i] : T(0);
}

__device__ __forceinline__ void named_bar_sync(int id, int nthreads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

}  // namespace epi
}  // namespace tec_sm100
