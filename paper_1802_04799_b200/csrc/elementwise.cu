// elementwise.cu -- the unary integer graph operators around the int8 conv
// path (int8 ResNet-18 end to end): a short member program
// (cast / scale / relu / requantize, in member order) applied to every
// element of an NHWC activation. HBM-bound: one thread moves 16 elements
// (16 B of i8 or 64 B of i32 in, the same out), the grid is a multiple of
// the SM count and strides over the tensor.
//
// Semantics (tests/graph_oracle.py restates them; graph.py _fold_eval folds
// them on constants):
//  * CAST        i8 -> i32 exact; i8 | i32 -> f32 rounded to nearest;
//  * SCALE       integer data: x * c in int64 with the i32 range check
//                (DenseTensor::set_i, R/include/tec/tensor.hpp:63-69; an
//                out-of-range value raises the error flag -> FoldOverflow);
//                f32 data: __fmul_rn(x, (float)c) (R/src/ops.cpp:260-281);
//  * RELU        max(x, 0) (R/src/ops.cpp:250-259);
//  * REQUANTIZE  i32 -> i8: clamp((x * mult + 2^(shift-1)) >> shift, -128,
//                127) -- int64 product (|x| < 2^31, mult < 2^31: exact),
//                arithmetic shift, so ties round toward +inf.
#include <cuda_runtime.h>

#include <cstdint>
#include <type_traits>

#include "conv_params.h"

namespace tec_sm100 {

namespace {

constexpr int kVec = 16;  // elements per thread per iteration

// A value of the program: integer (int64) until a CAST to f32.
struct Val {
  int64_t i;
  float f;
};

__device__ __forceinline__ bool run_prog(const ElemProg& p, Val& v, bool is_f) {
  bool ovf = false;
#pragma unroll
  for (int k = 0; k < kMaxElemOps; ++k) {
    if (k >= p.n_ops) break;
    const int op = p.kind[k];
    if (op == kElemCast) {
      if (!is_f && p.cast_to_f[k]) {
        v.f = static_cast<float>(v.i);  // cvt.rn.f32.s64
        is_f = true;
      }
    } else if (op == kElemScale) {
      if (is_f) {
        v.f = __fmul_rn(v.f, p.fscale[k]);
      } else {
        // |x| < 2^31 after every range check, |c| < 2^31: exact in int64
        v.i *= p.mult[k];
        ovf |= v.i < INT32_MIN || v.i > INT32_MAX;
      }
    } else if (op == kElemRelu) {
      if (is_f) v.f = v.f < 0.0f ? 0.0f : v.f;
      else v.i = v.i < 0 ? 0 : v.i;
    } else if (op == kElemRequant) {
      const int s = p.shift[k];
      int64_t t = v.i * p.mult[k];
      if (s > 0) t = (t + (int64_t(1) << (s - 1))) >> s;
      v.i = t < -128 ? -128 : (t > 127 ? 127 : t);
    }
  }
  return ovf;
}

template <typename TI>
__device__ __forceinline__ Val load_val(TI x) {
  Val v;
  if constexpr (std::is_floating_point<TI>::value) {
    v.f = x;
    v.i = 0;
  } else {
    v.i = static_cast<int64_t>(x);
    v.f = 0.0f;
  }
  return v;
}

template <typename TI, typename TO>
__global__ void __launch_bounds__(256) elementwise_kernel(ElemProg p, const TI* __restrict__ x,
                                                          TO* __restrict__ y, int32_t* err) {
  constexpr bool kInF = std::is_floating_point<TI>::value;
  const int64_t groups = p.count / kVec;
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  bool ovf = false;
  // whole 16-element groups with vector loads / stores
  for (int64_t g = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; g < groups; g += stride) {
    TI in[kVec];
    const uint4* src = reinterpret_cast<const uint4*>(x + g * kVec);
#pragma unroll
    for (int q = 0; q < int(sizeof(in) / 16); ++q) reinterpret_cast<uint4*>(in)[q] = __ldcs(src + q);
    TO out[kVec];
#pragma unroll
    for (int j = 0; j < kVec; ++j) {
      Val v = load_val(in[j]);
      ovf |= run_prog(p, v, kInF);
      if constexpr (std::is_floating_point<TO>::value) out[j] = p.out_f ? v.f : float(v.i);
      else out[j] = static_cast<TO>(v.i);
    }
    uint4* dst = reinterpret_cast<uint4*>(y + g * kVec);
#pragma unroll
    for (int q = 0; q < int(sizeof(out) / 16); ++q) dst[q] = reinterpret_cast<uint4*>(out)[q];
  }
  // tail (count % 16 elements), one element per thread of block 0
  if (blockIdx.x == 0) {
    const int64_t i = groups * kVec + threadIdx.x;
    if (i < p.count) {
      Val v = load_val(x[i]);
      ovf |= run_prog(p, v, kInF);
      if constexpr (std::is_floating_point<TO>::value) y[i] = p.out_f ? v.f : float(v.i);
      else y[i] = static_cast<TO>(v.i);
    }
  }
  if (ovf && err) atomicExch(err, 1);
}

template <typename TI, typename TO>
int launch_t(const ElemProg& p, const void* x, void* y, int32_t* err, int sms,
             cudaStream_t st) {
  const int64_t groups = p.count / kVec;
  int64_t blocks = (groups + 255) / 256;
  const int64_t cap = int64_t(sms) * 8;  // 8 x 256 threads resident per SM
  blocks = blocks < 1 ? 1 : (blocks > cap ? cap : blocks);
  elementwise_kernel<TI, TO><<<static_cast<int>(blocks), 256, 0, st>>>(
      p, static_cast<const TI*>(x), static_cast<TO*>(y), err);
  return static_cast<int>(cudaGetLastError());
}

}  // namespace

// Batch-norm weight fold (tec_weight_pretransform_bn): y = x * s[i / per_row],
// one f32 product per element (__fmul_rn: graph.py bn_fold_weight).
__global__ void scale_rows_kernel(const float* __restrict__ x, const float* __restrict__ s,
                                  float* __restrict__ y, int64_t count, int64_t per_row) {
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < count;
       i += int64_t(gridDim.x) * blockDim.x)
    y[i] = __fmul_rn(x[i], s[i / per_row]);
}

int launch_scale_rows(const float* x, const float* s, float* y, int64_t count, int64_t per_row,
                      int sms, cudaStream_t st) {
  if (count <= 0) return 0;
  int64_t blocks = (count + 255) / 256;
  if (blocks > int64_t(sms) * 8) blocks = int64_t(sms) * 8;
  scale_rows_kernel<<<static_cast<int>(blocks), 256, 0, st>>>(x, s, y, count, per_row);
  return static_cast<int>(cudaGetLastError());
}

// x / y must be 16-byte aligned (device allocations and 256-B arena slots
// are). Supported (in, out): (i8, i32), (i8, i8), (i32, i8), (i32, i32),
// (i8, f32), (i32, f32), (f32, f32); the host validates the program.
int launch_elementwise(const ElemProg& p, const void* x, void* y, int32_t* err, int sms,
                       cudaStream_t st) {
  if (p.count <= 0) return 0;
  const int it = p.in_type, ot = p.out_type;
  if (it == kI8 && ot == kI32) return launch_t<int8_t, int32_t>(p, x, y, err, sms, st);
  if (it == kI8 && ot == kI8) return launch_t<int8_t, int8_t>(p, x, y, err, sms, st);
  if (it == kI32 && ot == kI8) return launch_t<int32_t, int8_t>(p, x, y, err, sms, st);
  if (it == kI32 && ot == kI32) return launch_t<int32_t, int32_t>(p, x, y, err, sms, st);
  if (it == kI8 && ot == kF32) return launch_t<int8_t, float>(p, x, y, err, sms, st);
  if (it == kI32 && ot == kF32) return launch_t<int32_t, float>(p, x, y, err, sms, st);
  if (it == kF32 && ot == kF32) return launch_t<float, float>(p, x, y, err, sms, st);
  return static_cast<int>(cudaErrorInvalidValue);
}

}  // namespace tec_sm100
