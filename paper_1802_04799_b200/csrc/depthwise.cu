// depthwise.cu -- fused depthwise_conv2d (+scale/bias_add/add/mul/relu),
// the MobileNet D1-D9 path. HBM-bound (AI ~1-2 FLOP/B), so the design
// goal is to move every byte once at full width:
//  * NHWC activations: a thread owns VEC adjacent channels (one 128-bit
//    vector) and TW adjacent output pixels of one output row, so a warp
//    reads/writes contiguous channel runs (coalesced 16 B per lane);
//  * the TW-pixel strip reuses each loaded input column across the KW
//    taps in registers ("vectorize" + "unroll" knobs of the schedule);
//  * the epilogue members run in registers before one 128-bit store.
// Arithmetic follows the oracle exactly: per output, facc = 0 then
// facc = facc + x*w over (rh, rw) in order with float rounding per op
// (R/src/texpr.cpp:205-228, R/src/expr.cpp:137-145), so the f32 and
// bf16-input paths are bit-identical to evaluate_reference on the same
// (rounded) inputs, and the i8 path is exact.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <type_traits>

#include "conv_params.h"

namespace tec_sm100 {

namespace {

template <typename T>
struct Vec;  // VEC elements of T packed in 16 bytes
template <>
struct Vec<float> {
  static constexpr int N = 4;
  __device__ static void load(const float* p, float (&v)[4]) {
    const float4 t = *reinterpret_cast<const float4*>(p);
    v[0] = t.x; v[1] = t.y; v[2] = t.z; v[3] = t.w;
  }
};
template <>
struct Vec<__nv_bfloat16> {
  static constexpr int N = 8;
  __device__ static void load(const __nv_bfloat16* p, float (&v)[8]) {
    const uint4 t = *reinterpret_cast<const uint4*>(p);
    const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&t);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const float2 f = __bfloat1622float2(h[i]);
      v[2 * i] = f.x;
      v[2 * i + 1] = f.y;
    }
  }
};
template <>
struct Vec<int8_t> {
  static constexpr int N = 16;
  __device__ static void load(const int8_t* p, int32_t (&v)[16]) {
    const int4 t = *reinterpret_cast<const int4*>(p);
    const int8_t* b = reinterpret_cast<const int8_t*>(&t);
#pragma unroll
    for (int i = 0; i < 16; ++i) v[i] = b[i];
  }
};

template <typename T>
using AccT = typename std::conditional<std::is_same<T, int8_t>::value, int32_t,
                                       float>::type;

__device__ __forceinline__ float epi_f(float v, const EpilogueParams& e,
                                       int ch, const float* res,
                                       const float* mul) {
#pragma unroll 1
  for (int i = 0; i < e.n_ops; ++i) {
    switch (e.ops[i]) {
      case kEpiScale: v = __fmul_rn(v, e.fscale[i]); break;
      case kEpiBias: v = __fadd_rn(v, static_cast<const float*>(e.bias)[ch]); break;
      case kEpiAdd: v = __fadd_rn(v, *res); break;
      case kEpiMul: v = __fmul_rn(v, *mul); break;
      case kEpiRelu: v = (v < 0.0f) ? 0.0f : v; break;
      default: break;
    }
  }
  return v;
}

__device__ __forceinline__ int32_t epi_i(int64_t v, const EpilogueParams& e,
                                         int ch, int64_t flat, bool* ovf) {
#pragma unroll 1
  for (int i = 0; i < e.n_ops; ++i) {
    switch (e.ops[i]) {
      case kEpiScale: v = v * e.iscale[i]; break;
      case kEpiBias: v = v + static_cast<const int32_t*>(e.bias)[ch]; break;
      case kEpiAdd: v = v + static_cast<const int32_t*>(e.residual)[flat]; break;
      case kEpiMul: v = v * static_cast<const int32_t*>(e.mul_operand)[flat]; break;
      case kEpiRelu: v = v < 0 ? 0 : v; break;
      default: break;
    }
    if (v < INT32_MIN || v > INT32_MAX) *ovf = true;
  }
  return static_cast<int32_t>(v);
}

template <typename T>
__device__ __forceinline__ float ld_scalar(const void* p, int64_t i) {
  if constexpr (std::is_same<T, __nv_bfloat16>::value)
    return __bfloat162float(static_cast<const __nv_bfloat16*>(p)[i]);
  else
    return static_cast<const float*>(p)[i];
}

// One thread: VEC channels x TW output pixels of one output row.
template <typename InT, typename OutT, int TW, int KMAX>
__global__ void __launch_bounds__(256)
    depthwise_kernel(const DepthwiseParams p) {
  constexpr int VEC = Vec<InT>::N;
  using Acc = AccT<InT>;
  const int cgroups = p.c / VEC;
  const int wstrips = (p.ow + TW - 1) / TW;
  const int64_t total = static_cast<int64_t>(p.n) * p.oh * wstrips * cgroups;
  const int64_t tid = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (tid >= total) return;
  const int cg = static_cast<int>(tid % cgroups);
  int64_t t = tid / cgroups;
  const int ws = static_cast<int>(t % wstrips);
  t /= wstrips;
  const int oh = static_cast<int>(t % p.oh);
  const int n = static_cast<int>(t / p.oh);
  const int c0 = cg * VEC;
  const int ow0 = ws * TW;

  const InT* x = static_cast<const InT*>(p.x);
  const InT* wt = static_cast<const InT*>(p.wt);

  Acc acc[TW][VEC];
#pragma unroll
  for (int i = 0; i < TW; ++i)
#pragma unroll
    for (int v = 0; v < VEC; ++v) acc[i][v] = Acc(0);

  for (int rh = 0; rh < p.r; ++rh) {
    const int ih = oh * p.sh + rh - p.ph;
    const bool row_ok = ih >= 0 && ih < p.h;
    for (int rw = 0; rw < p.s; ++rw) {
      Acc wv[VEC];
      Vec<InT>::load(wt + static_cast<int64_t>(rh * p.s + rw) * p.c + c0, wv);
#pragma unroll
      for (int i = 0; i < TW; ++i) {
        const int iw = (ow0 + i) * p.sw + rw - p.pw;
        Acc xv[VEC];
        if (row_ok && iw >= 0 && iw < p.w && ow0 + i < p.ow) {
          Vec<InT>::load(
              x + ((static_cast<int64_t>(n) * p.h + ih) * p.w + iw) * p.c + c0,
              xv);
        } else {
#pragma unroll
          for (int v = 0; v < VEC; ++v) xv[v] = Acc(0);
        }
#pragma unroll
        for (int v = 0; v < VEC; ++v) {
          if constexpr (std::is_same<Acc, float>::value)
            acc[i][v] = __fadd_rn(acc[i][v], __fmul_rn(xv[v], wv[v]));
          else
            acc[i][v] += xv[v] * wv[v];
        }
      }
    }
  }

  bool ovf = false;
#pragma unroll
  for (int i = 0; i < TW; ++i) {
    const int ow = ow0 + i;
    if (ow >= p.ow) break;
    const int64_t base =
        ((static_cast<int64_t>(n) * p.oh + oh) * p.ow + ow) * p.c + c0;
    if constexpr (std::is_same<Acc, int32_t>::value) {
      int32_t o[VEC];
#pragma unroll
      for (int v = 0; v < VEC; ++v)
        o[v] = epi_i(acc[i][v], p.epi, c0 + v, base + v, &ovf);
      int4* dst = reinterpret_cast<int4*>(static_cast<int32_t*>(p.y) + base);
#pragma unroll
      for (int j = 0; j < VEC / 4; ++j)
        dst[j] = make_int4(o[4 * j], o[4 * j + 1], o[4 * j + 2], o[4 * j + 3]);
    } else {
      float o[VEC];
#pragma unroll
      for (int v = 0; v < VEC; ++v) {
        float r = 0.f, m = 0.f;
        if (p.epi.residual) r = ld_scalar<OutT>(p.epi.residual, base + v);
        if (p.epi.mul_operand) m = ld_scalar<OutT>(p.epi.mul_operand, base + v);
        o[v] = epi_f(acc[i][v], p.epi, c0 + v, &r, &m);
      }
      if constexpr (std::is_same<OutT, __nv_bfloat16>::value) {
        __nv_bfloat162 h[VEC / 2];
#pragma unroll
        for (int j = 0; j < VEC / 2; ++j)
          h[j] = __floats2bfloat162_rn(o[2 * j], o[2 * j + 1]);
        uint4* dst = reinterpret_cast<uint4*>(static_cast<__nv_bfloat16*>(p.y) + base);
        const uint4* src = reinterpret_cast<const uint4*>(h);
#pragma unroll
        for (int j = 0; j < VEC / 8; ++j) dst[j] = src[j];
      } else {
        float4* dst = reinterpret_cast<float4*>(static_cast<float*>(p.y) + base);
#pragma unroll
        for (int j = 0; j < VEC / 4; ++j)
          dst[j] = make_float4(o[4 * j], o[4 * j + 1], o[4 * j + 2], o[4 * j + 3]);
      }
    }
  }
  if (ovf && p.err) atomicOr(p.err, 1);
}

// Scalar variant for channel counts that are not a multiple of the 16-byte
// vector (one thread per output element, same arithmetic order).
template <typename InT, typename OutT>
__global__ void __launch_bounds__(256)
    depthwise_scalar_kernel(const DepthwiseParams p) {
  using Acc = AccT<InT>;
  const int64_t total = static_cast<int64_t>(p.n) * p.oh * p.ow * p.c;
  const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (i >= total) return;
  const int c = static_cast<int>(i % p.c);
  int64_t t = i / p.c;
  const int ow = static_cast<int>(t % p.ow);
  t /= p.ow;
  const int oh = static_cast<int>(t % p.oh);
  const int n = static_cast<int>(t / p.oh);
  const InT* x = static_cast<const InT*>(p.x);
  const InT* wt = static_cast<const InT*>(p.wt);
  Acc acc = Acc(0);
  for (int rh = 0; rh < p.r; ++rh) {
    const int ih = oh * p.sh + rh - p.ph;
    for (int rw = 0; rw < p.s; ++rw) {
      const int iw = ow * p.sw + rw - p.pw;
      Acc xv = Acc(0);
      if (ih >= 0 && ih < p.h && iw >= 0 && iw < p.w) {
        if constexpr (std::is_same<InT, __nv_bfloat16>::value)
          xv = __bfloat162float(x[((static_cast<int64_t>(n) * p.h + ih) * p.w + iw) * p.c + c]);
        else
          xv = static_cast<Acc>(x[((static_cast<int64_t>(n) * p.h + ih) * p.w + iw) * p.c + c]);
      }
      Acc wv;
      if constexpr (std::is_same<InT, __nv_bfloat16>::value)
        wv = __bfloat162float(wt[static_cast<int64_t>(rh * p.s + rw) * p.c + c]);
      else
        wv = static_cast<Acc>(wt[static_cast<int64_t>(rh * p.s + rw) * p.c + c]);
      if constexpr (std::is_same<Acc, float>::value)
        acc = __fadd_rn(acc, __fmul_rn(xv, wv));
      else
        acc += xv * wv;
    }
  }
  if constexpr (std::is_same<Acc, int32_t>::value) {
    bool ovf = false;
    static_cast<int32_t*>(p.y)[i] = epi_i(acc, p.epi, c, i, &ovf);
    if (ovf && p.err) atomicOr(p.err, 1);
  } else {
    float r = 0.f, m = 0.f;
    if (p.epi.residual) r = ld_scalar<OutT>(p.epi.residual, i);
    if (p.epi.mul_operand) m = ld_scalar<OutT>(p.epi.mul_operand, i);
    const float o = epi_f(acc, p.epi, c, &r, &m);
    if constexpr (std::is_same<OutT, __nv_bfloat16>::value)
      static_cast<__nv_bfloat16*>(p.y)[i] = __float2bfloat16_rn(o);
    else
      static_cast<float*>(p.y)[i] = o;
  }
}

// ------------------------------------------------------------ 3x3 fast path
// The MobileNet shape (3x3, stride 1 or 2, float data) with the member
// programs fuse_pass builds for it (none / bias / bias+relu), all fixed at
// compile time. A thread owns VEC channels x TW output pixels of one row:
// per filter row it loads the (TW-1)*SW + 3 input pixels ONCE into
// registers and reuses them for the three taps of all TW outputs (the
// generic kernel reloads per tap). Same per-output arithmetic order as the
// oracle (taps (rh, rw) in order, facc = facc + x*w, float rounding per op;
// out-of-image taps contribute x = 0 exactly like the reference's select).
enum DwProg { kDwNone = 0, kDwBias = 1, kDwBiasRelu = 2 };

// Division by a grid-invariant divisor as multiply-high + shift (dividend
// < 2^31): q = umulhi(n, m) >> s with m = ceil(2^(31+l) / d), l = ceil(log2 d).
struct FastDiv {
  uint32_t d, m, s;
  explicit FastDiv(uint32_t dd) : d(dd), m(0), s(0) {
    uint32_t l = 0;
    while ((1u << l) < dd) ++l;
    const uint64_t p = 31 + l;
    m = static_cast<uint32_t>(((uint64_t(1) << p) + dd - 1) / dd);
    s = static_cast<uint32_t>(p - 32);
  }
  __device__ __forceinline__ uint32_t divmod(uint32_t n, uint32_t* r) const {
    const uint32_t q = d == 1 ? n : (__umulhi(n, m) >> s);
    *r = n - q * d;
    return q;
  }
};

template <typename InT, typename OutT, int TW, int SW, int PROG>
__global__ void __launch_bounds__(256, 2)
    dw3x3_kernel(const DepthwiseParams p, const FastDiv div_cg, const FastDiv div_ws,
                 const FastDiv div_oh) {
  constexpr int VEC = Vec<InT>::N;
  constexpr int SPAN = (TW - 1) * SW + 3;
  // All 9 x C filter taps, converted to f32 once per CTA.
  extern __shared__ float s_w[];
  for (int i = threadIdx.x; i < 9 * p.c; i += blockDim.x)
    s_w[i] = ld_scalar<InT>(p.wt, i);
  __syncthreads();
  const uint32_t total = static_cast<uint32_t>(p.n) * p.oh * div_ws.d * div_cg.d;
  const uint32_t tid = blockIdx.x * blockDim.x + threadIdx.x;
  if (tid >= total) return;
  uint32_t t, cg, ws, oh;
  t = div_cg.divmod(tid, &cg);
  t = div_ws.divmod(t, &ws);
  const uint32_t n = div_oh.divmod(t, &oh);
  const int c0 = static_cast<int>(cg) * VEC;
  const int ow0 = static_cast<int>(ws) * TW;
  const int iw0 = ow0 * SW - p.pw;
  const InT* x = static_cast<const InT*>(p.x);

  float acc[TW][VEC];
#pragma unroll
  for (int i = 0; i < TW; ++i)
#pragma unroll
    for (int v = 0; v < VEC; ++v) acc[i][v] = 0.0f;

#pragma unroll
  for (int rh = 0; rh < 3; ++rh) {
    const int ih = static_cast<int>(oh) * p.sh + rh - p.ph;
    const bool row_ok = ih >= 0 && ih < p.h;
    float wv[3][VEC];
#pragma unroll
    for (int rw = 0; rw < 3; ++rw)
#pragma unroll
      for (int v = 0; v < VEC; v += 4) {
        const float4 q = *reinterpret_cast<const float4*>(s_w + (rh * 3 + rw) * p.c + c0 + v);
        wv[rw][v] = q.x; wv[rw][v + 1] = q.y; wv[rw][v + 2] = q.z; wv[rw][v + 3] = q.w;
      }
    const InT* xrow = x + (static_cast<int64_t>(n) * p.h + (row_ok ? ih : 0)) * p.w * p.c + c0;
    // Stream the row's input columns: column j feeds output i through tap
    // rw = j - i*SW; for a fixed output the taps arrive in rw order 0,1,2,
    // so the per-output accumulation order is the reference's.
#pragma unroll
    for (int j = 0; j < SPAN; ++j) {
      const int iw = iw0 + j;
      float xv[VEC];
      if (row_ok && iw >= 0 && iw < p.w) {
        Vec<InT>::load(xrow + static_cast<int64_t>(iw) * p.c, xv);
      } else {
#pragma unroll
        for (int v = 0; v < VEC; ++v) xv[v] = 0.0f;
      }
#pragma unroll
      for (int i = 0; i < TW; ++i) {
#pragma unroll
        for (int rw = 0; rw < 3; ++rw) {
          if (j == i * SW + rw) {
#pragma unroll
            for (int v = 0; v < VEC; ++v) {
              // bf16 x bf16 products are exact in f32 (8-bit mantissas), so
              // one fused multiply-add rounds exactly like the reference's
              // facc + (x*w); f32 operands keep the two roundings.
              if constexpr (std::is_same<InT, __nv_bfloat16>::value)
                acc[i][v] = __fmaf_rn(xv[v], wv[rw][v], acc[i][v]);
              else
                acc[i][v] = __fadd_rn(acc[i][v], __fmul_rn(xv[v], wv[rw][v]));
            }
          }
        }
      }
    }
  }
  const int oh_i = static_cast<int>(oh);

  float b[VEC];
  if constexpr (PROG != kDwNone) {
#pragma unroll
    for (int v = 0; v < VEC; v += 4) {
      const float4 q = *reinterpret_cast<const float4*>(static_cast<const float*>(p.epi.bias) + c0 + v);
      b[v] = q.x; b[v + 1] = q.y; b[v + 2] = q.z; b[v + 3] = q.w;
    }
  }
#pragma unroll
  for (int i = 0; i < TW; ++i) {
    const int ow = ow0 + i;
    if (ow >= p.ow) break;
    float o[VEC];
#pragma unroll
    for (int v = 0; v < VEC; ++v) {
      float r = acc[i][v];
      if constexpr (PROG != kDwNone) r = __fadd_rn(r, b[v]);
      if constexpr (PROG == kDwBiasRelu) r = r < 0.0f ? 0.0f : r;
      o[v] = r;
    }
    const int64_t base = ((static_cast<int64_t>(n) * p.oh + oh_i) * p.ow + ow) * p.c + c0;
    if constexpr (std::is_same<OutT, __nv_bfloat16>::value) {
      uint32_t h[VEC / 2];
#pragma unroll
      for (int j = 0; j < VEC / 2; ++j) {
        const __nv_bfloat162 q = __floats2bfloat162_rn(o[2 * j], o[2 * j + 1]);
        h[j] = *reinterpret_cast<const uint32_t*>(&q);
      }
      uint4* dst = reinterpret_cast<uint4*>(static_cast<__nv_bfloat16*>(p.y) + base);
#pragma unroll
      for (int j = 0; j < VEC / 8; ++j) dst[j] = make_uint4(h[4 * j], h[4 * j + 1], h[4 * j + 2], h[4 * j + 3]);
    } else {
      float4* dst = reinterpret_cast<float4*>(static_cast<float*>(p.y) + base);
#pragma unroll
      for (int j = 0; j < VEC / 4; ++j)
        dst[j] = make_float4(o[4 * j], o[4 * j + 1], o[4 * j + 2], o[4 * j + 3]);
    }
  }
}

// Which compile-time program matches the epilogue (-1: none does).
int dw_prog_of(const EpilogueParams& e) {
  if (e.n_ops == 0) return kDwNone;
  if (e.n_ops == 1 && e.ops[0] == kEpiBias) return kDwBias;
  if (e.n_ops == 2 && e.ops[0] == kEpiBias && e.ops[1] == kEpiRelu) return kDwBiasRelu;
  return -1;
}

template <typename InT, typename OutT, int TW, int SW>
int launch_dw3x3(const DepthwiseParams& p, int prog, cudaStream_t st) {
  constexpr int VEC = Vec<InT>::N;
  const int64_t total = static_cast<int64_t>(p.n) * p.oh * ((p.ow + TW - 1) / TW) * (p.c / VEC);
  if (total >= (int64_t(1) << 31)) return 1;  // 32-bit thread index
  const FastDiv dc(p.c / VEC), dw((p.ow + TW - 1) / TW), dh(p.oh);
  const unsigned blocks = static_cast<unsigned>((total + 255) / 256);
  const size_t smem = 9 * static_cast<size_t>(p.c) * sizeof(float);
  if (smem > 48 * 1024) return 1;
  switch (prog) {
    case kDwNone: dw3x3_kernel<InT, OutT, TW, SW, kDwNone><<<blocks, 256, smem, st>>>(p, dc, dw, dh); break;
    case kDwBias: dw3x3_kernel<InT, OutT, TW, SW, kDwBias><<<blocks, 256, smem, st>>>(p, dc, dw, dh); break;
    default: dw3x3_kernel<InT, OutT, TW, SW, kDwBiasRelu><<<blocks, 256, smem, st>>>(p, dc, dw, dh); break;
  }
  return cudaGetLastError();
}

// Fast path when applicable; returns 1 if it did not apply.
int try_dw3x3(const DepthwiseParams& p, int tw, cudaStream_t st) {
  const int prog = dw_prog_of(p.epi);
  if (prog < 0 || p.r != 3 || p.s != 3 || (p.sw != 1 && p.sw != 2)) return 1;
  if (p.in_type == kBF16 && p.c % 8 == 0) {
    if (p.out_type == kBF16) {
      if (p.sw == 1) return tw == 2 ? launch_dw3x3<__nv_bfloat16, __nv_bfloat16, 2, 1>(p, prog, st)
                                    : launch_dw3x3<__nv_bfloat16, __nv_bfloat16, 4, 1>(p, prog, st);
      return tw == 2 ? launch_dw3x3<__nv_bfloat16, __nv_bfloat16, 2, 2>(p, prog, st)
                     : launch_dw3x3<__nv_bfloat16, __nv_bfloat16, 4, 2>(p, prog, st);
    }
    if (p.out_type == kF32) {
      if (p.sw == 1) return launch_dw3x3<__nv_bfloat16, float, 4, 1>(p, prog, st);
      return launch_dw3x3<__nv_bfloat16, float, 4, 2>(p, prog, st);
    }
    return 1;
  }
  if (p.in_type == kF32 && p.out_type == kF32 && p.c % 4 == 0) {
    if (p.sw == 1) return tw == 2 ? launch_dw3x3<float, float, 2, 1>(p, prog, st)
                                  : launch_dw3x3<float, float, 4, 1>(p, prog, st);
    return tw == 2 ? launch_dw3x3<float, float, 2, 2>(p, prog, st)
                   : launch_dw3x3<float, float, 4, 2>(p, prog, st);
  }
  return 1;
}

}  // namespace

template <typename InT, typename OutT>
static int launch_dw_scalar(const DepthwiseParams& p, cudaStream_t st) {
  const int64_t total = static_cast<int64_t>(p.n) * p.oh * p.ow * p.c;
  const int64_t blocks = (total + 255) / 256;
  depthwise_scalar_kernel<InT, OutT><<<static_cast<unsigned>(blocks), 256, 0, st>>>(p);
  return cudaGetLastError();
}

template <typename InT, typename OutT, int TW>
static int launch_dw(const DepthwiseParams& p, cudaStream_t st) {
  constexpr int VEC = Vec<InT>::N;
  const int64_t total = static_cast<int64_t>(p.n) * p.oh *
                        ((p.ow + TW - 1) / TW) * (p.c / VEC);
  const int threads = 256;
  const int64_t blocks = (total + threads - 1) / threads;
  depthwise_kernel<InT, OutT, TW, 3><<<static_cast<unsigned>(blocks), threads, 0, st>>>(p);
  return cudaGetLastError();
}

// Returns cudaError_t; -1 when the (in, out) type pair is unsupported or
// C is not a multiple of the 16-byte vector.
int launch_depthwise(const DepthwiseParams& p, int tw, cudaStream_t st) {
  if (tw != 1) {  // knob unroll == 1 selects the generic kernel (diagnostics)
    const int e = try_dw3x3(p, tw, st);
    if (e != 1) return e;
  }
  const int vec = p.in_type == kBF16 ? 8 : p.in_type == kI8 ? 16 : 4;
  if (p.c % vec) {
    if (p.in_type == kBF16 && p.out_type == kBF16)
      return launch_dw_scalar<__nv_bfloat16, __nv_bfloat16>(p, st);
    if (p.in_type == kBF16 && p.out_type == kF32)
      return launch_dw_scalar<__nv_bfloat16, float>(p, st);
    if (p.in_type == kF32 && p.out_type == kF32)
      return launch_dw_scalar<float, float>(p, st);
    if (p.in_type == kI8 && p.out_type == kI32)
      return launch_dw_scalar<int8_t, int32_t>(p, st);
    return -1;
  }
  if (p.in_type == kBF16) {
    if (p.out_type == kBF16)
      return tw >= 4 ? launch_dw<__nv_bfloat16, __nv_bfloat16, 4>(p, st)
                     : launch_dw<__nv_bfloat16, __nv_bfloat16, 2>(p, st);
    if (p.out_type == kF32)
      return tw >= 4 ? launch_dw<__nv_bfloat16, float, 4>(p, st)
                     : launch_dw<__nv_bfloat16, float, 2>(p, st);
    return -1;
  }
  if (p.in_type == kF32) {
    if (p.c % 4 || p.out_type != kF32) return -1;
    return tw >= 4 ? launch_dw<float, float, 4>(p, st)
                   : launch_dw<float, float, 2>(p, st);
  }
  if (p.in_type == kI8) {
    if (p.c % 16 || p.out_type != kI32) return -1;
    return tw >= 4 ? launch_dw<int8_t, int32_t, 4>(p, st)
                   : launch_dw<int8_t, int32_t, 2>(p, st);
  }
  return -1;
}

}  // namespace tec_sm100
