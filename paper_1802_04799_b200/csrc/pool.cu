// pool.cu -- the two non-conv operators of the ResNet-18 graph:
// max_pool2d (stem, 3x3 stride 2 pad 1) and global_avg_pool (head). Both
// HBM-bound and on NHWC activations: a thread owns one 16-byte channel
// vector of one output pixel, so every warp access is a contiguous run.
//
// Semantics (oracle/tec_oracle.c restates them):
//  * max_pool2d: y[n,oh,ow,c] = max over the in-image window taps
//    (x[n, oh*sh+rh-ph, ow*sw+rw-pw, c]); out-of-image taps are skipped
//    (padding never wins). Exact for every dtype.
//  * global_avg_pool: the reference composition scale(sum(sum(x, axis=W),
//    axis=H), 1/(H*W)) (R/src/ops.cpp:111-149 sum, :260-281 scale): per
//    (n, c), each row is summed over w in order from 0.0f, the row sums are
//    summed over h in order, and the total is multiplied by the float-
//    rounded factor -- every step rounded to float, no FMA.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "conv_params.h"

namespace tec_sm100 {

namespace {

template <typename T>
struct Lanes { static constexpr int N = 16 / sizeof(T); };

__device__ __forceinline__ float to_f(float v) { return v; }
__device__ __forceinline__ float to_f(__nv_bfloat16 v) { return __bfloat162float(v); }

// One thread: one output pixel x 16 bytes of channels (32-bit index math:
// 64-bit divisions per element dominated the first version). K3 = the
// ResNet stem's 3x3 / stride-2 window at compile time: the tap loops unroll
// and the nine 16-byte loads issue together (runtime bounds kept the walk
// one dependent load at a time).
template <typename T, bool K3 = false>
__global__ void max_pool_kernel(PoolParams p) {
  const int pr = K3 ? 3 : p.r, ps = K3 ? 3 : p.s, psh = K3 ? 2 : p.sh, psw = K3 ? 2 : p.sw;
  constexpr int V = Lanes<T>::N;
  const int cv = p.c / V;
  const uint32_t total = static_cast<uint32_t>(p.n) * p.oh * p.ow * cv;
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x) {
    const uint32_t pix = i / cv;
    const int v = static_cast<int>(i - pix * cv);
    const uint32_t row = pix / p.ow;
    const int ow = static_cast<int>(pix - row * p.ow);
    const int n = static_cast<int>(row / p.oh);
    const int oh = static_cast<int>(row - n * p.oh);
    T best[V];
    bool any = false;
    const T* base = static_cast<const T*>(p.x) + static_cast<int64_t>(n) * p.h * p.w * p.c + v * V;
#pragma unroll
    for (int rh = 0; rh < pr; ++rh) {
      const int ih = oh * psh + rh - p.ph;
      if (ih < 0 || ih >= p.h) continue;
#pragma unroll
      for (int rw = 0; rw < ps; ++rw) {
        const int iw = ow * psw + rw - p.pw;
        if (iw < 0 || iw >= p.w) continue;
        uint4 raw = __ldg(reinterpret_cast<const uint4*>(base + (static_cast<int64_t>(ih) * p.w + iw) * p.c));
        const T* t = reinterpret_cast<const T*>(&raw);
#pragma unroll
        for (int j = 0; j < V; ++j) {
          if (!any) best[j] = t[j];
          else if constexpr (sizeof(T) == 2) best[j] = to_f(t[j]) > to_f(best[j]) ? t[j] : best[j];
          else best[j] = t[j] > best[j] ? t[j] : best[j];
        }
        any = true;
      }
    }
    T* dst = static_cast<T*>(p.y) + static_cast<int64_t>(pix) * p.c + v * V;
    if (!any) {
#pragma unroll
      for (int j = 0; j < V; ++j) best[j] = T{};
    }
    *reinterpret_cast<uint4*>(dst) = *reinterpret_cast<const uint4*>(best);
  }
}

// int8: the same walk on 16 channels as four SIMD words (__vmaxs4: a
// per-byte signed max per instruction; the generic kernel's per-byte
// compare/select went through local memory).
template <bool K3 = false>
__global__ void max_pool_i8_kernel(PoolParams p) {
  const int pr = K3 ? 3 : p.r, ps = K3 ? 3 : p.s, psh = K3 ? 2 : p.sh, psw = K3 ? 2 : p.sw;
  const int cv = p.c / 16;
  const uint32_t total = static_cast<uint32_t>(p.n) * p.oh * p.ow * cv;
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x) {
    const uint32_t pix = i / cv;
    const int v = static_cast<int>(i - pix * cv);
    const uint32_t row = pix / p.ow;
    const int ow = static_cast<int>(pix - row * p.ow);
    const int n = static_cast<int>(row / p.oh);
    const int oh = static_cast<int>(row - n * p.oh);
    uint4 best = make_uint4(0x80808080u, 0x80808080u, 0x80808080u, 0x80808080u);  // -128
    bool any = false;
    const int8_t* base = static_cast<const int8_t*>(p.x) + static_cast<int64_t>(n) * p.h * p.w * p.c + v * 16;
#pragma unroll
    for (int rh = 0; rh < pr; ++rh) {
      const int ih = oh * psh + rh - p.ph;
      if (ih < 0 || ih >= p.h) continue;
#pragma unroll
      for (int rw = 0; rw < ps; ++rw) {
        const int iw = ow * psw + rw - p.pw;
        if (iw < 0 || iw >= p.w) continue;
        const uint4 t = __ldg(reinterpret_cast<const uint4*>(base + (static_cast<int64_t>(ih) * p.w + iw) * p.c));
        best.x = __vmaxs4(best.x, t.x);
        best.y = __vmaxs4(best.y, t.y);
        best.z = __vmaxs4(best.z, t.z);
        best.w = __vmaxs4(best.w, t.w);
        any = true;
      }
    }
    if (!any) best = make_uint4(0u, 0u, 0u, 0u);
    *reinterpret_cast<uint4*>(static_cast<int8_t*>(p.y) + static_cast<int64_t>(pix) * p.c + v * 16) = best;
  }
}

// One thread: one (n, 16-byte channel vector); loops the H x W plane.
template <typename T, typename O>
__global__ void global_avg_pool_kernel(PoolParams p) {
  constexpr int V = Lanes<T>::N;
  const int cv = p.c / V;
  const int64_t total = static_cast<int64_t>(p.n) * cv;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int v = static_cast<int>(i % cv);
    const int n = static_cast<int>(i / cv);
    float tot[V];
#pragma unroll
    for (int j = 0; j < V; ++j) tot[j] = 0.0f;
    const T* base = static_cast<const T*>(p.x) + static_cast<int64_t>(n) * p.h * p.w * p.c + v * V;
    for (int h = 0; h < p.h; ++h) {
      float row[V];
#pragma unroll
      for (int j = 0; j < V; ++j) row[j] = 0.0f;
      for (int w = 0; w < p.w; ++w) {
        uint4 raw = *reinterpret_cast<const uint4*>(base + (static_cast<int64_t>(h) * p.w + w) * p.c);
        const T* t = reinterpret_cast<const T*>(&raw);
#pragma unroll
        for (int j = 0; j < V; ++j) row[j] = __fadd_rn(row[j], to_f(t[j]));
      }
#pragma unroll
      for (int j = 0; j < V; ++j) tot[j] = __fadd_rn(tot[j], row[j]);
    }
    O* dst = static_cast<O*>(p.y) + static_cast<int64_t>(n) * p.c + v * V;
#pragma unroll
    for (int j = 0; j < V; ++j) {
      const float r = __fmul_rn(tot[j], p.scale);
      if constexpr (sizeof(O) == 2) dst[j] = __float2bfloat16_rn(r);
      else dst[j] = r;
    }
  }
}

int grid_for(int64_t threads, int block) {
  int64_t g = (threads + block - 1) / block;
  return static_cast<int>(g < 148 * 32 ? (g < 1 ? 1 : g) : 148 * 32);
}

}  // namespace

// Returns cudaError_t, or -1 for an unsupported dtype / channel count.
int launch_max_pool(const PoolParams& p, cudaStream_t st) {
  const int bytes = p.type == kBF16 ? 2 : p.type == kI8 ? 1 : 4;
  if ((p.c * bytes) % 16) return -1;
  if (static_cast<int64_t>(p.n) * p.oh * p.ow * (p.c * bytes / 16) >= (int64_t(1) << 31)) return -1;
  const int64_t threads = static_cast<int64_t>(p.n) * p.oh * p.ow * (p.c * bytes / 16);
  const int block = 256, grid = grid_for(threads, block);
  const bool k3 = p.r == 3 && p.s == 3 && p.sh == 2 && p.sw == 2;
  switch (p.type) {
    case kBF16:
      if (k3) max_pool_kernel<__nv_bfloat16, true><<<grid, block, 0, st>>>(p);
      else max_pool_kernel<__nv_bfloat16><<<grid, block, 0, st>>>(p);
      break;
    case kF32:
      if (k3) max_pool_kernel<float, true><<<grid, block, 0, st>>>(p);
      else max_pool_kernel<float><<<grid, block, 0, st>>>(p);
      break;
    case kI32: max_pool_kernel<int32_t><<<grid, block, 0, st>>>(p); break;
    case kI8:
      if (k3) max_pool_i8_kernel<true><<<grid, block, 0, st>>>(p);
      else max_pool_i8_kernel<<<grid, block, 0, st>>>(p);
      break;
    default: return -1;
  }
  return cudaGetLastError();
}

int launch_global_avg_pool(const PoolParams& p, cudaStream_t st) {
  const int bytes = p.type == kBF16 ? 2 : 4;
  if (p.type != kBF16 && p.type != kF32) return -1;
  if (p.out_type != kBF16 && p.out_type != kF32) return -1;
  if ((p.c * bytes) % 16) return -1;
  const int64_t threads = static_cast<int64_t>(p.n) * (p.c * bytes / 16);
  const int block = 128, grid = grid_for(threads, block);
  if (p.type == kBF16) {
    if (p.out_type == kBF16)
      global_avg_pool_kernel<__nv_bfloat16, __nv_bfloat16><<<grid, block, 0, st>>>(p);
    else
      global_avg_pool_kernel<__nv_bfloat16, float><<<grid, block, 0, st>>>(p);
  } else {
    if (p.out_type == kBF16)
      global_avg_pool_kernel<float, __nv_bfloat16><<<grid, block, 0, st>>>(p);
    else
      global_avg_pool_kernel<float, float><<<grid, block, 0, st>>>(p);
  }
  return cudaGetLastError();
}

}  // namespace tec_sm100
