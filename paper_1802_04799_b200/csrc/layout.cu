// layout.cu -- graph-boundary layout kernels (the layout_transform operator,
// R/src/ops.cpp:419-489, specialised to the two layouts this backend uses):
//   * NCHW (the reference DenseTensor layout) <-> NHWC channel-packed
//     activations, converting to the compute element type on the way;
//   * OIHW weights -> KRSC (dense conv) / RSC (depthwise) packed weights.
// Both directions run as 32x32 shared-memory tiled transposes so reads and
// writes are coalesced.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>

#include "conv_params.h"

namespace tec_sm100 {

// Exact three-way bf16 split of an f32 value (the f32tc path, conv_f32tc.cu):
// x == h + m + l with h = bf16(x), m = bf16(x - h), l = bf16(x - h - m). Each
// residual is exact in f32 and the last one has <= 8 significant bits, so
// the split loses nothing (f32's 24-bit mantissa = 3 x 8).
__device__ __forceinline__ __nv_bfloat16 split3(float x, int plane) {
  const __nv_bfloat16 h = __float2bfloat16_rn(x);
  if (plane == 0) return h;
  const float r1 = __fsub_rn(x, __bfloat162float(h));
  const __nv_bfloat16 m = __float2bfloat16_rn(r1);
  if (plane == 1) return m;
  return __float2bfloat16_rn(__fsub_rn(r1, __bfloat162float(m)));
}

// Packed activation element kinds.
enum PackMode : int32_t {
  kPackBF16 = 0,    // bf16(x)
  kPackSplit3 = 1,  // bf16 planes [h | m | l], cp/3 channels each (split3)
  kPackI8 = 2,      // int8 copy
  kPackF32 = 3,     // f32 copy
  kPackI32 = 4,     // i32 copy
  kPackSplit3I = 5, // split3 interleaved: [h16 | m16 | l16 | 0] per 64-channel pixel
};

// Channels per plane of the split layouts (cp = stored channels per pixel).
__host__ __device__ __forceinline__ int64_t plane_channels(int mode, int64_t cp) {
  return mode == kPackSplit3I ? 16 : mode == kPackSplit3 ? cp / 3 : cp;
}
__host__ __device__ __forceinline__ bool split_mode(int mode) {
  return mode == kPackSplit3 || mode == kPackSplit3I;
}

// in: [n][c][hw] (f32, or i8 / i32), out: [n][hw][cp] with cp >= c (Split3:
// three bf16 planes of cp/3 channels), padded channels zero-filled.
template <typename InT>
__global__ void pack_nchw_to_nhwc_kernel(const InT* __restrict__ in,
                                         void* __restrict__ out, int64_t c,
                                         int64_t hw, int64_t cp, int mode) {
  __shared__ float tile[32][33];
  const int64_t n = blockIdx.z;
  const int64_t c0 = static_cast<int64_t>(blockIdx.y) * 32;
  const int64_t p0 = static_cast<int64_t>(blockIdx.x) * 32;
  const int tx = threadIdx.x, ty = threadIdx.y;  // 32 x 8
  for (int i = ty; i < 32; i += 8) {
    const int64_t cc = c0 + i, pp = p0 + tx;
    float v = 0.f;
    if (cc < c && pp < hw) v = static_cast<float>(in[(n * c + cc) * hw + pp]);
    tile[i][tx] = v;
  }
  __syncthreads();
  const int64_t cpp = plane_channels(mode, cp);  // channels per plane
  for (int i = ty; i < 32; i += 8) {
    const int64_t pp = p0 + i, cc = c0 + tx;
    if (pp >= hw) continue;
    const int64_t obase = (n * hw + pp) * cp;
    if (cc < c) {
      const float v = tile[tx][i];
      switch (mode) {
        case kPackBF16:
          static_cast<__nv_bfloat16*>(out)[obase + cc] = __float2bfloat16_rn(v);
          break;
        case kPackSplit3:
        case kPackSplit3I: {
          __nv_bfloat16* o = static_cast<__nv_bfloat16*>(out);
#pragma unroll
          for (int pl = 0; pl < 3; ++pl) o[obase + pl * cpp + cc] = split3(v, pl);
          break;
        }
        case kPackI8:
          static_cast<int8_t*>(out)[obase + cc] = static_cast<int8_t>(v);
          break;
        case kPackF32:
          static_cast<float*>(out)[obase + cc] = v;
          break;
        case kPackI32:
          static_cast<int32_t*>(out)[obase + cc] = static_cast<int32_t>(v);
          break;
      }
    }
    // zero the channel padding [ctot, cp) once per pixel (block column 0)
    if (blockIdx.y == 0) {
      for (int64_t z = c + tx; z < cpp; z += 32) {
        switch (mode) {
          case kPackBF16:
            static_cast<__nv_bfloat16*>(out)[obase + z] = __float2bfloat16_rn(0.f);
            break;
          case kPackSplit3:
          case kPackSplit3I:
#pragma unroll
            for (int pl = 0; pl < 3; ++pl)
              static_cast<__nv_bfloat16*>(out)[obase + pl * cpp + z] = __float2bfloat16_rn(0.f);
            break;
          case kPackF32:
            static_cast<float*>(out)[obase + z] = 0.f;
            break;
          case kPackI8:
            static_cast<int8_t*>(out)[obase + z] = 0;
            break;
          case kPackI32:
            static_cast<int32_t*>(out)[obase + z] = 0;
            break;
        }
      }
      if (mode == kPackSplit3I)  // the 4th (zero) slice of an interleaved pixel
        for (int64_t z = 3 * cpp + tx; z < cp; z += 32)
          static_cast<__nv_bfloat16*>(out)[obase + z] = __float2bfloat16_rn(0.f);
    }
  }
}

// in: [n][hw][c] (f32 / bf16 / i32), out: [n][c][hw] (f32 or i32).
template <typename InT, typename OutT>
__global__ void unpack_nhwc_to_nchw_kernel(const InT* __restrict__ in,
                                           OutT* __restrict__ out, int64_t c,
                                           int64_t hw) {
  __shared__ OutT tile[32][33];
  const int64_t n = blockIdx.z;
  const int64_t p0 = static_cast<int64_t>(blockIdx.y) * 32;
  const int64_t c0 = static_cast<int64_t>(blockIdx.x) * 32;
  const int tx = threadIdx.x, ty = threadIdx.y;
  for (int i = ty; i < 32; i += 8) {
    const int64_t pp = p0 + i, cc = c0 + tx;
    OutT v = OutT(0);
    if (pp < hw && cc < c) {
      if constexpr (sizeof(InT) == 2)
        v = static_cast<OutT>(__bfloat162float(in[(n * hw + pp) * c + cc]));
      else
        v = static_cast<OutT>(in[(n * hw + pp) * c + cc]);
    }
    tile[i][tx] = v;
  }
  __syncthreads();
  for (int i = ty; i < 32; i += 8) {
    const int64_t cc = c0 + i, pp = p0 + tx;
    if (cc < c && pp < hw) out[(n * c + cc) * hw + pp] = tile[tx][i];
  }
}

// OIHW -> [K][R][S][cp] (dense) with the compute-type conversion.
template <typename InT>
__global__ void pack_weights_krsc_kernel(const InT* __restrict__ w,
                                         void* __restrict__ out, int64_t k,
                                         int64_t c, int64_t r, int64_t s,
                                         int64_t cp, int mode) {
  const int64_t total = k * r * s * cp;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
       i < total; i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t ci = i % cp;
    int64_t t = i / cp;
    const int64_t ss = t % s;
    t /= s;
    const int64_t rr = t % r;
    const int64_t kk = t / r;
    const int64_t cpp = plane_channels(mode, cp);  // channels per plane
    const int64_t src_c = ci % cpp, plane = ci / cpp;
    float v = 0.f;
    if (src_c < c && plane < 3) v = static_cast<float>(w[((kk * c + src_c) * r + rr) * s + ss]);
    switch (mode) {
      case kPackBF16:
        static_cast<__nv_bfloat16*>(out)[i] = __float2bfloat16_rn(v);
        break;
      case kPackSplit3:
      case kPackSplit3I:
        static_cast<__nv_bfloat16*>(out)[i] = split3(v, static_cast<int>(plane));
        break;
      case kPackF32:
        static_cast<float*>(out)[i] = v;
        break;
      case kPackI8:
        static_cast<int8_t*>(out)[i] = static_cast<int8_t>(v);
        break;
      default:
        break;
    }
  }
}

// The same reorder one output channel per CTA: its C x R x S source block
// is read once, coalesced, into shared memory and written out as [R*S][cp]
// (32-bit index math; the per-element kernel above read with an R*S stride
// and divided in 64 bits: ~0.3 ms for a 512x512x3x3 f32 -> split3 pack,
// paid on every host-buffer call).
template <typename InT>
__global__ void pack_weights_krsc_smem_kernel(const InT* __restrict__ w, void* __restrict__ out,
                                              int c, int rs, int cp, int mode) {
  extern __shared__ float wtile[];  // [c][rs]
  const int kk = blockIdx.x;
  const InT* src = w + static_cast<int64_t>(kk) * c * rs;
  for (int i = threadIdx.x; i < c * rs; i += blockDim.x) wtile[i] = static_cast<float>(src[i]);
  __syncthreads();
  const int cpp = static_cast<int>(plane_channels(mode, cp));
  const int64_t obase = static_cast<int64_t>(kk) * rs * cp;
  for (int i = threadIdx.x; i < rs * cp; i += blockDim.x) {
    const int rr = i / cp, ci = i - rr * cp;
    const int plane = ci / cpp, sc = ci - plane * cpp;
    const float v = sc < c && plane < 3 ? wtile[sc * rs + rr] : 0.f;
    switch (mode) {
      case kPackBF16:
        static_cast<__nv_bfloat16*>(out)[obase + i] = __float2bfloat16_rn(v);
        break;
      case kPackSplit3:
      case kPackSplit3I:
        static_cast<__nv_bfloat16*>(out)[obase + i] = split3(v, plane);
        break;
      case kPackF32:
        static_cast<float*>(out)[obase + i] = v;
        break;
      case kPackI8:
        static_cast<int8_t*>(out)[obase + i] = static_cast<int8_t>(v);
        break;
      default:
        break;
    }
  }
}

// Depthwise [C][1][R][S] -> [R][S][C] in f32 / bf16 / i8.
template <typename InT>
__global__ void pack_weights_rsc_kernel(const InT* __restrict__ w,
                                        void* __restrict__ out, int64_t c,
                                        int64_t r, int64_t s, int mode) {
  const int64_t total = c * r * s;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
       i < total; i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t cc = i % c;
    const int64_t tap = i / c;
    const float v = static_cast<float>(w[cc * r * s + tap]);
    switch (mode) {
      case kPackBF16:
        static_cast<__nv_bfloat16*>(out)[i] = __float2bfloat16_rn(v);
        break;
      case kPackI8:
        static_cast<int8_t*>(out)[i] = static_cast<int8_t>(v);
        break;
      default:
        static_cast<float*>(out)[i] = v;
        break;
    }
  }
}

// Space-to-depth (factor 2) packing for strided stems (C1: 7x7 stride 2 on
// 3 channels). The padded input is folded 2x2 into channels so the strided
// conv becomes a stride-1 conv with ceil(R/2) x ceil(S/2) taps over 4*C
// channels -- every tensor-core K step then carries real data (12 of 16
// channels instead of 3 of 16) and the conv runs on the stride-1 kernels.
//   out[n][i][j][(dy*2+dx)*C + c] = x[n][c][2i+dy-ph][2j+dx-pw]  (0 outside)
template <typename InT>
__global__ void pack_s2d_kernel(const InT* __restrict__ in, void* __restrict__ out,
                                int64_t n, int64_t c, int64_t h, int64_t w, int64_t ph,
                                int64_t pw, int64_t h2, int64_t w2, int64_t cp, int mode) {
  const int64_t total = n * h2 * w2 * cp;
  const int64_t cpp = plane_channels(mode, cp);  // channels per plane
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t ch = (i % cp) % cpp, plane = (i % cp) / cpp;
    int64_t t = i / cp;
    const int64_t jj = t % w2;
    t /= w2;
    const int64_t ii = t % h2;
    const int64_t nn = t / h2;
    float v = 0.f;
    if (ch < 4 * c && plane < 3) {
      const int64_t q = ch / c, cc = ch % c;
      const int64_t y = 2 * ii + q / 2 - ph, x = 2 * jj + q % 2 - pw;
      if (y >= 0 && y < h && x >= 0 && x < w)
        v = static_cast<float>(in[((nn * c + cc) * h + y) * w + x]);
    }
    if (mode == kPackBF16)
      static_cast<__nv_bfloat16*>(out)[i] = __float2bfloat16_rn(v);
    else if (split_mode(mode))
      static_cast<__nv_bfloat16*>(out)[i] = split3(v, static_cast<int>(plane));
    else
      static_cast<int8_t*>(out)[i] = static_cast<int8_t>(v);
  }
}

// Fast path (bf16, cp = 16): one thread per space-to-depth pixel writes
// its 16 channels as two 16-byte stores; 32-bit index math (the per-element
// kernel above spent its time in 64-bit divisions).
__global__ void pack_s2d_bf16_kernel(const float* __restrict__ in, __nv_bfloat16* __restrict__ out,
                                     int n, int c, int h, int w, int ph, int pw, int h2, int w2) {
  const int total = n * h2 * w2;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x) {
    const int jj = i % w2;
    const int t = i / w2;
    const int ii = t % h2;
    const int nn = t / h2;
    uint32_t wd[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) wd[k] = 0u;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int y = 2 * ii + q / 2 - ph, x = 2 * jj + q % 2 - pw;
      const bool in_img = y >= 0 && y < h && x >= 0 && x < w;
#pragma unroll
      for (int cc = 0; cc < 4; ++cc) {
        if (cc >= c) break;
        const float v = in_img ? in[((static_cast<int64_t>(nn) * c + cc) * h + y) * w + x] : 0.0f;
        const uint32_t b = __bfloat16_as_ushort(__float2bfloat16_rn(v));
        const int e = q * c + cc;  // channel (dy*2+dx)*C + c
        wd[e >> 1] |= (e & 1) ? (b << 16) : b;
      }
    }
    uint4* dst = reinterpret_cast<uint4*>(out + static_cast<int64_t>(i) * 16);
    dst[0] = make_uint4(wd[0], wd[1], wd[2], wd[3]);
    dst[1] = make_uint4(wd[4], wd[5], wd[6], wd[7]);
  }
}

// f32tc interleaved split (cp = 64, c <= 4): one thread per space-to-depth
// pixel builds its [h16 | m16 | l16 | 0] 128-byte pixel; the block's 256
// pixels (32 KB, contiguous in the output) go through shared memory so the
// stores are coalesced 16-byte runs across the warp (the per-element kernel
// above took 1.7 ms for the ResNet-18 b256 stem; per-thread 128-byte rows
// stored directly, 254 us). Chunk c of pixel p sits at slot p * 8 + (c ^ (p
// & 7)): the row-per-thread writes are bank-conflict free.
constexpr int kS2dSplitPx = 256;
// C > 0: the channel count at compile time (the RGB stem: 3) -- the
// channel slot of every value is then a constant and the packed words stay
// in registers (with a runtime count they are dynamically indexed arrays)
template <int C>
__global__ void __launch_bounds__(kS2dSplitPx) pack_s2d_split3i_kernel(
    const float* __restrict__ in, __nv_bfloat16* __restrict__ out, int n, int c_arg, int h,
    int w, int ph, int pw, int h2, int w2) {
  const int c = C ? C : c_arg;
  __shared__ uint4 st[kS2dSplitPx * 8];
  const int total = n * h2 * w2;
  const int t = static_cast<int>(threadIdx.x);
  for (int base = blockIdx.x * kS2dSplitPx; base < total; base += gridDim.x * kS2dSplitPx) {
    const int i = base + t;
    uint32_t wd[3][8];  // plane x 16 channels as bf16 pairs
#pragma unroll
    for (int pl = 0; pl < 3; ++pl)
#pragma unroll
      for (int k = 0; k < 8; ++k) wd[pl][k] = 0u;
    if (i < total) {
      const int jj = i % w2;
      const int tt = i / w2;
      const int ii = tt % h2;
      const int nn = tt / h2;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int y = 2 * ii + q / 2 - ph, x = 2 * jj + q % 2 - pw;
        const bool in_img = y >= 0 && y < h && x >= 0 && x < w;
#pragma unroll
        for (int cc = 0; cc < 4; ++cc) {
          if (cc >= c) break;
          const float v = in_img ? in[((static_cast<int64_t>(nn) * c + cc) * h + y) * w + x] : 0.0f;
          const int e = q * c + cc;  // channel (dy*2+dx)*C + c
#pragma unroll
          for (int pl = 0; pl < 3; ++pl) {
            const uint32_t b = __bfloat16_as_ushort(split3(v, pl));
            wd[pl][e >> 1] |= (e & 1) ? (b << 16) : b;
          }
        }
      }
    }
    __syncthreads();  // the previous round's reads of st are done
    const int sw = t & 7;
#pragma unroll
    for (int pl = 0; pl < 3; ++pl) {
      st[t * 8 + ((2 * pl) ^ sw)] = make_uint4(wd[pl][0], wd[pl][1], wd[pl][2], wd[pl][3]);
      st[t * 8 + ((2 * pl + 1) ^ sw)] = make_uint4(wd[pl][4], wd[pl][5], wd[pl][6], wd[pl][7]);
    }
    st[t * 8 + (6 ^ sw)] = make_uint4(0u, 0u, 0u, 0u);
    st[t * 8 + (7 ^ sw)] = make_uint4(0u, 0u, 0u, 0u);
    __syncthreads();
    const int npx = min(kS2dSplitPx, total - base);
    uint4* dst = reinterpret_cast<uint4*>(out + static_cast<int64_t>(base) * 64);
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const int idx = k * kS2dSplitPx + t;  // 16-byte chunk of the block's output
      const int p = idx >> 3, ch = idx & 7;
      if (p < npx) dst[idx] = st[p * 8 + (ch ^ (p & 7))];
    }
  }
}

// int8 (cp = 32, c <= 8): one thread per space-to-depth pixel, its 32
// channel bytes as two 16-byte stores (the per-element kernel above made
// one 1-byte store per thread: 770 us for the ResNet-18 b256 stem).
template <int C>  // compile-time channel count (0: runtime), as above
__global__ void pack_s2d_i8_kernel(const int8_t* __restrict__ in, int8_t* __restrict__ out,
                                   int n, int c_arg, int h, int w, int ph, int pw, int h2, int w2) {
  const int c = C ? C : c_arg;
  const int total = n * h2 * w2;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x) {
    const int jj = i % w2;
    const int t = i / w2;
    const int ii = t % h2;
    const int nn = t / h2;
    uint32_t wd[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) wd[k] = 0u;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int y = 2 * ii + q / 2 - ph, x = 2 * jj + q % 2 - pw;
      const bool in_img = y >= 0 && y < h && x >= 0 && x < w;
#pragma unroll
      for (int cc = 0; cc < 8; ++cc) {
        if (cc >= c) break;
        const uint32_t b =
            in_img ? static_cast<uint8_t>(in[((static_cast<int64_t>(nn) * c + cc) * h + y) * w + x]) : 0u;
        const int e = q * c + cc;  // channel (dy*2+dx)*C + c
        wd[e >> 2] |= b << (8 * (e & 3));
      }
    }
    uint4* dst = reinterpret_cast<uint4*>(out + static_cast<int64_t>(i) * 32);
    dst[0] = make_uint4(wd[0], wd[1], wd[2], wd[3]);
    dst[1] = make_uint4(wd[4], wd[5], wd[6], wd[7]);
  }
}

// Row-staged variant (bf16, cp = 16, w % 4 == 0): one CTA per space-to-depth
// row (image nn, row ii). The CTA reads the two input rows of every channel
// with coalesced float4 loads into shared memory (zero padding included),
// then each thread assembles s2d pixels from there. The per-pixel kernel
// above reads 12 scattered floats per pixel (2.3 TB/s on ResNet-18 b256);
// this one streams both directions.
constexpr int kS2dMaxW2 = 128;
constexpr int kS2dRows = 4;  // s2d rows per CTA
template <int C>  // compile-time channel count (0: runtime), as above
__global__ void __launch_bounds__(256) pack_s2d_rows_bf16_kernel(
    const float* __restrict__ in, __nv_bfloat16* __restrict__ out, int c_arg, int h, int w, int ph,
    int pw, int h2, int w2) {
  const int c = C ? C : c_arg;
  // [channel][input row of the CTA][staged column]
  __shared__ float tile[4][2 * kS2dRows][2 * kS2dMaxW2];
  const int ii0 = blockIdx.x * kS2dRows, nn = blockIdx.y;
  const int wp2 = 2 * w2;  // staged columns: input x = col - pw
  const int w4 = w >> 2;
  const int nrows = c * 2 * kS2dRows;
  // zero what the loads below do not write: padding columns and rows
  // outside the image (one warp per staged row)
  for (int rr = threadIdx.x >> 5; rr < nrows; rr += blockDim.x >> 5) {
    const int cc = rr / (2 * kS2dRows), dy = rr - cc * 2 * kS2dRows;
    const int y = 2 * ii0 + dy - ph;
    float* row = tile[cc][dy];
    if (y < 0 || y >= h) {
      for (int col = threadIdx.x & 31; col < wp2; col += 32) row[col] = 0.0f;
    } else {
      for (int col = threadIdx.x & 31; col < pw; col += 32) row[col] = 0.0f;
      for (int col = pw + w + (threadIdx.x & 31); col < wp2; col += 32) row[col] = 0.0f;
    }
  }
  // Loads in batches of kB per thread, all in flight before any is used
  // (one outstanding load per thread left the kernel latency bound).
  constexpr int kB = 8;
  const int nvec = nrows * w4;
  for (int base = 0; base < nvec; base += kB * blockDim.x) {
    float4 v[kB];
    float* dst[kB];
#pragma unroll
    for (int u = 0; u < kB; ++u) {
      const int idx = base + u * blockDim.x + threadIdx.x;
      dst[u] = nullptr;
      v[u] = make_float4(0.f, 0.f, 0.f, 0.f);
      if (idx < nvec) {
        const int rr = idx / w4, k4 = idx - rr * w4;
        const int cc = rr / (2 * kS2dRows), dy = rr - cc * 2 * kS2dRows;
        const int y = 2 * ii0 + dy - ph;
        if (y >= 0 && y < h) {
          v[u] = __ldg(reinterpret_cast<const float4*>(
                           in + ((static_cast<int64_t>(nn) * c + cc) * h + y) * w) + k4);
          dst[u] = &tile[cc][dy][pw + 4 * k4];
        }
      }
    }
#pragma unroll
    for (int u = 0; u < kB; ++u)
      if (dst[u]) { dst[u][0] = v[u].x; dst[u][1] = v[u].y; dst[u][2] = v[u].z; dst[u][3] = v[u].w; }
  }
  __syncthreads();
  for (int t = threadIdx.x; t < kS2dRows * w2; t += blockDim.x) {
    const int r = t / w2, jj = t - r * w2;
    const int ii = ii0 + r;
    if (ii >= h2) break;
    uint32_t wd[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) wd[k] = 0u;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
#pragma unroll
      for (int cc = 0; cc < 4; ++cc) {
        if (cc >= c) break;
        const float v = tile[cc][2 * r + (q >> 1)][2 * jj + (q & 1)];
        const uint32_t b = __bfloat16_as_ushort(__float2bfloat16_rn(v));
        const int e = q * c + cc;  // channel (dy*2+dx)*C + c
        wd[e >> 1] |= (e & 1) ? (b << 16) : b;
      }
    }
    uint4* o = reinterpret_cast<uint4*>(out + ((static_cast<int64_t>(nn) * h2 + ii) * w2 + jj) * 16);
    o[0] = make_uint4(wd[0], wd[1], wd[2], wd[3]);
    o[1] = make_uint4(wd[4], wd[5], wd[6], wd[7]);
  }
}

// Matching weights: [K][R2][S2][cp], w2[k][ri][sj][(dy*2+dx)*C + c] =
// w[k][c][2ri+dy][2sj+dx] (0 past the original R x S window).
template <typename InT>
__global__ void pack_weights_s2d_kernel(const InT* __restrict__ w, void* __restrict__ out,
                                        int64_t k, int64_t c, int64_t r, int64_t s, int64_t r2,
                                        int64_t s2, int64_t cp, int mode) {
  const int64_t total = k * r2 * s2 * cp;
  const int64_t cpp = plane_channels(mode, cp);  // channels per plane
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t ch = (i % cp) % cpp, plane = (i % cp) / cpp;
    int64_t t = i / cp;
    const int64_t sj = t % s2;
    t /= s2;
    const int64_t ri = t % r2;
    const int64_t kk = t / r2;
    float v = 0.f;
    if (ch < 4 * c && plane < 3) {
      const int64_t q = ch / c, cc = ch % c;
      const int64_t rr = 2 * ri + q / 2, ss = 2 * sj + q % 2;
      if (rr < r && ss < s) v = static_cast<float>(w[((kk * c + cc) * r + rr) * s + ss]);
    }
    if (mode == kPackBF16)
      static_cast<__nv_bfloat16*>(out)[i] = __float2bfloat16_rn(v);
    else if (split_mode(mode))
      static_cast<__nv_bfloat16*>(out)[i] = split3(v, static_cast<int>(plane));
    else
      static_cast<int8_t*>(out)[i] = static_cast<int8_t>(v);
  }
}

// Weights of the interleaved f32tc path (<= 16 channels per plane, incl.
// the space-to-depth stem): [tap][plane][K][16] bf16 -- per tap the three
// planes are consecutive 16-channel row blocks, so one 3-D TMA box lands
// them as [B_h; B_m; B_l] rows (one N-concatenated MMA operand).
// s2d: tap = (ri, sj) over (r2, s2), channel (dy*2+dx)*C + c of w[k][c][2ri+dy][2sj+dx];
// else tap = (rr, ss) over (r, s), channel c.
template <typename InT>
__global__ void pack_weights_split3i_kernel(const InT* __restrict__ w, __nv_bfloat16* __restrict__ out,
                                            int64_t k, int64_t c, int64_t r, int64_t s,
                                            int64_t r2, int64_t s2, int s2d) {
  const int64_t taps = s2d ? r2 * s2 : r * s;
  const int64_t total = taps * 3 * k * 16;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t ch = i % 16;
    int64_t t = i / 16;
    const int64_t kk = t % k;
    t /= k;
    const int plane = static_cast<int>(t % 3);
    const int64_t tap = t / 3;
    float v = 0.f;
    if (s2d) {
      if (ch < 4 * c) {
        const int64_t q = ch / c, cc = ch % c;
        const int64_t rr = 2 * (tap / s2) + q / 2, ss = 2 * (tap % s2) + q % 2;
        if (rr < r && ss < s) v = static_cast<float>(w[((kk * c + cc) * r + rr) * s + ss]);
      }
    } else if (ch < c) {
      v = static_cast<float>(w[((kk * c + ch) * r + tap / s) * s + tap % s]);
    }
    out[i] = split3(v, plane);
  }
}

// f32 NHWC [pixels][c] (an f32tc layer's output) -> the next f32tc conv's
// packed input: three exact bf16 planes per pixel, [h | m | l] blocks of cpp
// channels (cp = 3 * cpp) or interleaved [h16 | m16 | l16 | 0] (cp = 64).
__global__ void split3_nhwc_kernel(const float* __restrict__ in, __nv_bfloat16* __restrict__ out,
                                   int64_t pixels, int64_t c, int64_t cp, int64_t cpp) {
  const int64_t total = pixels * cp;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t px = i / cp, ch = i - px * cp;
    const int64_t plane = ch / cpp, cc = ch - plane * cpp;
    const float v = plane < 3 && cc < c ? in[px * c + cc] : 0.0f;
    out[i] = split3(v, static_cast<int>(plane < 3 ? plane : 0));
  }
}

// Vector form (c == cpp, c % 4 == 0, planes in blocks): a thread reads 4
// channels (16 B) and writes 4 bf16 (8 B) into each plane.
__global__ void split3_nhwc_vec_kernel(const float4* __restrict__ in, uint2* __restrict__ out,
                                       int64_t pixels, int c4) {
  const int64_t total = pixels * c4;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t px = i / c4;
    const int q = static_cast<int>(i - px * c4);
    const float4 v = in[i];
    const float f[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int pl = 0; pl < 3; ++pl) {
      uint32_t h[2];
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        const uint32_t lo = __bfloat16_as_ushort(split3(f[2 * j], pl));
        const uint32_t hi = __bfloat16_as_ushort(split3(f[2 * j + 1], pl));
        h[j] = lo | (hi << 16);
      }
      out[(px * 3 + pl) * c4 + q] = make_uint2(h[0], h[1]);
    }
  }
}

// ----------------------------------------------------------- launchers
int launch_split3_nhwc(const float* in, void* out, int64_t pixels, int64_t c, int64_t cp,
                       int64_t cpp, cudaStream_t st) {
  if (c == cpp && cp == 3 * cpp && c % 4 == 0) {
    const int64_t total = pixels * (c / 4);
    const int blocks = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>((total + 255) / 256, 148 * 32)));
    split3_nhwc_vec_kernel<<<blocks, 256, 0, st>>>(reinterpret_cast<const float4*>(in),
                                                   static_cast<uint2*>(out), pixels,
                                                   static_cast<int>(c / 4));
    return cudaGetLastError();
  }
  const int64_t total = pixels * cp;
  const int blocks = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>((total + 255) / 256, 148 * 32)));
  split3_nhwc_kernel<<<blocks, 256, 0, st>>>(in, static_cast<__nv_bfloat16*>(out), pixels, c, cp,
                                             cpp);
  return cudaGetLastError();
}
int launch_pack_weights_split3i(const void* w, void* out, int64_t k, int64_t c, int64_t r,
                                int64_t s, int64_t r2, int64_t s2, int s2d, cudaStream_t st) {
  const int64_t taps = s2d ? r2 * s2 : r * s;
  const int64_t total = taps * 3 * k * 16;
  const int blocks = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>((total + 255) / 256, 4096)));
  pack_weights_split3i_kernel<float><<<blocks, 256, 0, st>>>(
      static_cast<const float*>(w), static_cast<__nv_bfloat16*>(out), k, c, r, s, r2, s2, s2d);
  return cudaGetLastError();
}
int launch_pack_s2d(const void* in, int in_type, void* out, int64_t n, int64_t c, int64_t h,
                    int64_t w, int64_t ph, int64_t pw, int64_t h2, int64_t w2, int64_t cp,
                    int mode, cudaStream_t st) {
  if (in_type != kI8 && mode == kPackBF16 && cp == 16 && c <= 4 && w % 4 == 0 &&
      w2 <= kS2dMaxW2 && 2 * w2 >= w + pw && n <= 65535 && h2 <= (1 << 30)) {
    auto kfn = c == 3 ? pack_s2d_rows_bf16_kernel<3> : pack_s2d_rows_bf16_kernel<0>;
    kfn<<<dim3(static_cast<unsigned>((h2 + kS2dRows - 1) / kS2dRows), static_cast<unsigned>(n)),
          256, 0, st>>>(static_cast<const float*>(in),
                                         static_cast<__nv_bfloat16*>(out), static_cast<int>(c),
                                         static_cast<int>(h), static_cast<int>(w),
                                         static_cast<int>(ph), static_cast<int>(pw),
                                         static_cast<int>(h2), static_cast<int>(w2));
    return cudaGetLastError();
  }
  if (in_type != kI8 && mode == kPackBF16 && cp == 16 && c <= 4 && n * h2 * w2 < (1ll << 31)) {
    const int64_t px = n * h2 * w2;
    const int blocks = static_cast<int>(std::min<int64_t>((px + 255) / 256, 148 * 32));
    pack_s2d_bf16_kernel<<<blocks, 256, 0, st>>>(
        static_cast<const float*>(in), static_cast<__nv_bfloat16*>(out), static_cast<int>(n),
        static_cast<int>(c), static_cast<int>(h), static_cast<int>(w), static_cast<int>(ph),
        static_cast<int>(pw), static_cast<int>(h2), static_cast<int>(w2));
    return cudaGetLastError();
  }
  if (in_type == kF32 && mode == kPackSplit3I && cp == 64 && c <= 4 && n * h2 * w2 < (1ll << 31)) {
    const int64_t px = n * h2 * w2;
    const int blocks = static_cast<int>(std::min<int64_t>((px + kS2dSplitPx - 1) / kS2dSplitPx, 148 * 16));
    auto kfn = c == 3 ? pack_s2d_split3i_kernel<3> : pack_s2d_split3i_kernel<0>;
    kfn<<<blocks, kS2dSplitPx, 0, st>>>(
        static_cast<const float*>(in), static_cast<__nv_bfloat16*>(out), static_cast<int>(n),
        static_cast<int>(c), static_cast<int>(h), static_cast<int>(w), static_cast<int>(ph),
        static_cast<int>(pw), static_cast<int>(h2), static_cast<int>(w2));
    return cudaGetLastError();
  }
  if (in_type == kI8 && mode == kPackI8 && cp == 32 && c <= 8 && n * h2 * w2 < (1ll << 31)) {
    const int64_t px = n * h2 * w2;
    const int blocks = static_cast<int>(std::min<int64_t>((px + 255) / 256, 148 * 32));
    auto kfn = c == 3 ? pack_s2d_i8_kernel<3> : pack_s2d_i8_kernel<0>;
    kfn<<<blocks, 256, 0, st>>>(
        static_cast<const int8_t*>(in), static_cast<int8_t*>(out), static_cast<int>(n),
        static_cast<int>(c), static_cast<int>(h), static_cast<int>(w), static_cast<int>(ph),
        static_cast<int>(pw), static_cast<int>(h2), static_cast<int>(w2));
    return cudaGetLastError();
  }
  const int64_t total = n * h2 * w2 * cp;
  const int blocks = static_cast<int>(std::min<int64_t>((total + 255) / 256, 148 * 32));
  if (in_type == kI8)
    pack_s2d_kernel<int8_t><<<blocks, 256, 0, st>>>(static_cast<const int8_t*>(in), out, n, c,
                                                    h, w, ph, pw, h2, w2, cp, mode);
  else
    pack_s2d_kernel<float><<<blocks, 256, 0, st>>>(static_cast<const float*>(in), out, n, c, h,
                                                   w, ph, pw, h2, w2, cp, mode);
  return cudaGetLastError();
}

int launch_pack_weights_s2d(const void* w, int in_type, void* out, int64_t k, int64_t c,
                            int64_t r, int64_t s, int64_t r2, int64_t s2, int64_t cp, int mode,
                            cudaStream_t st) {
  const int64_t total = k * r2 * s2 * cp;
  const int blocks = static_cast<int>(std::min<int64_t>((total + 255) / 256, 4096));
  if (in_type == kI8)
    pack_weights_s2d_kernel<int8_t><<<blocks, 256, 0, st>>>(static_cast<const int8_t*>(w), out,
                                                            k, c, r, s, r2, s2, cp, mode);
  else
    pack_weights_s2d_kernel<float><<<blocks, 256, 0, st>>>(static_cast<const float*>(w), out, k,
                                                           c, r, s, r2, s2, cp, mode);
  return cudaGetLastError();
}

int launch_pack_activation(const void* in, int in_type, void* out, int64_t n,
                           int64_t c, int64_t hw, int64_t cp, int mode,
                           cudaStream_t st) {
  dim3 grid(static_cast<unsigned>((hw + 31) / 32),
            static_cast<unsigned>((c + 31) / 32), static_cast<unsigned>(n));
  dim3 block(32, 8);
  if (in_type == kF32)
    pack_nchw_to_nhwc_kernel<float><<<grid, block, 0, st>>>(
        static_cast<const float*>(in), out, c, hw, cp, mode);
  else if (in_type == kI8)
    pack_nchw_to_nhwc_kernel<int8_t><<<grid, block, 0, st>>>(
        static_cast<const int8_t*>(in), out, c, hw, cp, mode);
  else
    pack_nchw_to_nhwc_kernel<int32_t><<<grid, block, 0, st>>>(
        static_cast<const int32_t*>(in), out, c, hw, cp, mode);
  return cudaGetLastError();
}

int launch_unpack_output(const void* in, int in_type, void* out, int out_type,
                         int64_t n, int64_t c, int64_t hw, cudaStream_t st) {
  dim3 grid(static_cast<unsigned>((c + 31) / 32),
            static_cast<unsigned>((hw + 31) / 32), static_cast<unsigned>(n));
  dim3 block(32, 8);
  if (out_type == kI32) {
    if (in_type == kI8)
      unpack_nhwc_to_nchw_kernel<int8_t, int32_t><<<grid, block, 0, st>>>(
          static_cast<const int8_t*>(in), static_cast<int32_t*>(out), c, hw);
    else if (in_type == kI32)
      unpack_nhwc_to_nchw_kernel<int32_t, int32_t><<<grid, block, 0, st>>>(
          static_cast<const int32_t*>(in), static_cast<int32_t*>(out), c, hw);
    else
      return cudaErrorInvalidValue;
  } else if (out_type == kI8) {
    if (in_type != kI8) return cudaErrorInvalidValue;
    unpack_nhwc_to_nchw_kernel<int8_t, int8_t><<<grid, block, 0, st>>>(
        static_cast<const int8_t*>(in), static_cast<int8_t*>(out), c, hw);
  } else if (in_type == kBF16) {
    unpack_nhwc_to_nchw_kernel<__nv_bfloat16, float><<<grid, block, 0, st>>>(
        static_cast<const __nv_bfloat16*>(in), static_cast<float*>(out), c, hw);
  } else if (in_type == kF32) {
    unpack_nhwc_to_nchw_kernel<float, float><<<grid, block, 0, st>>>(
        static_cast<const float*>(in), static_cast<float*>(out), c, hw);
  } else {
    return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

int launch_pack_weights(const void* w, int in_type, void* out, int64_t k,
                        int64_t c, int64_t r, int64_t s, int64_t cp,
                        int depthwise, int mode, cudaStream_t st) {
  const int threads = 256;
  const int64_t total = depthwise ? c * r * s : k * r * s * cp;
  int blocks = static_cast<int>((total + threads - 1) / threads);
  if (blocks > 4096) blocks = 4096;
  if (blocks < 1) blocks = 1;
  if (depthwise) {
    if (in_type == kI8)
      pack_weights_rsc_kernel<int8_t><<<blocks, threads, 0, st>>>(
          static_cast<const int8_t*>(w), out, c, r, s, mode);
    else
      pack_weights_rsc_kernel<float><<<blocks, threads, 0, st>>>(
          static_cast<const float*>(w), out, c, r, s, mode);
  } else if (c * r * s * 4 <= 48 * 1024 && k <= 65535 && r * s * cp < (int64_t(1) << 31)) {
    const int smem = static_cast<int>(c * r * s * 4);
    if (in_type == kI8)
      pack_weights_krsc_smem_kernel<int8_t><<<static_cast<unsigned>(k), threads, smem, st>>>(
          static_cast<const int8_t*>(w), out, static_cast<int>(c), static_cast<int>(r * s),
          static_cast<int>(cp), mode);
    else
      pack_weights_krsc_smem_kernel<float><<<static_cast<unsigned>(k), threads, smem, st>>>(
          static_cast<const float*>(w), out, static_cast<int>(c), static_cast<int>(r * s),
          static_cast<int>(cp), mode);
  } else {
    if (in_type == kI8)
      pack_weights_krsc_kernel<int8_t><<<blocks, threads, 0, st>>>(
          static_cast<const int8_t*>(w), out, k, c, r, s, cp, mode);
    else
      pack_weights_krsc_kernel<float><<<blocks, threads, 0, st>>>(
          static_cast<const float*>(w), out, k, c, r, s, cp, mode);
  }
  return cudaGetLastError();
}

}  // namespace tec_sm100
