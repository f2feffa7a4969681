// depthwise_tma.cu -- the HBM-roofline depthwise 3x3 kernel (MobileNet D1-D9).
//
// Persistent CTAs walk (image, row band, channel block) tiles. For each tile
// ONE tiled TMA box brings the input halo -- (TH-1)*SW+3 rows x (OW-1)*SW+3
// columns x CB channels, the zero padding supplied by TMA out-of-bounds fill
// -- into shared memory, double-buffered so the next tile's load overlaps this
// tile's arithmetic. Every input byte therefore leaves HBM once; the 9-fold
// tap reuse is served from shared memory. A thread owns one 16-byte channel
// vector (fixed for the CTA's lifetime, its 9 taps in registers) and walks
// output pixels; consecutive threads read consecutive 16-byte chunks of the
// same / next pixel, so each tap read is a conflict-free contiguous run.
//
// Arithmetic is the oracle's per-output sequence (taps (rh, rw) in order,
// facc = facc + x*w rounded to float; out-of-image taps contribute x = 0
// exactly like the reference's select): bf16 x bf16 products are exact in
// f32, so one FMA rounds like the reference's add -- for bf16 the mixed
// fma.rn.f32.bf16 (SASS FHFMA.BF16) reads both operands as halves of the
// packed smem / tap registers, so nothing is unpacked (-10 % on D1-D9 vs
// unpack + FFMA2); f32 operands keep the separate multiply and add.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <array>
#include <cstdint>
#include <map>
#include <mutex>
#include <type_traits>
#include <vector>

#include "conv_params.h"
#include "sm100_ptx.cuh"

namespace tec_sm100 {

namespace {

template <typename T>
__device__ __forceinline__ void load8(const T* p, float (&v)[16 / sizeof(T)]);
template <>
__device__ __forceinline__ void load8<__nv_bfloat16>(const __nv_bfloat16* p, float (&v)[8]) {
  const uint4 t = *reinterpret_cast<const uint4*>(p);
  const uint32_t w[4] = {t.x, t.y, t.z, t.w};
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    v[2 * i] = __uint_as_float(w[i] << 16);
    v[2 * i + 1] = __uint_as_float(w[i] & 0xFFFF0000u);
  }
}
template <>
__device__ __forceinline__ void load8<float>(const float* p, float (&v)[4]) {
  const float4 t = *reinterpret_cast<const float4*>(p);
  v[0] = t.x; v[1] = t.y; v[2] = t.z; v[3] = t.w;
}
__device__ __forceinline__ void lds_vec(uint32_t addr, float (&v)[8]) {  // 8 bf16
  uint32_t w0, w1, w2, w3;
  asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];"
               : "=r"(w0), "=r"(w1), "=r"(w2), "=r"(w3) : "r"(addr));
  const uint32_t w[4] = {w0, w1, w2, w3};
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    v[2 * i] = __uint_as_float(w[i] << 16);
    v[2 * i + 1] = __uint_as_float(w[i] & 0xFFFF0000u);
  }
}
__device__ __forceinline__ void lds_vec(uint32_t addr, float (&v)[4]) {  // 4 f32
  asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
               : "=f"(v[0]), "=f"(v[1]), "=f"(v[2]), "=f"(v[3]) : "r"(addr));
}

enum { kDwtNone = 0, kDwtBias = 1, kDwtBiasRelu = 2 };

constexpr int kDwtThreads = 384;  // 12 warps, up to 168 registers per thread
constexpr int kTW = 4;            // output columns per work item

// COLB: bytes per staged pixel (channel block) when known at compile time
// (128: every layer with >= 128 B of channels) -- the tap reads' addresses
// then become immediate offsets off one row address; 0 = runtime t.cb * ES.
template <typename InT, typename OutT, int SW, int PROG, int COLB = 0>
__global__ void __launch_bounds__(kDwtThreads, 1)
    dw_tma_kernel(const __grid_constant__ CUtensorMap tm_x, const DepthwiseParams p,
                  const DwTmaShape t) {
  constexpr int VEC = 16 / static_cast<int>(sizeof(InT));
  constexpr int ES = static_cast<int>(sizeof(InT));
  const int colb = COLB ? COLB : t.cb * ES;
  const float nz = t.neg_zero;
  extern __shared__ __align__(128) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 127) &
                                             ~uintptr_t(127));
  __shared__ uint64_t full[2];
  const int tid = threadIdx.x;
  const int nvec = t.cb / VEC;          // channel vectors per tile
  const int v = tid % nvec;             // this thread's vector (fixed)
  const int lane_pix = tid / nvec;      // first pixel slot
  const int pix_step = blockDim.x / nvec;
  const int ngroups = (p.n + t.ni - 1) / t.ni;  // images per tile: t.ni (small layers)
  const int tiles = ngroups * t.bands * t.cblocks;
  const uint32_t img_bytes = static_cast<uint32_t>(t.rows_in * t.cols_in * t.cb * ES);
  const uint32_t tx_bytes = img_bytes * t.ni;

  if (tid == 0) {
    tma_prefetch_desc(&tm_x);
    mbar_init(&full[0], 1);
    mbar_init(&full[1], 1);
    fence_barrier_init();
  }
  __syncthreads();
  // Only the TMA-issuing thread waits for the previous layer: every other
  // thread reads activations from the smem tiles it lands (mbarrier-ordered)
  // and meanwhile loads its taps and bias (parameters) early.
  pdl_launch_dependents();
  if (tid == 0) pdl_wait();

  // tile -> (cblk slowest, so a CTA's consecutive tiles mostly share taps)
  auto decode = [&](int tile, int* n, int* band, int* cblk) {
    const int per_c = ngroups * t.bands;
    *cblk = tile / per_c;
    const int r = tile - *cblk * per_c;
    *n = (r / t.bands) * t.ni;  // first image of the group
    *band = r - (r / t.bands) * t.bands;
  };
  auto issue = [&](int tile, int buf) {
    int n, band, cblk;
    decode(tile, &n, &band, &cblk);
    mbar_arrive_expect_tx(&full[buf], tx_bytes);
    tma_load_4d(smem + buf * t.buf_bytes, &tm_x, &full[buf], cblk * t.cb, -p.pw,
                band * t.th * SW - p.ph, n);
  };

  int first = blockIdx.x;
  if (tid == 0 && first < tiles) issue(first, 0);
  constexpr int V2 = VEC / 2;  // float2 lanes: packed f32x2 FMA (FFMA2)
  constexpr bool kBF = std::is_same<InT, __nv_bfloat16>::value;
  float2 w2[kBF ? 1 : 9][V2];
  uint32_t wb[kBF ? 9 : 1][4];  // bf16: the taps stay packed (FHFMA.BF16 reads halves)
  float bias[VEC];
  int cur_cblk = -1;
  int it = 0;
  for (int tile = first; tile < tiles; tile += gridDim.x, ++it) {
    const int buf = it & 1;
    const int next = tile + gridDim.x;
    if (tid == 0 && next < tiles) issue(next, buf ^ 1);  // its buffer was released last iteration
    int n, band, cblk;
    decode(tile, &n, &band, &cblk);
    const int c0 = cblk * t.cb + v * VEC;
    if (cblk != cur_cblk) {  // the 9 taps (and bias) of this thread's channels
      cur_cblk = cblk;
#pragma unroll
      for (int k = 0; k < 9; ++k) {
        if constexpr (kBF) {
          const uint4 q = *reinterpret_cast<const uint4*>(static_cast<const InT*>(p.wt) + k * p.c + c0);
          wb[k][0] = q.x; wb[k][1] = q.y; wb[k][2] = q.z; wb[k][3] = q.w;
        } else {
          float wk[VEC];
          load8<InT>(static_cast<const InT*>(p.wt) + k * p.c + c0, wk);
#pragma unroll
          for (int j = 0; j < V2; ++j) w2[k][j] = make_float2(wk[2 * j], wk[2 * j + 1]);
        }
      }
      if constexpr (PROG != kDwtNone) {
#pragma unroll
        for (int j = 0; j < VEC; j += 4) {
          const float4 q = *reinterpret_cast<const float4*>(static_cast<const float*>(p.epi.bias) + c0 + j);
          bias[j] = q.x; bias[j + 1] = q.y; bias[j + 2] = q.z; bias[j + 3] = q.w;
        }
      }
    }
    mbar_wait(&full[buf], static_cast<uint32_t>((it >> 1) & 1));
    const uint32_t sbase = smem_u32(smem + buf * t.buf_bytes) + v * 16;
    const int oh0 = band * t.th;
    const int rows = min(t.th, p.oh - oh0);
    const int strips = (p.ow + kTW - 1) / kTW;
    const int nimg = min(t.ni, p.n - n);
    const int items = nimg * rows * strips;
    // kTW consecutive output columns per item: each loaded (and unpacked)
    // input column serves up to 3 taps of neighbouring outputs.
    // (image, strip, row) of item it2 -- ROW fastest: neighbouring items
    // are the same strip of consecutive rows, cols_in * cb * ES bytes apart
    // (cols_in odd for 64-byte channel rows, see dw_tma_plan), so the two
    // pixels a 64-byte-row layer (D1: 32 bf16 channels) puts in one
    // 128-byte shared-memory wavefront fall in different banks;
    // strip-fastest put them kTW * 64 B apart, a 2-way conflict on every
    // tap read. Stepped by pix_step with carries: the divisions run once
    // per tile instead of twice per item.
    const int dr = pix_step % rows, dq = pix_step / rows;
    const int ds = dq % strips, dim = dq / strips;
    int r_i = lane_pix % rows, s_i = (lane_pix / rows) % strips, im_i = lane_pix / rows / strips;
    auto advance = [&]() {
      r_i += dr;
      if (r_i >= rows) { r_i -= rows; ++s_i; }
      s_i += ds;
      if (s_i >= strips) { s_i -= strips; ++im_i; }
      im_i += dim;
    };
    for (int it2 = lane_pix; it2 < items; it2 += pix_step, advance()) {
      const int im = im_i, r = r_i, ow0 = s_i * kTW;
      float2 acc2[kTW][V2];
#pragma unroll
      for (int i = 0; i < kTW; ++i)
#pragma unroll
        for (int j = 0; j < V2; ++j) acc2[i][j] = make_float2(0.0f, 0.0f);
#pragma unroll
      for (int rh = 0; rh < 3; ++rh) {
        const uint32_t rowa = sbase + im * img_bytes +
            static_cast<uint32_t>(((r * SW + rh) * t.cols_in + ow0 * SW) * colb);
#pragma unroll
        for (int jc = 0; jc < (kTW - 1) * SW + 3; ++jc) {
          float x[kBF ? 1 : VEC];
          uint32_t xb[4];
          if constexpr (kBF) {
            asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];"
                         : "=r"(xb[0]), "=r"(xb[1]), "=r"(xb[2]), "=r"(xb[3])
                         : "r"(rowa + static_cast<uint32_t>(jc * colb)));
          } else {
            lds_vec(rowa + static_cast<uint32_t>(jc * colb), x);
          }
#pragma unroll
          for (int i = 0; i < kTW; ++i) {
#pragma unroll
            for (int rw = 0; rw < 3; ++rw) {
              if (jc == i * SW + rw) {  // taps arrive in rw order per output
#pragma unroll
                for (int j = 0; j < V2; ++j) {
                  if constexpr (kBF) {
                    // f32 += bf16 x bf16, the product exact, one rounding:
                    // the reference's facc + x*w
                    asm("{.reg .b16 xl, xh, wl, wh;\n\t"
                        "mov.b32 {xl, xh}, %2;\n\t"
                        "mov.b32 {wl, wh}, %3;\n\t"
                        "fma.rn.f32.bf16 %0, xl, wl, %0;\n\t"
                        "fma.rn.f32.bf16 %1, xh, wh, %1;}"
                        : "+f"(acc2[i][j].x), "+f"(acc2[i][j].y)
                        : "r"(xb[j]), "r"(wb[rh * 3 + rw][j]));
                  } else {
                    // the reference's facc + x*w, each rounded, two lanes
                    // at a time: the product as FFMA2 x*w + (-0) -- exactly
                    // the rounded product -- with the -0 a kernel parameter
                    // ptxas cannot see through, then FADD2. (A plain packed
                    // multiply -- mul.rn.f32x2, __fmul2_rn -- is contracted
                    // with the add into one FFMA2 by ptxas even at
                    // -fmad=false: not bit-exact.)
                    float2 prod;
                    asm("{.reg .b64 xa, za, pa;\n\t"
                        "mov.b64 xa, {%2, %3};\n\t"
                        "mov.b64 za, {%5, %5};\n\t"
                        "fma.rn.f32x2 pa, xa, %4, za;\n\t"
                        "mov.b64 {%0, %1}, pa;}"
                        : "=f"(prod.x), "=f"(prod.y)
                        : "f"(x[2 * j]), "f"(x[2 * j + 1]),
                          "l"(*reinterpret_cast<const uint64_t*>(&w2[rh * 3 + rw][j])), "f"(nz));
                    acc2[i][j] = __fadd2_rn(acc2[i][j], prod);
                  }
                }
              }
            }
          }
        }
      }
#pragma unroll
      for (int i = 0; i < kTW; ++i) {
        const int ow = ow0 + i;
        if (ow >= p.ow) break;
        float acc[VEC];
#pragma unroll
        for (int j = 0; j < V2; ++j) {
          float2 a = acc2[i][j];
          if constexpr (PROG != kDwtNone)  // packed, each component rounded
            a = __fadd2_rn(a, make_float2(bias[2 * j], bias[2 * j + 1]));
          acc[2 * j] = a.x;
          acc[2 * j + 1] = a.y;
        }
#pragma unroll
        for (int j = 0; j < VEC; ++j) {
          if constexpr (PROG == kDwtBiasRelu) acc[j] = acc[j] < 0.0f ? 0.0f : acc[j];
        }
        const int64_t o = ((static_cast<int64_t>(n + im) * p.oh + oh0 + r) * p.ow + ow) * p.c + c0;
        if constexpr (std::is_same<OutT, __nv_bfloat16>::value) {
          uint32_t h[VEC / 2];
#pragma unroll
          for (int j = 0; j < VEC / 2; ++j) {
            const __nv_bfloat162 q = __floats2bfloat162_rn(acc[2 * j], acc[2 * j + 1]);
            h[j] = *reinterpret_cast<const uint32_t*>(&q);
          }
          *reinterpret_cast<uint4*>(static_cast<__nv_bfloat16*>(p.y) + o) =
              make_uint4(h[0], h[1], h[2], h[3]);
        } else if constexpr (VEC == 8) {
          float4* dst = reinterpret_cast<float4*>(static_cast<float*>(p.y) + o);
          dst[0] = make_float4(acc[0], acc[1], acc[2], acc[3]);
          dst[1] = make_float4(acc[4], acc[5], acc[6], acc[7]);
        } else {
          *reinterpret_cast<float4*>(static_cast<float*>(p.y) + o) =
              make_float4(acc[0], acc[1], acc[2], acc[3]);
        }
      }
    }
    __syncthreads();  // every thread is done with `buf` before it is refilled
  }
}

// 3x3 max-pool on bf16 NHWC through the same TMA tiles. The map's
// out-of-bounds fill is NaN and __hmax2 returns the non-NaN operand, so
// padding never wins -- exactly max over the in-image taps. (A NaN *input*
// is skipped the same way.) bf16 max is exact, so no conversions.
template <int SW>
__global__ void __launch_bounds__(kDwtThreads, 1)
    pool_tma_kernel(const __grid_constant__ CUtensorMap tm_x, const DepthwiseParams p,
                    const DwTmaShape t) {
  constexpr int ES = 2;
  extern __shared__ __align__(128) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 127) &
                                             ~uintptr_t(127));
  __shared__ uint64_t full[2];
  const int tid = threadIdx.x;
  const int nvec = t.cb / 8;
  const int v = tid % nvec;
  const int lane_pix = tid / nvec;
  const int pix_step = blockDim.x / nvec;
  const int ngroups = (p.n + t.ni - 1) / t.ni;
  const int tiles = ngroups * t.bands * t.cblocks;
  const uint32_t img_bytes = static_cast<uint32_t>(t.rows_in * t.cols_in * t.cb * ES);
  const uint32_t tx_bytes = img_bytes * t.ni;
  if (tid == 0) {
    tma_prefetch_desc(&tm_x);
    mbar_init(&full[0], 1);
    mbar_init(&full[1], 1);
    fence_barrier_init();
  }
  __syncthreads();
  pdl_launch_dependents();
  if (tid == 0) pdl_wait();  // only the TMA issuer touches the previous layer's output
  auto decode = [&](int tile, int* n, int* band, int* cblk) {
    const int per_c = ngroups * t.bands;
    *cblk = tile / per_c;
    const int r = tile - *cblk * per_c;
    *n = (r / t.bands) * t.ni;
    *band = r - (r / t.bands) * t.bands;
  };
  auto issue = [&](int tile, int buf) {
    int n, band, cblk;
    decode(tile, &n, &band, &cblk);
    mbar_arrive_expect_tx(&full[buf], tx_bytes);
    tma_load_4d(smem + buf * t.buf_bytes, &tm_x, &full[buf], cblk * t.cb, -p.pw,
                band * t.th * SW - p.ph, n);
  };
  if (tid == 0 && static_cast<int>(blockIdx.x) < tiles) issue(blockIdx.x, 0);
  int it = 0;
  for (int tile = blockIdx.x; tile < tiles; tile += gridDim.x, ++it) {
    const int buf = it & 1;
    const int next = tile + gridDim.x;
    if (tid == 0 && next < tiles) issue(next, buf ^ 1);
    int n, band, cblk;
    decode(tile, &n, &band, &cblk);
    const int c0 = cblk * t.cb + v * 8;
    mbar_wait(&full[buf], static_cast<uint32_t>((it >> 1) & 1));
    const uint32_t sbase = smem_u32(smem + buf * t.buf_bytes) + v * 16;
    const int oh0 = band * t.th;
    const int rows = min(t.th, p.oh - oh0);
    const int nimg = min(t.ni, p.n - n);
    const int per_img = rows * p.ow;
    for (int it2 = lane_pix; it2 < nimg * per_img; it2 += pix_step) {
      const int im = it2 / per_img;
      const int rem_i = it2 - im * per_img;
      const int r = rem_i / p.ow, ow = rem_i - r * p.ow;
      __nv_bfloat162 m[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) m[j] = __float2bfloat162_rn(__int_as_float(0x7fc00000));  // NaN
#pragma unroll
      for (int rh = 0; rh < 3; ++rh)
#pragma unroll
        for (int rw = 0; rw < 3; ++rw) {
          uint32_t w0, w1, w2, w3;
          asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];"
                       : "=r"(w0), "=r"(w1), "=r"(w2), "=r"(w3)
                       : "r"(sbase + im * img_bytes +
                             static_cast<uint32_t>(((r * SW + rh) * t.cols_in + ow * SW + rw) * t.cb * ES)));
          const uint32_t wv[4] = {w0, w1, w2, w3};
#pragma unroll
          for (int j = 0; j < 4; ++j)
            m[j] = __hmax2(m[j], *reinterpret_cast<const __nv_bfloat162*>(&wv[j]));
        }
      const int64_t o = ((static_cast<int64_t>(n + im) * p.oh + oh0 + r) * p.ow + ow) * p.c + c0;
      *reinterpret_cast<uint4*>(static_cast<__nv_bfloat16*>(p.y) + o) =
          *reinterpret_cast<const uint4*>(m);
    }
    __syncthreads();
  }
}

}  // namespace

int launch_pool_tma(const DepthwiseParams& p, const CUtensorMap& tm_x, const DwTmaShape& t,
                    int sms, cudaStream_t st) {
  const int tiles = ((p.n + t.ni - 1) / t.ni) * t.bands * t.cblocks;
  const int grid = tiles < sms ? tiles : sms;
  const int smem = 2 * t.buf_bytes + 128;
  auto go = [&](auto kfn) -> int {
    cudaError_t e = cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    e = launch_pdl(kfn, dim3(grid), dim3(kDwtThreads), smem, st, tm_x, p, t);
    if (e != cudaSuccess) return e;
    return cudaGetLastError();
  };
  if (p.in_type != kBF16 || p.out_type != kBF16) return -1;
  return p.sw == 1 ? go(pool_tma_kernel<1>) : go(pool_tma_kernel<2>);
}

// Plans the tile (rows per band, channel block) for the shared-memory
// budget; returns false when the layer does not fit this kernel.
bool dw_tma_plan(const DepthwiseParams& p, DwTmaShape* t) {
  if (p.r != 3 || p.s != 3 || (p.sw != 1 && p.sw != 2) || p.sh != p.sw) return false;
  const int es = p.in_type == kBF16 ? 2 : 4;
  const int cb = p.c >= 128 / es ? 128 / es : p.c;  // 128-byte channel rows
  if (p.c % cb || (cb * es) % 16) return false;
  t->cb = cb;
  t->cblocks = p.c / cb;
  t->neg_zero = -0.0f;
  // whole kTW-column strips: the last strip reads TMA zero-fill columns
  t->cols_in = (((p.ow + kTW - 1) / kTW) * kTW - 1) * p.sw + 3;
  // 64-byte channel rows (D1: 32 bf16 channels): an odd number of columns
  // per input row, so vertically adjacent pixels (the row-fastest items'
  // neighbours) sit 64 B apart modulo 128 -- different banks
  if ((cb * es) % 128 && t->cols_in % 2 == 0) ++t->cols_in;
  if (t->cols_in > 256) return false;
  const int budget = 100 * 1024;  // per buffer (two buffers + slack < 227 KB)
  int th_max = p.oh;
  while (th_max > 1 && ((th_max - 1) * p.sw + 3) * t->cols_in * cb * es > budget) --th_max;
  // Band height: tiles go to CTAs round-robin (tile = cta + k * grid, band
  // fastest), so bands of unequal height can land all the tall ones on the
  // same CTAs -- D5 with th = 24 (+ a 4-row band) put every 24-row band on
  // the even CTAs (148 is even): half the SMs did 6x the work of the other
  // half. Pick the height whose round-robin makespan is smallest, in rows
  // (+ 2 per tile for the halo rows / pipeline step); ties keep the taller.
  // The search walks every tile (~10^4 steps per candidate): cache it per
  // shape so eager launches (tec_measure, the e2e host path) do not pay it.
  static std::mutex mu;
  static std::map<std::array<int, 4>, int> memo;
  const std::array<int, 4> key{p.n, p.oh, th_max, t->cblocks};
  int th = th_max;
  bool cached = false;
  {
    std::lock_guard<std::mutex> g(mu);
    auto f = memo.find(key);
    if (f != memo.end()) { th = f->second; cached = true; }
  }
  if (!cached && th_max < p.oh) {
    const int sms = 148;
    long best = -1;
    std::vector<long> load(sms);
    for (int h = th_max; h >= 1 && h * 4 >= th_max; --h) {
      const int bands = (p.oh + h - 1) / h;
      const long tiles = static_cast<long>(p.n) * bands * t->cblocks;
      const int grid = tiles < sms ? static_cast<int>(tiles) : sms;
      std::fill(load.begin(), load.end(), 0L);
      // a tile's cost: its passes over the CTA's threads (items of kTW
      // outputs, pix_step per pass; a part-filled last pass costs a whole
      // one) plus ~one pass of load / barrier overhead
      const int strips = (p.ow + kTW - 1) / kTW;
      const int pix_step = kDwtThreads / (cb * es / 16);
      for (long tile = 0; tile < tiles; ++tile) {
        const int band = static_cast<int>(tile % bands);
        const int rows = std::min(h, p.oh - band * h);
        load[tile % grid] += (rows * strips + pix_step - 1) / pix_step + 1;
      }
      const long span = *std::max_element(load.begin(), load.begin() + grid);
      if (best < 0 || span < best) { best = span; th = h; }
    }
    std::lock_guard<std::mutex> g(mu);
    memo[key] = th;
  }
  t->th = th;
  t->rows_in = (th - 1) * p.sw + 3;
  if (t->rows_in > 256) return false;
  t->bands = (p.oh + th - 1) / th;
  const int img = t->rows_in * t->cols_in * cb * es;
  // Images per tile when a whole image is one band: fewest rounds of tiles
  // per CTA x (ni + 1) -- one image-time per image plus ~one of per-tile
  // load/barrier overhead, ties to the larger ni (fewer tiles). Measured on
  // D7-D9 b64 (ni swept 1-8, tools/prof_dw.py): D7 2 (15.5 -> 12.9 us),
  // D8 2 (10.3 -> 8.4), D9 8 (10.4 -> 7.5); the earlier ">= 2 tiles per SM"
  // rule chose 1 / 1 / 3.
  t->ni = 1;
  if (t->bands == 1) {
    const int sms = 148;
    long best = -1;
    for (int ni = 1; ni <= 8 && ni <= p.n && ni * img <= budget; ++ni) {
      const long tiles = static_cast<long>((p.n + ni - 1) / ni) * t->cblocks;
      const long cost = ((tiles + sms - 1) / sms) * (ni + 1);
      if (best < 0 || cost <= best) { best = cost; t->ni = ni; }
    }
  }
  t->buf_bytes = ((img * t->ni) + 127) & ~127;
  return t->buf_bytes <= budget;
}

int launch_dw_tma(const DepthwiseParams& p, const CUtensorMap& tm_x, const DwTmaShape& t,
                  int prog, int sms, cudaStream_t st) {
  const int tiles = ((p.n + t.ni - 1) / t.ni) * t.bands * t.cblocks;
  const int grid = tiles < sms ? tiles : sms;
  const int smem = 2 * t.buf_bytes + 128;
  auto go = [&](auto kfn) -> int {
    cudaError_t e = cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    e = launch_pdl(kfn, dim3(grid), dim3(kDwtThreads), smem, st, tm_x, p, t);
    if (e != cudaSuccess) return e;
    return cudaGetLastError();
  };
  const bool col128 = t.cb * (p.in_type == kBF16 ? 2 : 4) == 128;
#define TEC_DWT_C(IN, OUT, SW_, CB_)                                             \
  switch (prog) {                                                               \
    case kDwtNone: return go(dw_tma_kernel<IN, OUT, SW_, kDwtNone, CB_>);       \
    case kDwtBias: return go(dw_tma_kernel<IN, OUT, SW_, kDwtBias, CB_>);       \
    default: return go(dw_tma_kernel<IN, OUT, SW_, kDwtBiasRelu, CB_>);         \
  }
#define TEC_DWT(IN, OUT, SW_)                                                    \
  if (col128) { TEC_DWT_C(IN, OUT, SW_, 128) }                                  \
  TEC_DWT_C(IN, OUT, SW_, 0)
  if (p.in_type == kBF16 && p.out_type == kBF16) {
    if (p.sw == 1) { TEC_DWT(__nv_bfloat16, __nv_bfloat16, 1) }
    TEC_DWT(__nv_bfloat16, __nv_bfloat16, 2)
  }
  if (p.in_type == kBF16 && p.out_type == kF32) {
    if (p.sw == 1) { TEC_DWT(__nv_bfloat16, float, 1) }
    TEC_DWT(__nv_bfloat16, float, 2)
  }
  if (p.in_type == kF32 && p.out_type == kF32) {
    if (p.sw == 1) { TEC_DWT(float, float, 1) }
    TEC_DWT(float, float, 2)
  }
#undef TEC_DWT
#undef TEC_DWT_C
  return -1;
}

}  // namespace tec_sm100
