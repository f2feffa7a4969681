// tec_sm100_abi.cpp -- the C ABI declared in include/tec_sm100.h.
//
// Host side of the backend: argument validation with the reference's error
// taxonomy (infer_conv, R/src/ops.cpp:163-192), kernel-native layout
// planning, TMA descriptor encoding, kernel selection from schedule knobs
// (the "lowering" of a Config for target sm100), and the host-buffer entry
// point that stands in for eval_graph_node / native_eval.
//
// There is NO CPU fallback: every compute entry point runs the sm_100a
// kernels or returns an error.
#include "tec_sm100.h"

#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <vector>

#include "conv_params.h"
#include "sm100_ptx.cuh"

namespace tec_sm100 {
template <MmaKind KIND, int BN, int STAGES, int SWZ, bool PAIR>
int launch_conv_fprop_tc(const CUtensorMap& tm_a, const CUtensorMap& tm_b,
                         const CUtensorMap& tm_y, const ConvGemmParams& p, int grid,
                         cudaStream_t stream);
int launch_pack_activation(const void* in, int in_type, void* out, int64_t n,
                           int64_t c, int64_t hw, int64_t cp, int mode,
                           cudaStream_t st);
int launch_unpack_output(const void* in, int in_type, void* out, int out_type,
                         int64_t n, int64_t c, int64_t hw, cudaStream_t st);
int launch_pack_weights(const void* w, int in_type, void* out, int64_t k,
                        int64_t c, int64_t r, int64_t s, int64_t cp,
                        int depthwise, int mode, cudaStream_t st);
int launch_depthwise(const DepthwiseParams& p, int tw, cudaStream_t st);
int launch_pack_s2d(const void* in, int in_type, void* out, int64_t n, int64_t c, int64_t h,
                    int64_t w, int64_t ph, int64_t pw, int64_t h2, int64_t w2, int64_t cp,
                    int mode, cudaStream_t st);
int launch_split3_nhwc(const float* in, void* out, int64_t pixels, int64_t c, int64_t cp,
                       int64_t cpp, cudaStream_t st);
int launch_pack_weights_split3i(const void* w, void* out, int64_t k, int64_t c, int64_t r,
                                int64_t s, int64_t r2, int64_t s2, int s2d, cudaStream_t st);
int launch_pack_weights_s2d(const void* w, int in_type, void* out, int64_t k, int64_t c,
                            int64_t r, int64_t s, int64_t r2, int64_t s2, int64_t cp, int mode,
                            cudaStream_t st);
int launch_conv_f32_exact(const float* x, const float* w,
                          const ConvGemmParams& p, cudaStream_t st);
template <MmaKind KIND, int BN, int MS, int SWZ, int WSTAGES, bool kPair>
int launch_conv_halo(const CUtensorMap& tm_x, const CUtensorMap& tm_w,
                     const CUtensorMap& tm_y, const ConvHaloParams& p, int grid,
                     cudaStream_t stream);
int conv_halo_smem_bytes(int bn, int swz, int wstages, int halo_px, int stage_bytes, int ms,
                         bool pair);
int launch_max_pool(const PoolParams& p, cudaStream_t st);
bool dw_tma_plan(const DepthwiseParams& p, DwTmaShape* t);
int launch_dw_tma(const DepthwiseParams& p, const CUtensorMap& tm_x, const DwTmaShape& t,
                  int prog, int sms, cudaStream_t st);
int launch_pool_tma(const DepthwiseParams& p, const CUtensorMap& tm_x, const DwTmaShape& t,
                    int sms, cudaStream_t st);
int launch_global_avg_pool(const PoolParams& p, cudaStream_t st);
int launch_elementwise(const ElemProg& p, const void* x, void* y, int32_t* err, int sms,
                       cudaStream_t st);
int launch_scale_rows(const float* x, const float* s, float* y, int64_t count, int64_t per_row,
                      int sms, cudaStream_t st);
int launch_conv_f32tc(const CUtensorMap& tm_a, const CUtensorMap& tm_b, const CUtensorMap& tm_y,
                      const ConvGemmParams& p, int bn, int swz, bool inter, bool res, bool halo,
                      int prog, int grid, cudaStream_t st, bool pair);
int conv_f32tc_smem_bytes(int bn, int swz, bool inter, bool res, bool halo);
int conv_f32tc_pair_smem_bytes(int bn, int swz, bool inter, bool res, bool halo);
int conv_f32tc_stages(int bn, int swz, bool inter, bool res, bool halo);
int conv_f32tc_b_stage_bytes(int bn, int swz, bool inter);
}  // namespace tec_sm100

using namespace tec_sm100;

namespace {

thread_local std::string g_last_error;
// tec_conv_plan: when set, the launch paths record their decision here and
// return before launching anything.
thread_local tec_kernel_plan* g_plan = nullptr;
// Caller-owned workspace of the current tec_conv2d_fused_ws call (null:
// the per-(device, stream) internal pool of tec_conv2d_fused).
thread_local void* g_ws = nullptr;
thread_local size_t g_ws_bytes = 0;

bool plan_only(int family, int bn, int tile_m, int stages, int grid, int smem, int tmem_cols,
               int tma_store, int splits, int cluster) {
  if (!g_plan) return false;
  g_plan->family = family;
  g_plan->tile_n = bn;
  g_plan->tile_m = tile_m;
  g_plan->stages = stages;
  g_plan->grid = grid;
  g_plan->smem_bytes = smem;
  g_plan->tmem_cols = tmem_cols;
  g_plan->tma_store = tma_store;
  g_plan->split_k = splits;
  g_plan->cluster = cluster;
  return true;
}

int tmem_cols_for(int cols) {
  int c = 32;
  while (c < cols) c *= 2;
  return c;
}

tec_status fail(tec_status code, const std::string& msg) {
  g_last_error = msg;
  return code;
}

tec_status cuda_fail(int err, const char* what) {
  return fail(TEC_E_CUDA,
              std::string(what) + ": " +
                  cudaGetErrorString(static_cast<cudaError_t>(err)));
}

#define TEC_CUDA(call)                                  \
  do {                                                  \
    cudaError_t _e = (call);                            \
    if (_e != cudaSuccess) return cuda_fail(_e, #call); \
  } while (0)

// ------------------------------------------------ driver entry points
using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType,
                                   cuuint32_t, void*, const cuuint64_t*,
                                   const cuuint64_t*, const cuuint32_t*,
                                   const cuuint32_t*, CUtensorMapInterleave,
                                   CUtensorMapSwizzle, CUtensorMapL2promotion,
                                   CUtensorMapFloatOOBfill);
using EncodeIm2colFn = CUresult (*)(
    CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
    const cuuint64_t*, const int*, const int*, cuuint32_t, cuuint32_t,
    const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
    CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

struct DriverFns {
  EncodeTiledFn tiled = nullptr;    // cached (tensor-map cache below)
  EncodeIm2colFn im2col = nullptr;  // cached
  EncodeTiledFn raw_tiled = nullptr;
  EncodeIm2colFn raw_im2col = nullptr;
  int driver_version = 0;
  bool ok = false;
};

const DriverFns& driver_fns();

// Tensor-map cache (the library-owned state of SURVEY 8b): an encoded
// CUtensorMap is a pure function of its arguments (address, dims, strides,
// box, swizzle, ...), so eager launches reuse it instead of re-encoding on
// every call. Keyed by the argument bytes; a mutex on the map, bounded.
struct MapCache {
  std::mutex mu;
  std::map<std::string, CUtensorMap> maps;
};
MapCache& map_cache() {
  static MapCache c;
  return c;
}
template <typename T>
void key_add(std::string* k, const T* p, size_t n) {
  k->append(reinterpret_cast<const char*>(p), n * sizeof(T));
}
CUresult cached_tiled(CUtensorMap* tm, CUtensorMapDataType dt, cuuint32_t rank, void* addr,
                      const cuuint64_t* dims, const cuuint64_t* strides, const cuuint32_t* box,
                      const cuuint32_t* estr, CUtensorMapInterleave il, CUtensorMapSwizzle sw,
                      CUtensorMapL2promotion l2, CUtensorMapFloatOOBfill oob) {
  std::string k("T");
  const int64_t scal[7] = {(int64_t)dt, (int64_t)rank, (int64_t)(uintptr_t)addr, (int64_t)il,
                           (int64_t)sw, (int64_t)l2, (int64_t)oob};
  key_add(&k, scal, 7);
  key_add(&k, dims, rank);
  key_add(&k, strides, rank > 0 ? rank - 1 : 0);
  key_add(&k, box, rank);
  key_add(&k, estr, rank);
  MapCache& c = map_cache();
  {
    std::lock_guard<std::mutex> lock(c.mu);
    auto it = c.maps.find(k);
    if (it != c.maps.end()) {
      *tm = it->second;
      return CUDA_SUCCESS;
    }
  }
  const CUresult r =
      driver_fns().raw_tiled(tm, dt, rank, addr, dims, strides, box, estr, il, sw, l2, oob);
  if (r == CUDA_SUCCESS) {
    std::lock_guard<std::mutex> lock(c.mu);
    if (c.maps.size() >= 4096) c.maps.clear();
    c.maps.emplace(std::move(k), *tm);
  }
  return r;
}
CUresult cached_im2col(CUtensorMap* tm, CUtensorMapDataType dt, cuuint32_t rank, void* addr,
                       const cuuint64_t* dims, const cuuint64_t* strides, const int* lower,
                       const int* upper, cuuint32_t ch, cuuint32_t px, const cuuint32_t* estr,
                       CUtensorMapInterleave il, CUtensorMapSwizzle sw, CUtensorMapL2promotion l2,
                       CUtensorMapFloatOOBfill oob) {
  std::string k("I");
  const int64_t scal[9] = {(int64_t)dt, (int64_t)rank, (int64_t)(uintptr_t)addr, (int64_t)ch,
                           (int64_t)px, (int64_t)il, (int64_t)sw, (int64_t)l2, (int64_t)oob};
  key_add(&k, scal, 9);
  key_add(&k, dims, rank);
  key_add(&k, strides, rank > 0 ? rank - 1 : 0);
  key_add(&k, lower, rank > 2 ? rank - 2 : 0);
  key_add(&k, upper, rank > 2 ? rank - 2 : 0);
  key_add(&k, estr, rank);
  MapCache& c = map_cache();
  {
    std::lock_guard<std::mutex> lock(c.mu);
    auto it = c.maps.find(k);
    if (it != c.maps.end()) {
      *tm = it->second;
      return CUDA_SUCCESS;
    }
  }
  const CUresult r = driver_fns().raw_im2col(tm, dt, rank, addr, dims, strides, lower, upper,
                                             ch, px, estr, il, sw, l2, oob);
  if (r == CUDA_SUCCESS) {
    std::lock_guard<std::mutex> lock(c.mu);
    if (c.maps.size() >= 4096) c.maps.clear();
    c.maps.emplace(std::move(k), *tm);
  }
  return r;
}

const DriverFns& driver_fns() {
  static DriverFns fns;
  static std::once_flag once;
  std::call_once(once, [] {
    cudaDriverEntryPointQueryResult q1, q2;
    void* p1 = nullptr;
    void* p2 = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p1,
                                cudaEnableDefault, &q1) != cudaSuccess ||
        cudaGetDriverEntryPoint("cuTensorMapEncodeIm2col", &p2,
                                cudaEnableDefault, &q2) != cudaSuccess)
      return;
    fns.raw_tiled = reinterpret_cast<EncodeTiledFn>(p1);
    fns.raw_im2col = reinterpret_cast<EncodeIm2colFn>(p2);
    fns.tiled = &cached_tiled;
    fns.im2col = &cached_im2col;
    cudaDriverGetVersion(&fns.driver_version);
    fns.ok = fns.raw_tiled && fns.raw_im2col;
  });
  return fns;
}

CUtensorMapSwizzle swizzle_of(int bytes) {
  return bytes == 128  ? CU_TENSOR_MAP_SWIZZLE_128B
         : bytes == 64 ? CU_TENSOR_MAP_SWIZZLE_64B
         : bytes == 32 ? CU_TENSOR_MAP_SWIZZLE_32B
                       : CU_TENSOR_MAP_SWIZZLE_NONE;
}

// TMA store map for a float output y (bf16 / f32): `rank` dims innermost
// first (dims[0] = OC), box 32 channels x `box_px` pixels (x 1 x 1),
// swizzled to match epi::box_off. Leaves *ok false when the layout does not
// allow it (integer output, or an OC row pitch that is not a multiple of 16 B).
int elem_bytes(int32_t t) { return t == TEC_DT_I8 ? 1 : t == TEC_DT_BF16 ? 2 : 4; }

void make_store_map(CUtensorMap* tm, void* y, int32_t out_dtype, int rank,
                    const cuuint64_t* dims, int box_px, bool* ok) {
  *ok = false;
  std::memset(tm, 0, sizeof(*tm));
  if (out_dtype != TEC_DT_BF16 && out_dtype != TEC_DT_F32 && out_dtype != TEC_DT_I32 &&
      out_dtype != TEC_DT_I8)
    return;
  const int es = elem_bytes(out_dtype);
  if ((dims[0] * es) % 16 || box_px < 1 || box_px > 256) return;
  cuuint64_t strides[3];
  cuuint64_t pitch = es;
  for (int i = 0; i + 1 < rank; ++i) strides[i] = (pitch *= dims[i]);
  cuuint32_t box[4] = {32, (cuuint32_t)box_px, 1, 1};
  cuuint32_t estr[4] = {1, 1, 1, 1};
  const CUresult r = driver_fns().tiled(
      tm,
      es == 1 ? CU_TENSOR_MAP_DATA_TYPE_UINT8
      : es == 2 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16
      : out_dtype == TEC_DT_I32 ? CU_TENSOR_MAP_DATA_TYPE_INT32 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32,
      (cuuint32_t)rank, y, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
      // 32-column boxes: rows of 32 (i8), 64 (bf16) or 128 (f32 / i32) bytes,
      // each with the swizzle of its row width (conv_epilogue.cuh box_off)
      es == 1 ? CU_TENSOR_MAP_SWIZZLE_32B : es == 2 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_128B,
      CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  *ok = r == CUDA_SUCCESS;
}

// ------------------------------------------------------ layout planning

int64_t round_up(int64_t a, int64_t b) { return (a + b - 1) / b * b; }

struct Plan {
  int64_t oh, ow, m;
  int64_t cp;       // stored channels of the packed activation (all planes)
  int64_t cpp = 0;  // channels per plane (F32TC: cp = 3 * cpp, or 64 interleaved)
  bool inter = false;  // F32TC with <= 16 channels per plane: [h16|m16|l16|0] pixels
  int32_t act;      // packed element type (tec_dtype)
  int32_t acc;      // accumulator type
  int pack_mode;    // layout.cu PackMode
  int swz;          // channel-block bytes (128/64/32)
  MmaKind kind;
  // Space-to-depth stem layout (stride-2 conv on <= 4 / 8 channels): the
  // op runs as a stride-1 (r2 x s2) conv over an (h2 x w2 x cp) input.
  bool s2d = false;
  int64_t h2 = 0, w2 = 0, r2 = 0, s2 = 0;
};

tec_status infer(const tec_conv_desc* d, int64_t* oh, int64_t* ow) {
  // infer_conv (R/src/ops.cpp:163-192) plus positive-shape validation
  // (TensorType::validate, R/include/tec/dtype.hpp:78-84).
  if (!d) return fail(TEC_E_INTERNAL, "null descriptor");
  if (d->n <= 0 || d->c <= 0 || d->h <= 0 || d->w <= 0 || d->k <= 0 ||
      d->r <= 0 || d->s <= 0)
    return fail(TEC_E_SHAPE_MISMATCH, "tensor dimensions must be positive");
  if (d->stride_h <= 0 || d->stride_w <= 0 || d->pad_h < 0 || d->pad_w < 0)
    return fail(TEC_E_SHAPE_MISMATCH, "strides/padding must be pairs of valid values");
  if (d->depthwise && d->k != d->c)
    return fail(TEC_E_SHAPE_MISMATCH,
                "depthwise_conv2d weights must be [C,1,kh,kw] with C=" +
                    std::to_string(d->c));
  // The reference's truncating division (R/src/ops.cpp:187-188) accepts
  // -stride < h + 2p - r < 0 with OH = 1, and its evaluation then reads past
  // the input; a window larger than the padded input is rejected here.
  *oh = (d->h + 2 * d->pad_h - d->r) / d->stride_h + 1;
  *ow = (d->w + 2 * d->pad_w - d->s) / d->stride_w + 1;
  if (*oh <= 0 || *ow <= 0 || d->h + 2 * d->pad_h < d->r || d->w + 2 * d->pad_w < d->s)
    return fail(TEC_E_SHAPE_MISMATCH, std::string(d->depthwise ? "depthwise_conv2d" : "conv2d") +
                                          ": window larger than input");
  return TEC_OK;
}

tec_status make_plan(const tec_conv_desc* d, Plan* p) {
  tec_status st = infer(d, &p->oh, &p->ow);
  if (st) return st;
  p->m = d->n * p->oh * p->ow;
  switch (d->compute) {
    case TEC_COMPUTE_BF16:
      p->act = TEC_DT_BF16;
      p->acc = TEC_DT_F32;
      p->pack_mode = 0;
      p->kind = MmaKind::kF16;
      if (d->depthwise) {
        p->cp = d->c;
      } else {
        p->cp = round_up(d->c, 16);
        if (p->cp % 64) p->swz = 32; else p->swz = 128;
      }
      break;
    case TEC_COMPUTE_F32TC:
      p->acc = TEC_DT_F32;
      p->kind = MmaKind::kF16;
      if (d->depthwise) {
        // exact f32 SIMT path (bit-identical to the oracle's order)
        p->act = TEC_DT_F32;
        p->pack_mode = 3;
        p->cp = d->c;
      } else {
        // three exact bf16 planes [h | m | l] (conv_f32tc.cu); <= 16
        // channels per plane: interleaved in one 64-channel pixel
        p->act = TEC_DT_BF16;
        p->cpp = round_up(d->c, 16);
        p->inter = p->cpp == 16;
        p->pack_mode = p->inter ? 5 : 1;
        p->cp = p->inter ? 64 : 3 * p->cpp;
        p->swz = p->inter || p->cpp % 64 == 0 ? 128 : 32;
      }
      break;
    case TEC_COMPUTE_F32:
      // exact-order SIMT path; dense conv reads the reference NCHW layout
      // as is (pack = copy), depthwise uses the f32 NHWC kernel.
      p->act = TEC_DT_F32;
      p->acc = TEC_DT_F32;
      p->kind = MmaKind::kTF32;  // unused
      p->pack_mode = d->depthwise ? 3 : -1;
      p->cp = d->c;
      break;
    case TEC_COMPUTE_I8:
      p->act = TEC_DT_I8;
      p->acc = TEC_DT_I32;
      p->pack_mode = 2;
      p->kind = MmaKind::kI8;
      if (d->depthwise) {
        p->cp = d->c;
      } else {
        p->cp = round_up(d->c, 32);
        p->swz = p->cp % 128 == 0 ? 128 : p->cp % 64 == 0 ? 64 : 32;
      }
      break;
    default:
      return fail(TEC_E_LOWERING, "unknown compute mode " + std::to_string(d->compute));
  }
  // Strided stem on few channels -> space-to-depth, when the folded
  // stride-1 conv has exactly the same output grid.
  const int64_t s2d_c = d->compute == TEC_COMPUTE_BF16 || d->compute == TEC_COMPUTE_F32TC ? 16
                        : d->compute == TEC_COMPUTE_I8                                    ? 32
                                                                                          : 0;
  if (!d->depthwise && s2d_c && d->stride_h == 2 && d->stride_w == 2 && 4 * d->c <= s2d_c) {
    const int64_t h2 = (d->h + 2 * d->pad_h + 1) / 2, w2 = (d->w + 2 * d->pad_w + 1) / 2;
    const int64_t r2 = (d->r + 1) / 2, s2 = (d->s + 1) / 2;
    if (h2 - r2 + 1 == p->oh && w2 - s2 + 1 == p->ow && h2 <= 65535 && w2 <= 256) {
      p->s2d = true;
      p->h2 = h2; p->w2 = w2; p->r2 = r2; p->s2 = s2;
      p->cpp = s2d_c;
      p->swz = 32;
      if (d->compute == TEC_COMPUTE_F32TC) {  // interleaved planes
        p->inter = true;
        p->pack_mode = 5;
        p->cp = 64;
        p->swz = 128;
      } else {
        p->cp = s2d_c;
      }
    }
  }
  return TEC_OK;
}

tec_status build_epilogue(const tec_epilogue* e, bool integer, EpilogueParams* out) {
  std::memset(out, 0, sizeof(*out));
  if (!e) return TEC_OK;
  if (e->n_ops < 0 || e->n_ops > kMaxEpi)
    return fail(TEC_E_LOWERING, "too many fused epilogue members");
  out->n_ops = e->n_ops;
  int n_bias = 0, n_add = 0, n_mul = 0;
  for (int i = 0; i < e->n_ops; ++i) {
    n_bias += e->ops[i] == TEC_EPI_BIAS;
    n_add += e->ops[i] == TEC_EPI_ADD;
    n_mul += e->ops[i] == TEC_EPI_MUL;
  }
  // one operand pointer per kind: a repeated member would read the same operand
  if (n_bias > 1 || n_add > 1 || n_mul > 1)
    return fail(TEC_E_LOWERING, "more than one bias_add / add / mul member in one fused conv");
  for (int i = 0; i < e->n_ops; ++i) {
    const int op = e->ops[i];
    if (op < TEC_EPI_SCALE || op > TEC_EPI_REQUANTIZE)
      return fail(TEC_E_UNKNOWN_OPERATOR, "unknown epilogue op " + std::to_string(op));
    if (op == TEC_EPI_REQUANTIZE) {
      if (!integer) return fail(TEC_E_SHAPE_MISMATCH, "requantize wants i32 data (I8 compute)");
      if (i != e->n_ops - 1) return fail(TEC_E_LOWERING, "requantize must be the last member");
      if (e->rq_mult < 1 || e->rq_mult >= (int64_t(1) << 31) || e->rq_shift < 0 || e->rq_shift > 62)
        return fail(TEC_E_SHAPE_MISMATCH, "requantize needs 1 <= multiplier < 2^31, 0 <= shift <= 62");
    }
    out->ops[i] = op;
    if (op == TEC_EPI_SCALE) {
      const double c = e->scale[i];
      if (integer && c != std::floor(c))
        return fail(TEC_E_SHAPE_MISMATCH, "integer scale requires an integral factor");
      out->fscale[i] = static_cast<float>(c);           // cstf(c)
      out->iscale[i] = static_cast<int64_t>(c);         // cst(int64(c))
    }
    if (op == TEC_EPI_BIAS && !e->bias)
      return fail(TEC_E_SHAPE_MISMATCH, "bias_add needs a bias operand");
    if (op == TEC_EPI_ADD && !e->residual)
      return fail(TEC_E_SHAPE_MISMATCH, "add needs a second operand");
    if (op == TEC_EPI_MUL && !e->mul_operand)
      return fail(TEC_E_SHAPE_MISMATCH, "mul needs a second operand");
  }
  if (e->residual_i8) {
    if (!integer || !n_add) return fail(TEC_E_LOWERING, "an i8 residual needs I8 compute and an add");
    if (e->residual_scale < -(int64_t(1) << 24) || e->residual_scale > (int64_t(1) << 24))
      return fail(TEC_E_LOWERING, "|residual_scale| > 2^24");
  }
  out->bias = e->bias;
  out->residual = e->residual;
  out->mul_operand = e->mul_operand;
  out->rq_mult = e->rq_mult;
  out->rq_shift = e->rq_shift;
  out->res_i8 = e->residual_i8 ? 1 : 0;
  out->res_scale = e->residual_i8 ? e->residual_scale : 1;
  return TEC_OK;
}

// The requantize member (last) makes y i8.
bool epi_requant(const EpilogueParams& e) { return e.n_ops > 0 && e.ops[e.n_ops - 1] == kEpiRequant; }

// I8 output / i8 residual constraints the kernels rely on (whole 16-byte
// i8 vectors per row, the coalesced / TMA epilogues).
tec_status check_int8_epilogue(const EpilogueParams& e, const tec_conv_desc* d, int32_t out_dtype,
                               const tec_knobs* kn) {
  const bool rq = epi_requant(e);
  if (rq != (out_dtype == TEC_DT_I8))
    return fail(TEC_E_SHAPE_MISMATCH, rq ? "a requantize epilogue writes i8 (out_dtype I8)"
                                         : "i8 output needs a requantize member");
  if ((rq || e.res_i8) && (d->k % (e.res_i8 ? 32 : 16) || (kn && kn->vec != 0)))
    return fail(TEC_E_LOWERING, "i8 output / i8 residual: K a multiple of 16 (32 with an i8 "
                                "residual) and the default epilogue");
  return TEC_OK;
}

int sm_count(int dev) {
  int n = 148;
  cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
  return n;
}

// ------------------------------------------------------ dense conv launch
using Launcher = int (*)(const CUtensorMap&, const CUtensorMap&, const CUtensorMap&,
                         const ConvGemmParams&, int, cudaStream_t);

Launcher pick_launcher(MmaKind kind, int bn, int swz, bool pair = false) {
#define TEC_CASE_PAIR(K, BN, ST, SW) \
  if (pair && kind == K && bn == BN && swz == SW) return &launch_conv_fprop_tc<K, BN, ST, SW, true>;
  TEC_CASE_PAIR(MmaKind::kF16, 64, 9, 128)
  TEC_CASE_PAIR(MmaKind::kF16, 128, 8, 128)
  TEC_CASE_PAIR(MmaKind::kF16, 256, 5, 128)
  TEC_CASE_PAIR(MmaKind::kI8, 64, 9, 128)
  TEC_CASE_PAIR(MmaKind::kI8, 128, 8, 128)
  TEC_CASE_PAIR(MmaKind::kI8, 256, 5, 128)
  TEC_CASE_PAIR(MmaKind::kI8, 64, 9, 64)
  TEC_CASE_PAIR(MmaKind::kI8, 128, 8, 64)
#undef TEC_CASE_PAIR
  if (pair) return nullptr;
#define TEC_CASE(K, BN, ST, SW) \
  if (kind == K && bn == BN && swz == SW) return &launch_conv_fprop_tc<K, BN, ST, SW, false>;
  TEC_CASE(MmaKind::kF16, 64, 8, 128)
  TEC_CASE(MmaKind::kF16, 128, 6, 128)
  TEC_CASE(MmaKind::kF16, 256, 3, 128)
  TEC_CASE(MmaKind::kF16, 64, 8, 32)
  TEC_CASE(MmaKind::kI8, 64, 8, 128)
  TEC_CASE(MmaKind::kI8, 128, 6, 128)
  TEC_CASE(MmaKind::kI8, 256, 3, 128)
  TEC_CASE(MmaKind::kI8, 64, 8, 64)
  TEC_CASE(MmaKind::kI8, 128, 6, 64)
  TEC_CASE(MmaKind::kI8, 64, 8, 32)
#undef TEC_CASE
  return nullptr;
}

// ------------------------------------------- shifted-window (halo) path
using HaloLauncher = int (*)(const CUtensorMap&, const CUtensorMap&, const CUtensorMap&,
                             const ConvHaloParams&, int, cudaStream_t);
struct HaloInst {
  MmaKind kind;
  int bn, ms, swz, wstages;
  HaloLauncher fn;
  bool pair;  // paired taps (conv_halo.cu, kPair)
};
#define TEC_H(K, BN, MS, SW, WS) {K, BN, MS, SW, WS, &launch_conv_halo<K, BN, MS, SW, WS, false>, false}
#define TEC_HP(K, BN, MS, SW, WS) {K, BN, MS, SW, WS, &launch_conv_halo<K, BN, MS, SW, WS, true>, true}
const HaloInst kHaloInsts[] = {
    TEC_H(MmaKind::kF16, 64, 1, 128, 6),  TEC_H(MmaKind::kF16, 64, 2, 128, 6),
    TEC_H(MmaKind::kF16, 64, 4, 128, 4),  TEC_H(MmaKind::kF16, 128, 1, 128, 6),
    TEC_H(MmaKind::kF16, 128, 2, 128, 4), TEC_H(MmaKind::kF16, 256, 1, 128, 4),
    TEC_H(MmaKind::kF16, 64, 2, 32, 8),   TEC_H(MmaKind::kF16, 64, 4, 32, 8),
    TEC_H(MmaKind::kI8, 64, 1, 128, 6),   TEC_H(MmaKind::kI8, 128, 1, 128, 6),
    TEC_H(MmaKind::kI8, 64, 2, 128, 6),   TEC_H(MmaKind::kI8, 64, 4, 128, 4),
    TEC_H(MmaKind::kI8, 128, 2, 128, 4),  TEC_H(MmaKind::kI8, 256, 1, 128, 4),
    TEC_H(MmaKind::kI8, 64, 2, 64, 6),    TEC_H(MmaKind::kI8, 64, 4, 64, 6),
    TEC_H(MmaKind::kI8, 64, 1, 32, 8),    TEC_H(MmaKind::kI8, 64, 1, 64, 6),
    TEC_H(MmaKind::kI8, 64, 2, 32, 8),    TEC_H(MmaKind::kI8, 64, 4, 32, 8),
    TEC_HP(MmaKind::kF16, 64, 1, 128, 6), TEC_HP(MmaKind::kF16, 64, 2, 128, 6),
    TEC_HP(MmaKind::kF16, 64, 1, 32, 8),  TEC_HP(MmaKind::kF16, 64, 2, 32, 8),
};
#undef TEC_H
#undef TEC_HP

constexpr int kStageMin = 8 * 4096;  // epilogue stage: 8 warps x 4 KB
constexpr int kSmemMax = 227 * 1024;

struct HaloChoice {
  const HaloInst* inst = nullptr;
  int th = 0, halo_px = 0, bands = 0, n_tiles = 0, tiles = 0;
  int resident = 0, w_slots = 0, grid = 0;
  int cl = 1;  // cluster size of the weight multicast (streamed weights)
};

// Picks (BN, MS, rows per tile) by a two-term model per tile --
// max(MMA cycles, L2->SM bytes / 40 B/cycle) -- times the number of waves
// over the SMs. Returns false when no halo instance fits.
// pair_ok: the epilogue program has the TMA-store path the paired-tap
// instances need (kPair). Knob tile_k: 2 = halo without pairing, 4 = paired.
// Padded halo row width: even (bf16 / f32 / i32 output) or a multiple of 4
// (i8 output), so every output row of the group-staged TMA epilogue starts
// on a 128-byte boundary (wp * 32 * elem % 128 == 0).
int halo_wp(const tec_conv_desc* d, int32_t out_dtype) {
  const int64_t a = out_dtype == TEC_DT_I8 ? 4 : 2;
  return (int)((d->w + 2 * d->pad_w + a - 1) / a * a);
}

bool plan_halo(const tec_conv_desc* d, const Plan& pl, const tec_knobs* kn, int sms,
               int32_t out_dtype, bool pair_ok, HaloChoice* out) {
  if (d->stride_h != 1 || d->stride_w != 1) return false;
  const int wp = halo_wp(d, out_dtype);
  const int es = elem_bytes(pl.act);
  if (wp > 256 || (pl.oh + d->r - 1) < 1) return false;
  double best = 1e30;
  for (const HaloInst& hi : kHaloInsts) {
    if (hi.kind != pl.kind || hi.swz != pl.swz) continue;
    if (kn && kn->tile_n && kn->tile_n != hi.bn) continue;
    if (kn && kn->tile_m && kn->tile_m != 128 * hi.ms) continue;
    if (hi.bn > 64 && hi.bn > d->k) continue;
    // Paired taps only on request (knob tile_k = 4): they cut the MMA time
    // (C2: 54 -> 39 cycles per tap-equivalent) but double the accumulator the
    // epilogue reads from TMEM, and the epilogue then bounds the ResNet
    // layers (C2 b64: 25.0 us paired vs 23.8 us plain, C1: 58 vs 43).
    if (hi.pair && (!pair_ok || d->s < 2 || !(kn && kn->tile_k == 4) ||
                    (kn && (kn->stages == 1 || kn->cluster_n > 1))))
      continue;
    if (!hi.pair && kn && kn->tile_k == 4) continue;
    const int th = (int)std::min<int64_t>(pl.oh, (128 * hi.ms) / wp);
    if (th < 1 || th + d->r - 1 > 256) continue;
    // Small images waste most MMA rows on junk virtual rows / padding: keep
    // the halo form for tiles that are at least half real outputs.
    if (!(kn && (kn->tile_k == 2 || kn->tile_k == 4)) && 2 * th * pl.ow < 128 * hi.ms) continue;
    const int halo_px = 128 * hi.ms + (int)((d->r - 1) * wp + d->s) + 8;
    const int bands = (int)((pl.oh + th - 1) / th);
    const int n_tiles = (int)((d->k + hi.bn - 1) / hi.bn);
    const int64_t spatial = d->n * bands;
    const int64_t tiles = spatial * n_tiles;
    const int taps_cb = (int)(d->r * d->s * (pl.cp * es / hi.swz));
    const double ktot = (double)d->r * d->s * pl.cp;
    double mma = 128.0 * hi.ms * hi.bn * ktot * 2 / 8192.0 *
                 (pl.kind == MmaKind::kTF32 ? 2 : pl.kind == MmaKind::kI8 ? 0.5 : 1);
    if (hi.pair)  // measured N=128 64 cycles vs N=64 54 (tools/microbench/RESULTS.md)
      mma *= ((d->s / 2) * 64.0 + (d->s % 2) * 54.0) / (d->s * 54.0);
    const double halo_bytes = (double)(th + d->r - 1) * wp * pl.cp * es;
    // Epilogue term: the group-staged TMA-store path (run_conv_halo) moves
    // ~48 B/cycle of output, the SIMT fallback ~12 (measured, round 1).
    const int rowb = 32 * elem_bytes(out_dtype);
    const int cbytes = hi.ms * 128 * rowb;  // one 32-column chunk of a tile
    // knob `stages`: 0 auto, 1 streamed weight ring, 2 resident weights
    for (int res = 0; res < 2; ++res) {
      if (kn && kn->stages == 1 && res) continue;
      if (kn && kn->stages == 2 && !res) continue;
      const int w_slots = res ? taps_cb : hi.wstages;
      static const bool dbg = std::getenv("TEC_SM100_PLAN_DEBUG") != nullptr;
      if (dbg)
        std::fprintf(stderr, "[tec-plan] halo bn=%d ms=%d swz=%d res=%d th=%d smem=%d\n", hi.bn,
                     hi.ms, hi.swz, res, th,
                     conv_halo_smem_bytes(hi.bn, hi.swz, w_slots, halo_px, kStageMin, hi.ms, hi.pair));
      if (conv_halo_smem_bytes(hi.bn, hi.swz, w_slots, halo_px, kStageMin, hi.ms, hi.pair) > kSmemMax) continue;
      // The TMA-store epilogue needs one chunk per epilogue group in the stage.
      const bool tma_epi =
          (wp * rowb) % 128 == 0 &&
          conv_halo_smem_bytes(hi.bn, hi.swz, w_slots, halo_px, std::max(kStageMin, 2 * cbytes), hi.ms, hi.pair) <=
              kSmemMax;
      const double epi = (double)th * pl.ow * std::min<int64_t>(hi.bn, d->k) *
                         elem_bytes(out_dtype) / (tma_epi ? 48.0 : 12.0);
      // knob cluster_n: 0 / 1 no multicast, 2 weight multicast over CTA
      // pairs. Not chosen automatically: measured slower on ResNet layers
      // (the pair runs in lockstep on the weight ring), so only the tuner
      // or an explicit knob enables it.
      for (int cl = 1; cl <= 2; ++cl) {
        if (cl != (kn && kn->cluster_n ? kn->cluster_n : 1)) continue;
        if (cl > 1 && (res || hi.bn / cl < 8 || sms < 2)) continue;
        int grid;
        double per_tile, waves;
        if (res) {
          const int per_n = (int)std::min<int64_t>(sms / n_tiles, spatial);
          if (per_n < 1) continue;
          grid = per_n * n_tiles;
          waves = (double)((spatial + per_n - 1) / per_n);
          per_tile = std::max(std::max(mma, halo_bytes / 40.0), epi);
        } else {
          const int64_t units = ((spatial + cl - 1) / cl) * n_tiles;
          const int64_t clusters = std::min<int64_t>(units, sms / cl);
          grid = (int)(clusters * cl);
          waves = (double)((units + clusters - 1) / clusters);
          per_tile = std::max(std::max(mma, ((double)hi.bn * ktot * es / cl + halo_bytes) / 40.0),
                              epi);
        }
        const double cost = waves * per_tile;
        if (cost < best) {
          best = cost;
          out->inst = &hi;
          out->th = th;
          out->halo_px = halo_px;
          out->bands = bands;
          out->n_tiles = n_tiles;
          out->tiles = (int)tiles;
          out->resident = res;
          out->w_slots = w_slots;
          out->grid = grid;
          out->cl = cl;
        }
      }
    }
  }
  return out->inst != nullptr;
}

tec_status run_conv_halo(const tec_conv_desc* d, const Plan& pl, const HaloChoice& hc,
                         const EpilogueParams& epi, const tec_knobs* kn, const void* x,
                         const void* w, void* y, int32_t out_dtype, int32_t* err,
                         cudaStream_t st, int sms) {
  const DriverFns& fns = driver_fns();
  const int es = elem_bytes(pl.act);
  const int cb = pl.swz / es;
  const int wp = halo_wp(d, out_dtype);
  const CUtensorMapDataType tdt = pl.act == TEC_DT_BF16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16
                                  : pl.act == TEC_DT_I8 ? CU_TENSOR_MAP_DATA_TYPE_UINT8
                                                        : CU_TENSOR_MAP_DATA_TYPE_FLOAT32;
  CUtensorMap tm_x, tm_w;
  {
    cuuint64_t dims[4] = {(cuuint64_t)pl.cp, (cuuint64_t)d->w, (cuuint64_t)d->h,
                          (cuuint64_t)d->n};
    cuuint64_t strides[3] = {(cuuint64_t)(pl.cp * es), (cuuint64_t)(pl.cp * es * d->w),
                             (cuuint64_t)(pl.cp * es * d->w * d->h)};
    cuuint32_t box[4] = {(cuuint32_t)cb, (cuuint32_t)wp, (cuuint32_t)(hc.th + d->r - 1), 1};
    cuuint32_t estr[4] = {1, 1, 1, 1};
    CUresult r = fns.tiled(&tm_x, tdt, 4, const_cast<void*>(x), dims, strides, box, estr,
                           CU_TENSOR_MAP_INTERLEAVE_NONE, swizzle_of(pl.swz),
                           CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                           CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS)
      return fail(TEC_E_CUDA, "cuTensorMapEncodeTiled (halo) failed: " + std::to_string(r));
  }
  {
    const int64_t ktot = d->r * d->s * pl.cp;
    cuuint64_t dims[2] = {(cuuint64_t)ktot, (cuuint64_t)d->k};
    cuuint64_t strides[1] = {(cuuint64_t)(ktot * es)};
    cuuint32_t box[2] = {(cuuint32_t)cb, (cuuint32_t)(hc.inst->bn / hc.cl)};  // multicast slice
    cuuint32_t estr[2] = {1, 1};
    CUresult r = fns.tiled(&tm_w, tdt, 2, const_cast<void*>(w), dims, strides, box, estr,
                           CU_TENSOR_MAP_INTERLEAVE_NONE, swizzle_of(pl.swz),
                           CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                           CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS)
      return fail(TEC_E_CUDA, "cuTensorMapEncodeTiled (weights) failed: " + std::to_string(r));
  }
  ConvHaloParams p{};
  p.n = (int32_t)d->n; p.h = (int32_t)d->h; p.w = (int32_t)d->w; p.cp = (int32_t)pl.cp;
  p.oh = (int32_t)pl.oh; p.ow = (int32_t)pl.ow; p.oc = (int32_t)d->k;
  p.r = (int32_t)d->r; p.s = (int32_t)d->s;
  p.ph = (int32_t)d->pad_h; p.pw = (int32_t)d->pad_w;
  p.th = hc.th; p.wp = wp; p.bands = hc.bands; p.n_tiles = hc.n_tiles;
  p.cblocks = (int32_t)(pl.cp / cb);
  p.halo_px = hc.halo_px;
  p.resident = hc.resident;
  p.w_slots = hc.w_slots;
  p.cl = hc.cl;
  // knob acc_bufs: TMEM accumulator buffers (2 or 4; 0 = 4 when they fit)
  if (kn && kn->acc_bufs && kn->acc_bufs != 2 && kn->acc_bufs != 4)
    return fail(TEC_E_LOWERING, "acc_bufs must be 2 or 4");
  p.nacc = kn && kn->acc_bufs ? (int32_t)kn->acc_bufs : 4;
  p.out_type = out_dtype;
  p.y = y;
  p.err = err;
  p.epi = epi;
  // knob vec: 1 = per-thread epilogue rows, 2 = no epilogue (diagnostic only)
  p.epi_mode = kn && (kn->vec == 1 || kn->vec == 2) ? (int32_t)kn->vec : 0;
  CUtensorMap tm_y;
  {
    cuuint64_t dims[4] = {(cuuint64_t)d->k, (cuuint64_t)pl.ow, (cuuint64_t)pl.oh,
                          (cuuint64_t)d->n};
    // Group-staged TMA epilogue (conv_halo.cu): the tile's MS*128 virtual
    // rows x 32 columns must fit a group's 16 KB stage, and every output
    // row's first virtual row must sit on a 128-byte boundary.
    const int rowb = 32 * elem_bytes(out_dtype);
    bool ok = false;
    const int cbytes = hc.inst->ms * 128 * rowb;
    const int stage1 = std::max(kStageMin, 2 * cbytes);  // one chunk per group
    if ((wp * rowb) % 128 == 0 &&
        conv_halo_smem_bytes(hc.inst->bn, hc.inst->swz, hc.w_slots, hc.halo_px, stage1, hc.inst->ms, hc.inst->pair) <=
            kSmemMax)
      make_store_map(&tm_y, y, out_dtype, 4, dims, (int)pl.ow, &ok);
    else std::memset(&tm_y, 0, sizeof(tm_y));
    // Room left in shared memory -> a 2-chunk ring per group, so one chunk
    // is written while the previous one's TMA stores drain.
    p.stage_bytes = ok ? stage1 : kStageMin;
    if (ok && 4 * cbytes > p.stage_bytes &&
        conv_halo_smem_bytes(hc.inst->bn, hc.inst->swz, hc.w_slots, hc.halo_px, 4 * cbytes, hc.inst->ms, hc.inst->pair) <=
            kSmemMax)
      p.stage_bytes = 4 * cbytes;
    p.tma_store = ok && !(kn && kn->vec == 3) ? 1 : 0;  // vec 3: SIMT stores
  }
  int grid = hc.grid;
  if (kn && kn->grid > 0 && !hc.resident)
    grid = (int)std::min<int64_t>(grid, kn->grid / hc.cl * hc.cl);
  if (grid < hc.cl) return fail(TEC_E_LOWERING, "grid smaller than the cluster");
  static const bool prof = std::getenv("TEC_SM100_PROFILE") != nullptr;
  unsigned long long* dbg = nullptr;
  if (prof) {
    TEC_CUDA(cudaMalloc(&dbg, 16 * sizeof(unsigned long long)));
    TEC_CUDA(cudaMemsetAsync(dbg, 0, 16 * sizeof(unsigned long long), st));
    p.dbg = dbg;
  }
  if (hc.inst->pair && !p.tma_store)
    return fail(TEC_E_INTERNAL, "paired-tap halo instance without its TMA-store epilogue");
  if (plan_only(TEC_KERNEL_HALO, hc.inst->bn, 128 * hc.inst->ms, hc.resident ? 2 : 1, grid,
                conv_halo_smem_bytes(hc.inst->bn, hc.inst->swz, hc.w_slots, hc.halo_px,
                                     p.stage_bytes, hc.inst->ms, hc.inst->pair),
                tmem_cols_for((4 * hc.inst->ms * hc.inst->bn * (hc.inst->pair ? 2 : 1) <= 512 ? 4 : 2) *
                              hc.inst->ms * hc.inst->bn * (hc.inst->pair ? 2 : 1)),
                p.tma_store, 1, hc.cl))
    return TEC_OK;
  const int e = hc.inst->fn(tm_x, tm_w, tm_y, p, grid, st);
  if (e) return cuda_fail(e, "conv_halo launch");
  if (prof) {
    unsigned long long h[16];
    TEC_CUDA(cudaMemcpyAsync(h, dbg, sizeof(h), cudaMemcpyDeviceToHost, st));
    TEC_CUDA(cudaStreamSynchronize(st));
    cudaFree(dbg);
    const double ctas = (double)grid;
    std::fprintf(stderr,
                 "[tec-prof] halo cl=%d tma_store=%d stage=%d bn=%d ms=%d th=%d wp=%d taps=%d cblocks=%d tiles/cta=%.2f "
                 "cta_cycles=%.0f | prod_wait_empty=%.0f mma_wait_data=%.0f mma_wait_acc=%.0f "
                 "epi_wait_acc=%.0f epi_busy=%.0f | blk_tmem=%.0f blk_ops=%.0f blk_store=%.0f "
                 "(per CTA)\n",
                 p.cl, p.tma_store, p.stage_bytes, hc.inst->bn, hc.inst->ms, hc.th, wp, (int)(d->r * d->s), p.cblocks,
                 h[6] / ctas, h[5] / ctas, h[0] / ctas, h[1] / ctas, h[2] / ctas, h[3] / ctas,
                 h[4] / ctas, h[8] / ctas, h[9] / ctas, h[10] / ctas);
  }
  return TEC_OK;
}

// The epilogue programs with a compile-time fast path (epi::classify_prog).
bool fast_program(const EpilogueParams& e) {
  if (e.n_ops == 0) return true;
  if (e.n_ops == 1) return e.ops[0] == kEpiBias;
  return e.n_ops == 2 && e.ops[0] == kEpiBias && e.ops[1] == kEpiRelu;
}

// Split-K scratch layout: [per-tile arrival counters: a FIXED kSplitKTiles
// slots][f32 partial tiles]. The counters are zero before the first launch
// and every launch leaves them zero (the last split of a tile resets its
// counter); because their region has the same size for every shape, one
// scratch can serve launches of different shapes (a plan's steps, the
// per-stream pool) without a counter ever landing on stale partial sums.
constexpr size_t kSplitKTiles = 1 << 16;
constexpr size_t kSplitKCounterBytes = kSplitKTiles * sizeof(int32_t);
size_t splitk_bytes(size_t partial_bytes, size_t /*tiles*/) {
  return kSplitKCounterBytes + ((partial_bytes + 255) & ~size_t(255));
}

// The scratch a split-K launch uses: the caller's (tec_conv2d_fused_ws /
// a tec_plan's own buffer), else an internal pool per (device, stream) --
// grow-only: a buffer a captured CUDA graph may still reference is never
// freed, and launches on different streams never share tile counters.
// Growing is a synchronous allocation, refused during stream capture.
tec_status splitk_workspace(int dev, size_t partial_bytes, size_t tiles, cudaStream_t st,
                            float** ws, int32_t** cnt) {
  if (tiles > kSplitKTiles)
    return fail(TEC_E_LOWERING, "split-K over more than 65536 output tiles");
  const size_t need = splitk_bytes(partial_bytes, tiles);
  uint8_t* base = nullptr;
  if (g_ws) {
    if (g_ws_bytes < need)
      return fail(TEC_E_CAPACITY, "workspace too small: " + std::to_string(g_ws_bytes) + " < " +
                                      std::to_string(need) + " bytes (tec_workspace_bytes)");
    base = static_cast<uint8_t*>(g_ws);
  } else {
    struct Pool { void* p = nullptr; size_t bytes = 0; };
    static std::mutex mu;
    static std::map<std::pair<int, cudaStream_t>, Pool> pools;
    static std::vector<void*> retired;  // kept alive: captured graphs may use them
    std::lock_guard<std::mutex> lock(mu);
    Pool& pool = pools[{dev, st}];
    if (pool.bytes < need) {
      cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
      cudaStreamIsCapturing(st, &cs);
      if (cs != cudaStreamCaptureStatusNone)
        return fail(TEC_E_LOWERING, "split-K workspace must be sized by an eager launch before "
                                    "capture (or pass one: tec_conv2d_fused_ws)");
      void* p = nullptr;
      TEC_CUDA(cudaMalloc(&p, need));
      TEC_CUDA(cudaMemsetAsync(p, 0, need, st));
      if (pool.p) retired.push_back(pool.p);
      pool.p = p;
      pool.bytes = need;
    }
    base = static_cast<uint8_t*>(pool.p);
  }
  *cnt = reinterpret_cast<int32_t*>(base);
  *ws = reinterpret_cast<float*>(base + kSplitKCounterBytes);
  return TEC_OK;
}

tec_status run_conv(const tec_conv_desc* d, const Plan& pl,
                    const EpilogueParams& epi, const tec_knobs* kn,
                    const void* x, const void* w, void* y, int32_t out_dtype,
                    int32_t* err, cudaStream_t st) {
  const DriverFns& fns = driver_fns();
  if (!fns.ok) return fail(TEC_E_CUDA, "cuTensorMapEncode* entry points unavailable");
  const int es = elem_bytes(pl.act);
  const int cb = pl.swz / es;  // channels per block
  if (pl.cp % cb) return fail(TEC_E_INTERNAL, "channel padding does not match block");
  if (pl.kind == MmaKind::kI8 && out_dtype != TEC_DT_I32 && out_dtype != TEC_DT_I8)
    return fail(TEC_E_LOWERING, "int8 conv produces i32 (i8 after a requantize member)");
  if (pl.kind != MmaKind::kI8 && out_dtype != TEC_DT_F32 && out_dtype != TEC_DT_BF16)
    return fail(TEC_E_LOWERING, "float conv produces f32 or bf16");

  int dev = 0;
  cudaGetDevice(&dev);
  const int sms = sm_count(dev);
  // Path: knob tile_k selects the A-operand strategy -- 0 auto, 1 im2col
  // TMA (conv_tc.cu), 2 shifted-window halo (conv_halo.cu, stride 1 only),
  // 4 halo with paired filter taps (N=128 MMAs, conv_halo.cu kPair).
  const int64_t path = kn ? kn->tile_k : 0;
  // knob cluster_n on the im2col path: 2 = CTA pairs (cta_group::2, M = 256,
  // each CTA loading half the weight rows); the halo path multicasts weights
  if (path == 1 && kn && kn->cluster_n > 2)
    return fail(TEC_E_LOWERING, "cluster_n on the im2col path is 1 or 2 (CTA pair)");
  if ((path == 2 || path == 4) && kn && kn->split_k > 1)
    return fail(TEC_E_LOWERING, "split_k applies to the im2col path (tile_k=1)");
  if (path != 1 && !(kn && kn->split_k > 1)) {
    // paired taps need the TMA-store epilogue program (conv_halo.cu tma_epi)
    const bool res_prog = epi.n_ops == 3 && epi.ops[0] == kEpiBias && epi.ops[1] == kEpiAdd &&
                          epi.ops[2] == kEpiRelu;
    const bool pair_ok = pl.kind == MmaKind::kF16 && !(kn && kn->vec != 0) &&
                         (fast_program(epi) || (res_prog && pl.swz == 128 && d->k % 32 == 0));
    HaloChoice hc;
    if (plan_halo(d, pl, kn, sms, out_dtype, pair_ok, &hc))
      return run_conv_halo(d, pl, hc, epi, kn, x, w, y, out_dtype, err, st, sms);
    if (path == 2 || path == 4) return fail(TEC_E_LOWERING, "no halo configuration for this conv");
  }
  const int64_t m_tiles = (pl.m + 127) / 128;

  // tile_n knob: the "split" of the OC axis.
  int bn = kn && kn->tile_n ? static_cast<int>(kn->tile_n) : 0;
  if (!bn) {  // widest tile that still gives ~0.6 x #SMs output tiles
    bn = d->k >= 256 ? 256 : d->k >= 128 ? 128 : 64;
    if (pl.swz != 128) bn = 64;
    while (bn > 64 && m_tiles * ((d->k + bn - 1) / bn) * 5 < 3 * sms) bn /= 2;
  }
  const bool pair = kn && kn->cluster_n == 2;
  Launcher launch = pick_launcher(pl.kind, bn, pl.swz, pair);
  if (!launch)
    return fail(TEC_E_LOWERING, "no sm100 conv instance for tile_n=" +
                                    std::to_string(bn) + " block=" +
                                    std::to_string(pl.swz) + "B" + (pair ? " (CTA pair)" : ""));
  if (pair && kn->split_k > 1) return fail(TEC_E_LOWERING, "CTA pairs do not split K");
  if (kn && kn->tile_m && kn->tile_m != 128)
    return fail(TEC_E_LOWERING, "tile_m must be 128 (tcgen05 M)");

  // A: im2col TMA over the NHWC activation (dims c, w, h, n).
  CUtensorMap tm_a, tm_b;
  const CUtensorMapDataType tdt = pl.act == TEC_DT_BF16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16
                                  : pl.act == TEC_DT_I8 ? CU_TENSOR_MAP_DATA_TYPE_UINT8
                                                        : CU_TENSOR_MAP_DATA_TYPE_FLOAT32;
  {
    cuuint64_t dims[4] = {(cuuint64_t)pl.cp, (cuuint64_t)d->w, (cuuint64_t)d->h,
                          (cuuint64_t)d->n};
    cuuint64_t strides[3] = {(cuuint64_t)(pl.cp * es), (cuuint64_t)(pl.cp * es * d->w),
                             (cuuint64_t)(pl.cp * es * d->w * d->h)};
    // Bounding box of the window origins (w first, then h), as in the
    // fprop im2col convention: lower = -pad, upper = pad - (k-1).
    int lower[2] = {-(int)d->pad_w, -(int)d->pad_h};
    int upper[2] = {(int)(d->pad_w - (d->s - 1)), (int)(d->pad_h - (d->r - 1))};
    cuuint32_t estr[4] = {1, (cuuint32_t)d->stride_w, (cuuint32_t)d->stride_h, 1};
    if (lower[0] < -128 || lower[1] < -128 || upper[0] < -128 || upper[1] < -128 ||
        d->stride_w > 8 || d->stride_h > 8)
      return fail(TEC_E_LOWERING, "window outside the TMA im2col range");
    CUresult r = fns.im2col(&tm_a, tdt, 4, const_cast<void*>(x), dims, strides, lower,
                            upper, (cuuint32_t)cb, 128, estr,
                            CU_TENSOR_MAP_INTERLEAVE_NONE, swizzle_of(pl.swz),
                            CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS)
      return fail(TEC_E_CUDA, "cuTensorMapEncodeIm2col failed: " + std::to_string(r));
    // Same workaround CUTLASS applies for drivers <= 13.1 on small tensors.
    const int64_t bytes = d->n * d->h * d->w * pl.cp * es;
    if (fns.driver_version <= 13010 && bytes < 131072)
      reinterpret_cast<uint64_t*>(&tm_a)[1] &= ~(1ull << 21);
  }
  {
    const int64_t ktot = d->r * d->s * pl.cp;
    cuuint64_t dims[2] = {(cuuint64_t)ktot, (cuuint64_t)d->k};
    cuuint64_t strides[1] = {(cuuint64_t)(ktot * es)};
    // a CTA of a pair loads half of the tile's weight rows
    cuuint32_t box[2] = {(cuuint32_t)cb, (cuuint32_t)(pair ? bn / 2 : bn)};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = fns.tiled(&tm_b, tdt, 2, const_cast<void*>(w), dims, strides, box,
                           estr, CU_TENSOR_MAP_INTERLEAVE_NONE, swizzle_of(pl.swz),
                           CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                           CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS)
      return fail(TEC_E_CUDA, "cuTensorMapEncodeTiled failed: " + std::to_string(r));
  }

  ConvGemmParams p{};
  p.n = (int32_t)d->n; p.h = (int32_t)d->h; p.w = (int32_t)d->w; p.cp = (int32_t)pl.cp;
  p.oh = (int32_t)pl.oh; p.ow = (int32_t)pl.ow; p.oc = (int32_t)d->k;
  p.r = (int32_t)d->r; p.s = (int32_t)d->s;
  p.sh = (int32_t)d->stride_h; p.sw = (int32_t)d->stride_w;
  p.ph = (int32_t)d->pad_h; p.pw = (int32_t)d->pad_w;
  p.m = (int32_t)pl.m;
  p.m_tiles = (int32_t)m_tiles;
  p.n_tiles = (int32_t)((d->k + bn - 1) / bn);
  p.cblocks = (int32_t)(pl.cp / cb);
  p.out_type = out_dtype;
  p.y = y;
  p.err = err;
  p.epi = epi;
  // knob vec: 1 = per-thread epilogue rows, 2 = no epilogue (diagnostic only)
  p.epi_mode = kn && (kn->vec == 1 || kn->vec == 2) ? (int32_t)kn->vec : 0;
  // knob acc_bufs: TMEM accumulator buffers (2 or 4; 0 = 4 when they fit)
  if (kn && kn->acc_bufs && kn->acc_bufs != 2 && kn->acc_bufs != 4)
    return fail(TEC_E_LOWERING, "acc_bufs must be 2 or 4");
  p.nacc = kn && kn->acc_bufs ? (int32_t)kn->acc_bufs : 4;
  CUtensorMap tm_y;
  {
    cuuint64_t dims[2] = {(cuuint64_t)d->k, (cuuint64_t)pl.m};
    bool ok = false;
    make_store_map(&tm_y, y, out_dtype, 2, dims, 32, &ok);
    p.tma_store = ok && !(kn && kn->vec == 3) ? 1 : 0;  // vec 3: SIMT stores
  }
  const int64_t tiles = (int64_t)p.m_tiles * p.n_tiles;
  // Split-K (knob split_k; 0 = auto): more work items when the output has
  // fewer tiles than SMs (small-image, deep-K layers). Only on the TMA-store
  // fast programs of the float kinds.
  p.splits = 1;
  {
    const int k_iters = (int)(d->r * d->s * p.cblocks);
    const bool able = pl.kind != MmaKind::kI8 && p.tma_store && fast_program(epi);
    int want = kn && kn->split_k > 0 ? (int)kn->split_k : 0;
    if (want > 1 && !able)
      return fail(TEC_E_LOWERING, "split_k needs a float conv with a none/bias/bias+relu epilogue");
    // No automatic split: measured slower than more, narrower tiles on
    // every ResNet layer (the partials round-trip through L2), and it would
    // make results depend on the batch size. The tuner explores split_k.
    if (want > 1) {
      if (want > k_iters) want = k_iters;
      p.splits = want;
      p.kps = (k_iters + want - 1) / want;
    }
  }
  const size_t partials = (size_t)tiles * p.splits * 128 * bn * sizeof(float);
  if (g_plan) g_plan->workspace_bytes = p.splits > 1 ? (int64_t)splitk_bytes(partials, tiles) : 0;
  if (p.splits > 1 && !g_plan) {  // sized without allocating when only planning
    tec_status wst = splitk_workspace(dev, partials, (size_t)tiles, st, &p.ws, &p.tile_cnt);
    if (wst) return wst;
  }
  int grid = (int)std::min<int64_t>(tiles * p.splits, sms);
  if (kn && kn->grid > 0) grid = (int)std::min<int64_t>(grid, kn->grid);
  if (pair) {  // whole pairs, one per (M-tile pair, N tile) unit at most
    const int64_t units = ((m_tiles + 1) / 2) * p.n_tiles;
    int pairs = (int)std::min<int64_t>(units, sms / 2);
    if (kn->grid > 0) pairs = std::max(1, std::min(pairs, (int)kn->grid / 2));
    grid = 2 * pairs;
  }
  // TEC_SM100_PROFILE=1: per-role pipeline wait breakdown on stderr
  // (synchronises the stream; diagnostics only).
  static const bool prof = std::getenv("TEC_SM100_PROFILE") != nullptr;
  unsigned long long* dbg = nullptr;
  if (prof) {
    TEC_CUDA(cudaMalloc(&dbg, 8 * sizeof(unsigned long long)));
    TEC_CUDA(cudaMemsetAsync(dbg, 0, 8 * sizeof(unsigned long long), st));
    p.dbg = dbg;
  }
  if (plan_only(TEC_KERNEL_IM2COL, bn, pair ? 256 : 128, 0, grid, 0,
                tmem_cols_for((4 * bn <= 512 ? 4 : 2) * bn), p.tma_store, p.splits, pair ? 2 : 1))
    return TEC_OK;
  const int e = launch(tm_a, tm_b, tm_y, p, grid, st);
  if (e) return cuda_fail(e, "conv_fprop_tc launch");
  if (prof) {
    unsigned long long h[8];
    TEC_CUDA(cudaMemcpyAsync(h, dbg, sizeof(h), cudaMemcpyDeviceToHost, st));
    TEC_CUDA(cudaStreamSynchronize(st));
    cudaFree(dbg);
    const double ctas = (double)grid;
    std::fprintf(stderr,
                 "[tec-prof] im2col tma_store=%d bn=%d k_iters=%d tiles/cta=%.2f cta_cycles=%.0f | "
                 "prod_wait_empty=%.0f mma_wait_full=%.0f mma_wait_acc=%.0f "
                 "epi_wait_acc=%.0f epi_busy=%.0f (per CTA)\n",
                 p.tma_store, bn, (int)(d->r * d->s * p.cblocks), h[6] / ctas, h[5] / ctas, h[0] / ctas,
                 h[1] / ctas, h[2] / ctas, h[3] / ctas, h[4] / ctas);
  }
  return TEC_OK;
}

// ------------------------------------------- f32 on tensor cores (F32TC)
// conv_f32tc.cu: the activation and weights are three exact bf16 planes;
// six products per K16 step, the hh term folded into RN registers every
// 256 K elements. Programs: none / bias / bias+relu / bias+add+relu with an
// f32 NHWC output; anything else is a LoweringError (the exact F32 path
// runs every program).
tec_status run_conv_f32tc(const tec_conv_desc* d, const Plan& pl, const EpilogueParams& epi,
                          const tec_knobs* kn, const void* x, const void* w, void* y,
                          int32_t out_dtype, cudaStream_t st) {
  const DriverFns& fns = driver_fns();
  if (!fns.ok) return fail(TEC_E_CUDA, "cuTensorMapEncode* entry points unavailable");
  if (out_dtype != TEC_DT_F32) return fail(TEC_E_LOWERING, "f32tc produces f32");
  int prog;
  if (epi.n_ops == 0) prog = 1;
  else if (epi.n_ops == 1 && epi.ops[0] == kEpiBias) prog = 2;
  else if (epi.n_ops == 2 && epi.ops[0] == kEpiBias && epi.ops[1] == kEpiRelu) prog = 3;
  else if (epi.n_ops == 3 && epi.ops[0] == kEpiBias && epi.ops[1] == kEpiAdd &&
           epi.ops[2] == kEpiRelu) prog = 4;
  else return fail(TEC_E_LOWERING, "f32tc: fused program not supported (compute f32 runs it)");
  if (kn && kn->tile_m && kn->tile_m != 128) return fail(TEC_E_LOWERING, "tile_m must be 128 (tcgen05 M)");
  // knob cluster_n = 2: CTA pairs (cta_group::2) on the im2col path, tile_n 128
  if (kn && kn->cluster_n > 2) return fail(TEC_E_LOWERING, "f32tc: cluster_n is 1 or 2 (CTA pair)");
  const bool pair = kn && kn->cluster_n == 2;
  const int path = kn ? (int)kn->tile_k : 0;  // 0 auto, 1 im2col, 2 shifted window
  if (path != 0 && path != 1 && path != 2) return fail(TEC_E_LOWERING, "f32tc: tile_k is 1 or 2");
  const int swz = pl.swz;
  const bool inter = pl.inter;
  const int cb = inter ? 16 : swz / 2;  // channels per plane per k-iteration
  if (pl.cpp % cb) return fail(TEC_E_INTERNAL, "channel padding does not match block");
  int dev = 0;
  cudaGetDevice(&dev);
  const int sms = sm_count(dev);
  const int64_t m_tiles_i2c = (pl.m + 127) / 128;
  int bn = kn && kn->tile_n ? (int)kn->tile_n : (d->k >= 128 ? 128 : 64);
  if (!(kn && kn->tile_n)) {
    while (bn > 64 && m_tiles_i2c * ((d->k + bn - 1) / bn) * 5 < 3 * sms) bn /= 2;
  }
  if (bn != 64 && bn != 128) return fail(TEC_E_LOWERING, "f32tc: tile_n must be 64 or 128");
  const int n_tiles = (int)((d->k + bn - 1) / bn);
  const int k_iters = (int)(d->r * d->s * (pl.cpp / cb));
  const int b_stage = conv_f32tc_b_stage_bytes(bn, swz, inter);
  const int res_bytes = k_iters * b_stage;
  const int want_res = kn && kn->stages ? (int)kn->stages : 0;  // 1 streamed, 2 resident
  constexpr int kBudget = 227 * 1024;
  const int a_planes = inter ? 1 : 3;

  // ---- shifted-window (halo) plan (knob tile_k = 2): stride 1, 128-B
  // channel blocks, a tile of th output rows (th * wp <= 128 virtual rows).
  // Interleaved planes need resident weights (the only such instance); no
  // split-K. Not chosen automatically: measured no faster than the im2col
  // path on C1 (169 vs 172 us b64) and slower on C2 / C6 / C9 (134 / 126 /
  // 107 vs 86 / 70 / 70 us) -- with three planes the halo plus a weight
  // ring leave room for one halo buffer, and th > 1 tiles store per element.
  bool halo = false, res = false;
  int th = 0, wp = 0, bands = 0, halo_bytes = 0, halo_box = 0, hbuf = 0, ring_rows = 0;
  // Row ring (th == 1, one channel block, one N tile -- the stem C1): the
  // halo buffers hold single input rows, each CTA walks a contiguous range
  // of output rows, and a row is loaded once for the r rows that read it
  // (conv_f32tc.cu `ring`); TEC_SM100_F32TC_NO_RING=1 keeps per-tile boxes.
  static const bool no_ring = std::getenv("TEC_SM100_F32TC_NO_RING") != nullptr;
  if (path != 1 && d->stride_h == 1 && d->stride_w == 1 && swz == 128 &&
      !(kn && kn->split_k > 1)) {
    wp = (int)(d->w + 2 * d->pad_w);
    th = (int)std::min<int64_t>(pl.oh, 128 / std::max(1, wp));
    const int row_px = 128 + (int)d->s - 1;  // an A operand: 128 virtual rows from pixel s
    if (path == 2 && !no_ring && th == 1 && pl.cpp / cb == 1 && n_tiles == 1 && inter &&
        want_res != 1 && row_px <= 256) {
      const int fixed = conv_f32tc_smem_bytes(bn, swz, inter, true, true);
      const int row_bytes = (row_px * 128 + 1023) & ~1023;
      const int rows = fixed > 0 ? std::min(8, (kBudget - fixed - res_bytes) / row_bytes) : 0;
      if (rows >= d->r + 1) {
        halo = true;
        res = true;
        ring_rows = hbuf = rows;
        halo_bytes = row_bytes;
        halo_box = row_px * 128;
        bands = (int)pl.oh;
      }
    }
    if (path == 2 && !halo && th >= 1 && wp <= 256 && th + d->r - 1 <= 256) {
      const int halo_px = 128 + (int)((d->r - 1) * wp + d->s);
      halo_bytes = (halo_px * 128 + 1023) & ~1023;
      halo_box = 128 * wp * (int)(th + d->r - 1);
      const bool r_ = inter;  // interleaved: resident weights; others: streamed
      if (!(r_ && want_res == 1) && !(!r_ && want_res == 2)) {
        const int fixed = conv_f32tc_smem_bytes(bn, swz, inter, r_, true);
        for (int hb = 2; hb >= 1 && !halo; --hb) {
          if (fixed > 0 && fixed + hb * a_planes * halo_bytes + (r_ ? res_bytes : 0) <= kBudget) {
            halo = true;
            res = r_;
            hbuf = hb;
          }
        }
      }
      bands = (int)((pl.oh + th - 1) / th);
    }
    if (path == 2 && !halo) return fail(TEC_E_LOWERING, "f32tc: no shifted-window configuration fits");
  }
  if (path == 2 && !halo) return fail(TEC_E_LOWERING, "f32tc: the shifted window needs stride 1");
  if (pair && (halo || conv_f32tc_pair_smem_bytes(bn, swz, inter, false, false) < 0))
    return fail(TEC_E_LOWERING, "f32tc: CTA pairs run the im2col path at tile_n 128");

  CUtensorMap tm_a, tm_b, tm_y;
  if (halo) {
    // tiled 4-D map over the packed NHWC activation: one box = (128 B of
    // channels) x wp pixels x (th + r - 1) rows, padding by OOB zero fill
    cuuint64_t dims[4] = {(cuuint64_t)pl.cp, (cuuint64_t)d->w, (cuuint64_t)d->h, (cuuint64_t)d->n};
    cuuint64_t strides[3] = {(cuuint64_t)(pl.cp * 2), (cuuint64_t)(pl.cp * 2 * d->w),
                             (cuuint64_t)(pl.cp * 2 * d->w * d->h)};
    // row ring: one input row of 128 + s - 1 pixels (past the row end: zero fill)
    cuuint32_t box[4] = {64, ring_rows ? (cuuint32_t)(halo_box / 128) : (cuuint32_t)wp,
                         ring_rows ? 1u : (cuuint32_t)(th + d->r - 1), 1};
    cuuint32_t estr[4] = {1, 1, 1, 1};
    CUresult r = fns.tiled(&tm_a, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(x), dims,
                           strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                           CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                           CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS)
      return fail(TEC_E_CUDA, "cuTensorMapEncodeTiled (f32tc halo) failed: " + std::to_string(r));
  } else {
    cuuint64_t dims[4] = {(cuuint64_t)pl.cp, (cuuint64_t)d->w, (cuuint64_t)d->h,
                          (cuuint64_t)d->n};
    cuuint64_t strides[3] = {(cuuint64_t)(pl.cp * 2), (cuuint64_t)(pl.cp * 2 * d->w),
                             (cuuint64_t)(pl.cp * 2 * d->w * d->h)};
    int lower[2] = {-(int)d->pad_w, -(int)d->pad_h};
    int upper[2] = {(int)(d->pad_w - (d->s - 1)), (int)(d->pad_h - (d->r - 1))};
    cuuint32_t estr[4] = {1, (cuuint32_t)d->stride_w, (cuuint32_t)d->stride_h, 1};
    if (lower[0] < -128 || lower[1] < -128 || upper[0] < -128 || upper[1] < -128 ||
        d->stride_w > 8 || d->stride_h > 8)
      return fail(TEC_E_LOWERING, "window outside the TMA im2col range");
    CUresult r = fns.im2col(&tm_a, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(x),
                            dims, strides, lower, upper, (cuuint32_t)(swz / 2), 128, estr,
                            CU_TENSOR_MAP_INTERLEAVE_NONE, swizzle_of(swz),
                            CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS)
      return fail(TEC_E_CUDA, "cuTensorMapEncodeIm2col (f32tc) failed: " + std::to_string(r));
    const int64_t bytes = d->n * d->h * d->w * pl.cp * 2;
    if (fns.driver_version <= 13010 && bytes < 131072)
      reinterpret_cast<uint64_t*>(&tm_a)[1] &= ~(1ull << 21);
  }
  if (inter) {
    // [tap][plane][K][16]: one box {16 ch, bn rows, 3 planes} per tap lands
    // as [B_h; B_m; B_l] rows with the 32-B swizzle
    cuuint64_t dims[3] = {16, (cuuint64_t)d->k, (cuuint64_t)(3 * d->r * d->s)};
    cuuint64_t strides[2] = {32, (cuuint64_t)(d->k * 32)};
    cuuint32_t box[3] = {16, (cuuint32_t)bn, 3};
    cuuint32_t estr[3] = {1, 1, 1};
    CUresult r = fns.tiled(&tm_b, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(w), dims,
                           strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, swizzle_of(32),
                           CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS)
      return fail(TEC_E_CUDA, "cuTensorMapEncodeTiled (f32tc weights, 3-D) failed: " + std::to_string(r));
  } else {
    const int64_t ktot = d->r * d->s * pl.cp;
    cuuint64_t dims[2] = {(cuuint64_t)ktot, (cuuint64_t)d->k};
    cuuint64_t strides[1] = {(cuuint64_t)(ktot * 2)};
    // a CTA of a pair loads half of the tile's weight rows
    cuuint32_t box[2] = {(cuuint32_t)(swz / 2), (cuuint32_t)(pair ? bn / 2 : bn)};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = fns.tiled(&tm_b, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(w), dims,
                           strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, swizzle_of(swz),
                           CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS)
      return fail(TEC_E_CUDA, "cuTensorMapEncodeTiled (f32tc weights) failed: " + std::to_string(r));
  }
  // TMA-store epilogue when OC is a multiple of 32 (whole 32-column boxes
  // and residual rows) and -- shifted window -- a tile is one output row
  // ((OC, OW, N*OH) map: junk virtual rows are clipped); per-element stores
  // otherwise
  bool tma_ok = false;
  std::memset(&tm_y, 0, sizeof(tm_y));
  if (d->k % 32 == 0) {
    if (!halo) {
      cuuint64_t dims[2] = {(cuuint64_t)d->k, (cuuint64_t)pl.m};
      make_store_map(&tm_y, y, TEC_DT_F32, 2, dims, 32, &tma_ok);
    } else {
      // (OC, OW, N*OH): th == 1 -- a 32-pixel box per warp (pixels past OW
      // clipped); th > 1 -- one {32 ch, OW px} box per output row, stored
      // from the half-group's staged rows (conv_f32tc.cu `group`)
      cuuint64_t dims[3] = {(cuuint64_t)d->k, (cuuint64_t)pl.ow, (cuuint64_t)(d->n * pl.oh)};
      make_store_map(&tm_y, y, TEC_DT_F32, 3, dims, th == 1 ? 32 : (int)pl.ow, &tma_ok);
    }
  }
  ConvGemmParams p{};
  p.n = (int32_t)d->n; p.h = (int32_t)d->h; p.w = (int32_t)d->w; p.cp = (int32_t)pl.cpp;
  p.oh = (int32_t)pl.oh; p.ow = (int32_t)pl.ow; p.oc = (int32_t)d->k;
  p.r = (int32_t)d->r; p.s = (int32_t)d->s;
  p.sh = (int32_t)d->stride_h; p.sw = (int32_t)d->stride_w;
  p.ph = (int32_t)d->pad_h; p.pw = (int32_t)d->pad_w;
  p.m = (int32_t)pl.m;
  p.m_tiles = halo ? (int32_t)(d->n * bands) : (int32_t)m_tiles_i2c;
  p.n_tiles = n_tiles;
  p.cblocks = (int32_t)(pl.cpp / cb);
  p.out_type = kF32;
  p.y = y;
  p.epi = epi;
  p.tma_store = tma_ok ? 1 : 0;
  p.th = th; p.wp = wp; p.bands = bands;
  p.halo_bytes = halo_bytes; p.halo_box_bytes = halo_box; p.hbuf = hbuf; p.rows = ring_rows;
  // hh promotion chunk: 256 K elements per plane (TEC_SM100_F32TC_CHUNK
  // overrides, for the accuracy experiments only)
  static const int chunk_k = [] {
    const char* e = std::getenv("TEC_SM100_F32TC_CHUNK");
    return e ? std::max(16, std::atoi(e)) : 256;
  }();
  p.chunk_iters = std::max(1, chunk_k / cb);
  static const int fault = [] {  // test-only: the watchdog mutation test
    const char* e = std::getenv("TEC_SM100_FAULT");
    return e ? std::atoi(e) : 0;
  }();
  p.fault = fault;
  static const int producers = [] {  // experiment switch: 1 or 2 TMA issuers
    const char* e = std::getenv("TEC_SM100_F32TC_PRODUCERS");
    return e ? std::atoi(e) : 2;
  }();
  p.producers = halo ? 2 : producers;  // the halo pipeline needs its two issuers
  const int64_t tiles = (int64_t)p.m_tiles * p.n_tiles;
  // Split-K (knob split_k; 0 = auto, im2col only): for outputs with few
  // tiles, the split count with the smallest makespan waves x (k-iterations
  // per split + ~2 k-iterations of partial write/read per item).
  // knob split_k = -1: stream-K (im2col) -- every CTA takes an equal share of
  // the flattened (tile, k-iteration) work; a tile cut by a share boundary is
  // finished by its last segment. Removes the tile-count quantisation
  // (2.65 tiles per SM -> 3 rounds) at the cost of partial round trips for
  // the cut tiles. Results then depend on the grid / batch through the cuts
  // (within the f32tc bar), so it is a tuner knob, not a default.
  const bool stream_k = !halo && kn && kn->split_k == -1;
  int splits = halo || stream_k ? 1 : (kn && kn->split_k > 0 ? (int)kn->split_k : 0);
  if (!splits) {
    double best = 1e30;
    for (int sp : {1, 2, 3, 4, 6, 8}) {
      if (sp > 1 && k_iters / sp < 4) break;
      const int64_t waves = (tiles * sp + sms - 1) / sms;
      const double cost = (double)waves * ((k_iters + sp - 1) / sp + (sp > 1 ? 2 : 0));
      if (cost < best - 1e-9) { best = cost; splits = sp; }
    }
  }
  splits = std::max(1, std::min(splits, k_iters));
  p.splits = splits;
  p.kps = (k_iters + splits - 1) / splits;
  p.splits = (k_iters + p.kps - 1) / p.kps;  // no empty split
  // a pair's work unit is (M-tile pair, N tile), run by sms / 2 clusters
  const int64_t units = pair ? ((p.m_tiles + 1) / 2) * (int64_t)p.n_tiles : tiles;
  const int64_t slots = pair ? sms / 2 : sms;
  if (stream_k) {
    // segments per tile <= 1 + the share boundaries inside it
    const int64_t w = units * k_iters;
    const int64_t g = std::min<int64_t>(slots, w);
    const int64_t share = w / g;
    p.stream_k = 1;
    p.splits = (int32_t)std::min<int64_t>(k_iters, (k_iters + share - 1) / std::max<int64_t>(1, share) + 1);
    p.kps = k_iters;
  }
  const size_t partials = (size_t)tiles * p.splits * 128 * bn * sizeof(float);
  if (g_plan) g_plan->workspace_bytes = p.splits > 1 ? (int64_t)splitk_bytes(partials, tiles) : 0;
  int grid = p.stream_k ? (int)std::min<int64_t>(slots, units * k_iters)
                        : (int)std::min<int64_t>(units * p.splits, slots);
  if (kn && kn->grid > 0) grid = (int)std::min<int64_t>(grid, pair ? kn->grid / 2 : kn->grid);
  if (pair) grid = 2 * std::max(1, grid);  // whole CTA pairs
  // Resident weights (im2col: knob stages 1 streamed, 2 resident, 0 =
  // resident when they fit): every B tile of the CTA's output-channel tile
  // loaded once per CTA, the ring carries activations only -- fewer TMA
  // rows per k-step. Needs a fixed N tile per CTA: no split, grid a
  // multiple of the N tiles.
  if (!halo) {
    const int res_fixed = conv_f32tc_smem_bytes(bn, swz, inter, true, false);
    res = !pair && want_res != 1 && p.splits == 1 && !p.stream_k && res_fixed > 0 &&
          res_fixed + res_bytes <= kBudget && grid >= p.n_tiles;
    if (want_res == 2 && !res)
      return fail(TEC_E_LOWERING, "f32tc: resident weights do not fit (or split-K is on)");
  }
  if (res) {
    if (grid < p.n_tiles) return fail(TEC_E_LOWERING, "f32tc: grid smaller than the N tiles");
    grid = grid / p.n_tiles * p.n_tiles;
    p.res_bytes = res_bytes;
  }
  const int stages = conv_f32tc_stages(bn, swz, inter, res, halo);
  if (stages < 0) return fail(TEC_E_LOWERING, "f32tc: no instance for this tile / block");
  const int smem = (pair ? conv_f32tc_pair_smem_bytes(bn, swz, inter, res, halo)
                        : conv_f32tc_smem_bytes(bn, swz, inter, res, halo)) +
                   (res ? res_bytes : 0) + (halo ? hbuf * a_planes * halo_bytes : 0);
  if (plan_only(halo ? TEC_KERNEL_F32TC_HALO : TEC_KERNEL_F32TC, bn, pair ? 256 : 128,
                res ? 2 : 1, grid, smem, bn == 64 ? 512 : 4 * bn <= 256 ? 256 : 512, p.tma_store,
                p.splits, pair ? 2 : 1))
    return TEC_OK;
  if (p.splits > 1) {
    tec_status wst = splitk_workspace(dev, partials, (size_t)tiles, st, &p.ws, &p.tile_cnt);
    if (wst) return wst;
  }
  static const bool prof = std::getenv("TEC_SM100_PROFILE") != nullptr;
  unsigned long long* dbg = nullptr;
  if (prof) {  // diagnostics only: synchronises the stream
    TEC_CUDA(cudaMalloc(&dbg, 16 * sizeof(unsigned long long)));
    TEC_CUDA(cudaMemsetAsync(dbg, 0, 16 * sizeof(unsigned long long), st));
    p.dbg = dbg;
  }
  const int e = launch_conv_f32tc(tm_a, tm_b, tm_y, p, bn, swz, inter, res, halo, prog, grid, st,
                                  pair);
  if (e == -1) return fail(TEC_E_LOWERING, "f32tc: no instance for this tile / block");
  if (e) return cuda_fail(e, "conv_f32tc launch");
  if (prof) {
    unsigned long long h[16];
    TEC_CUDA(cudaMemcpyAsync(h, dbg, sizeof(h), cudaMemcpyDeviceToHost, st));
    TEC_CUDA(cudaStreamSynchronize(st));
    cudaFree(dbg);
    const double c = (double)grid;
    std::fprintf(stderr,
                 "[tec-prof] f32tc halo=%d ring=%d res=%d bn=%d inter=%d splits=%d items/cta=%.2f "
                 "cta_cycles=%.0f | prodA_wait=%.0f prodB_wait=%.0f mma_wait_tile=%.0f "
                 "mma_wait_chunk=%.0f mma_wait_data=%.0f epi_wait_chunk=%.0f epi_wait_tile=%.0f "
                 "epi_busy=%.0f (per CTA)\n",
                 (int)halo, ring_rows, (int)res, bn, (int)inter, p.splits, h[9] / c, h[8] / c, h[0] / c, h[1] / c,
                 h[2] / c, h[3] / c, h[4] / c, h[5] / c, h[6] / c, h[7] / c);
  }
  return TEC_OK;
}

// ------------------------------------------------- host-path workspace
struct DevBuf {
  void* p = nullptr;
  size_t n = 0;
};

tec_status ensure(DevBuf* b, size_t bytes) {
  if (b->n >= bytes && b->p) return TEC_OK;
  if (b->p) cudaFree(b->p);
  b->p = nullptr;
  b->n = 0;
  TEC_CUDA(cudaMalloc(&b->p, std::max<size_t>(bytes, 256)));
  b->n = std::max<size_t>(bytes, 256);
  return TEC_OK;
}

struct HostWorkspace {
  std::mutex mu;
  cudaStream_t stream = nullptr;
  cudaStream_t h2d = nullptr, d2h = nullptr;  // copy streams of the pipelined host path
  std::vector<cudaEvent_t> ev;                 // [2 * chunk]: inputs landed, outputs ready
  DevBuf x_src, w_src, x_pack, w_pack, y_nhwc, y_nchw, bias, res_src, res_pack,
      mul_src, mul_pack, err;
};

HostWorkspace& workspace(int dev) {
  static HostWorkspace ws[16];
  return ws[dev & 15];
}

}  // namespace

// ====================================================================
extern "C" {

int tec_api_version(void) { return TEC_SM100_API_VERSION; }

const char* tec_last_error(void) { return g_last_error.c_str(); }

int tec_device_sm_count(int device) { return sm_count(device); }

tec_status tec_conv_infer(const tec_conv_desc* d, int64_t out_shape[4]) {
  int64_t oh, ow;
  tec_status st = infer(d, &oh, &ow);
  if (st) return st;
  out_shape[0] = d->n;
  out_shape[1] = d->k;
  out_shape[2] = oh;
  out_shape[3] = ow;
  return TEC_OK;
}

tec_status tec_conv_layout_of(const tec_conv_desc* d, tec_conv_layout* out) {
  Plan pl{};
  tec_status st = make_plan(d, &pl);
  if (st) return st;
  out->oh = pl.oh;
  out->ow = pl.ow;
  out->cp = pl.cp;
  out->act_dtype = pl.act;
  out->acc_dtype = pl.acc;
  const int es = elem_bytes(pl.act);
  out->act_bytes = d->n * d->h * d->w * pl.cp * es;
  out->wt_bytes = d->depthwise ? d->c * d->r * d->s * es : d->k * d->r * d->s * pl.cp * es;
  if (pl.s2d) {
    out->act_bytes = d->n * pl.h2 * pl.w2 * pl.cp * es;
    out->wt_bytes = d->k * pl.r2 * pl.s2 * pl.cp * es;
  }
  if (pl.inter)  // [tap][3 planes][K][16]
    out->wt_bytes = d->k * (pl.s2d ? pl.r2 * pl.s2 : d->r * d->s) * 48 * es;
  out->out_elems = d->n * d->k * pl.oh * pl.ow;
  return TEC_OK;
}

tec_status tec_activation_pack(const tec_conv_desc* d, const void* x_nchw,
                               void* x_packed, void* stream) {
  Plan pl{};
  tec_status st = make_plan(d, &pl);
  if (st) return st;
  if (pl.s2d) {
    const int e = launch_pack_s2d(x_nchw, d->compute == TEC_COMPUTE_I8 ? kI8 : kF32, x_packed,
                                  d->n, d->c, d->h, d->w, d->pad_h, d->pad_w, pl.h2, pl.w2,
                                  pl.cp, pl.pack_mode, (cudaStream_t)stream);
    if (e) return cuda_fail(e, "pack_s2d");
    return TEC_OK;
  }
  if (pl.pack_mode < 0) {  // F32 exact path reads the NCHW tensor as is
    TEC_CUDA(cudaMemcpyAsync(x_packed, x_nchw, d->n * d->c * d->h * d->w * 4,
                             cudaMemcpyDeviceToDevice, (cudaStream_t)stream));
    return TEC_OK;
  }
  const int in_t = d->compute == TEC_COMPUTE_I8 ? kI8 : kF32;
  const int e = launch_pack_activation(x_nchw, in_t, x_packed, d->n, d->c, d->h * d->w,
                                       pl.cp, pl.pack_mode, (cudaStream_t)stream);
  if (e) return cuda_fail(e, "pack_activation");
  return TEC_OK;
}

tec_status tec_weight_pretransform(const tec_conv_desc* d, const void* w_oihw,
                                   void* w_packed, void* stream) {
  Plan pl{};
  tec_status st = make_plan(d, &pl);
  if (st) return st;
  if (pl.inter) {  // [tap][plane][K][16] (conv_f32tc.cu, interleaved planes)
    const int e = launch_pack_weights_split3i(w_oihw, w_packed, d->k, d->c, d->r, d->s, pl.r2,
                                              pl.s2, pl.s2d ? 1 : 0, (cudaStream_t)stream);
    if (e) return cuda_fail(e, "pack_weights_split3i");
    return TEC_OK;
  }
  if (pl.s2d) {
    const int e = launch_pack_weights_s2d(w_oihw, d->compute == TEC_COMPUTE_I8 ? kI8 : kF32,
                                          w_packed, d->k, d->c, d->r, d->s, pl.r2, pl.s2, pl.cp,
                                          pl.pack_mode, (cudaStream_t)stream);
    if (e) return cuda_fail(e, "pack_weights_s2d");
    return TEC_OK;
  }
  if (pl.pack_mode < 0) {  // OIHW == [oc][(ic, rh, rw)]: the reduce order
    TEC_CUDA(cudaMemcpyAsync(w_packed, w_oihw, d->k * d->c * d->r * d->s * 4,
                             cudaMemcpyDeviceToDevice, (cudaStream_t)stream));
    return TEC_OK;
  }
  const int in_t = d->compute == TEC_COMPUTE_I8 ? kI8 : kF32;
  const int e = launch_pack_weights(w_oihw, in_t, w_packed, d->k, d->c, d->r, d->s,
                                    pl.cp, d->depthwise, pl.pack_mode, (cudaStream_t)stream);
  if (e) return cuda_fail(e, "pack_weights");
  return TEC_OK;
}

tec_status tec_weight_pretransform_bn(const tec_conv_desc* d, const void* w_oihw,
                                      const float* scale, void* w_packed, void* stream) {
  if (!d || !w_oihw || !scale || !w_packed) return fail(TEC_E_INTERNAL, "null argument");
  if (d->compute == TEC_COMPUTE_I8)
    return fail(TEC_E_LOWERING, "batch-norm folding applies to float weights");
  Plan pl{};
  tec_status st = make_plan(d, &pl);
  if (st) return st;
  const int64_t rows = d->k;
  const int64_t per_row = (d->depthwise ? 1 : d->c) * d->r * d->s;
  cudaStream_t s = (cudaStream_t)stream;
  // parameter binding time, not the execution path: a stream-ordered
  // temporary for the folded OIHW weights
  void* tmp = nullptr;
  TEC_CUDA(cudaMallocAsync(&tmp, rows * per_row * sizeof(float), s));
  int dev = 0;
  cudaGetDevice(&dev);
  const int e = launch_scale_rows(static_cast<const float*>(w_oihw), scale,
                                  static_cast<float*>(tmp), rows * per_row, per_row,
                                  sm_count(dev), s);
  if (e) {
    cudaFreeAsync(tmp, s);
    return cuda_fail(e, "bn weight fold");
  }
  st = tec_weight_pretransform(d, tmp, w_packed, stream);
  cudaFreeAsync(tmp, s);
  return st;
}

tec_status tec_activation_pack_nhwc(const tec_conv_desc* d, const void* x_nhwc_f32,
                                    void* x_packed, void* stream) {
  Plan pl{};
  tec_status st = make_plan(d, &pl);
  if (st) return st;
  if (d->compute != TEC_COMPUTE_F32TC || d->depthwise || pl.s2d)
    return fail(TEC_E_LOWERING, "NHWC packing is the f32tc dense-conv input (no space-to-depth)");
  const int e = launch_split3_nhwc(static_cast<const float*>(x_nhwc_f32), x_packed,
                                   d->n * d->h * d->w, d->c, pl.cp, pl.inter ? 16 : pl.cpp,
                                   (cudaStream_t)stream);
  if (e) return cuda_fail(e, "split3_nhwc");
  return TEC_OK;
}

tec_status tec_nchw_to_nhwc(const void* src, int32_t src_dtype, void* dst,
                            int32_t dst_dtype, int64_t n, int64_t c, int64_t h,
                            int64_t w, void* stream) {
  int mode;
  if (dst_dtype == TEC_DT_BF16) mode = 0;
  else if (dst_dtype == TEC_DT_F32) mode = 3;
  else if (dst_dtype == TEC_DT_I32) mode = 4;
  else if (dst_dtype == TEC_DT_I8) mode = 2;
  else return fail(TEC_E_LOWERING, "unsupported nhwc dtype");
  const int in_t = src_dtype == TEC_DT_I32 ? kI32 : src_dtype == TEC_DT_I8 ? kI8 : kF32;
  const int e = launch_pack_activation(src, in_t, dst, n, c, h * w, c, mode,
                                       (cudaStream_t)stream);
  if (e) return cuda_fail(e, "nchw_to_nhwc");
  return TEC_OK;
}

tec_status tec_output_unpack(const void* y_nhwc, int32_t y_dtype, void* y_nchw,
                             int32_t dst_dtype, int64_t n, int64_t c, int64_t h,
                             int64_t w, void* stream) {
  const int e = launch_unpack_output(y_nhwc, y_dtype, y_nchw, dst_dtype, n, c, h * w,
                                     (cudaStream_t)stream);
  if (e) return cuda_fail(e, "output_unpack");
  return TEC_OK;
}

tec_status tec_conv2d_fused(const tec_conv_desc* d, const tec_epilogue* epi,
                            const tec_knobs* knobs, const void* x_packed,
                            const void* w_packed, void* y, int32_t out_dtype,
                            int32_t* err_flag, void* stream) {
  if (d && d->depthwise)
    return tec_depthwise_fused(d, epi, knobs, x_packed, w_packed, y, out_dtype,
                               err_flag, stream);
  Plan pl{};
  tec_status st = make_plan(d, &pl);
  if (st) return st;
  EpilogueParams ep;
  st = build_epilogue(epi, pl.kind == MmaKind::kI8, &ep);
  if (st) return st;
  if (pl.kind == MmaKind::kI8 && (st = check_int8_epilogue(ep, d, out_dtype, knobs))) return st;
  if (!x_packed || !w_packed || !y) return fail(TEC_E_INTERNAL, "null buffer");
  if (d->compute == TEC_COMPUTE_F32) {
    if (out_dtype != TEC_DT_F32) return fail(TEC_E_LOWERING, "f32 path produces f32");
    ConvGemmParams p{};
    p.n = (int32_t)d->n; p.h = (int32_t)d->h; p.w = (int32_t)d->w; p.cp = (int32_t)d->c;
    p.oh = (int32_t)pl.oh; p.ow = (int32_t)pl.ow; p.oc = (int32_t)d->k;
    p.r = (int32_t)d->r; p.s = (int32_t)d->s;
    p.sh = (int32_t)d->stride_h; p.sw = (int32_t)d->stride_w;
    p.ph = (int32_t)d->pad_h; p.pw = (int32_t)d->pad_w;
    p.m = (int32_t)pl.m;
    p.out_type = kF32;
    p.y = y;
    p.err = err_flag;
    p.epi = ep;
    if (plan_only(TEC_KERNEL_F32_EXACT, 64, 64, 0, 0, 0, 0, 0, 1, 1)) return TEC_OK;
    const int e = launch_conv_f32_exact(static_cast<const float*>(x_packed),
                                        static_cast<const float*>(w_packed), p,
                                        (cudaStream_t)stream);
    if (e) return cuda_fail(e, "conv_f32_exact launch");
    return TEC_OK;
  }
  const bool f32tc = d->compute == TEC_COMPUTE_F32TC;
  if (pl.s2d) {
    // The folded stem: a stride-1, unpadded (r2 x s2) conv over the
    // space-to-depth input; same output grid (checked in make_plan).
    tec_conv_desc d2 = *d;
    d2.c = pl.cpp; d2.h = pl.h2; d2.w = pl.w2; d2.r = pl.r2; d2.s = pl.s2;
    d2.stride_h = d2.stride_w = 1;
    d2.pad_h = d2.pad_w = 0;
    Plan pl2 = pl;
    pl2.s2d = false;
    if (f32tc)
      return run_conv_f32tc(&d2, pl2, ep, knobs, x_packed, w_packed, y, out_dtype,
                            (cudaStream_t)stream);
    return run_conv(&d2, pl2, ep, knobs, x_packed, w_packed, y, out_dtype, err_flag,
                    (cudaStream_t)stream);
  }
  if (f32tc)
    return run_conv_f32tc(d, pl, ep, knobs, x_packed, w_packed, y, out_dtype,
                          (cudaStream_t)stream);
  return run_conv(d, pl, ep, knobs, x_packed, w_packed, y, out_dtype, err_flag,
                  (cudaStream_t)stream);
}

tec_status tec_conv2d_fused_ws(const tec_conv_desc* d, const tec_epilogue* epi,
                               const tec_knobs* knobs, const void* x_packed,
                               const void* w_packed, void* y, int32_t out_dtype,
                               int32_t* err_flag, void* ws, size_t ws_bytes, void* stream) {
  g_ws = ws;
  g_ws_bytes = ws ? ws_bytes : 0;
  const tec_status st = tec_conv2d_fused(d, epi, knobs, x_packed, w_packed, y, out_dtype,
                                         err_flag, stream);
  g_ws = nullptr;
  g_ws_bytes = 0;
  return st;
}

tec_status tec_workspace_bytes(const tec_conv_desc* d, const tec_epilogue* epi,
                               const tec_knobs* knobs, size_t* bytes) {
  if (!bytes) return fail(TEC_E_INTERNAL, "null output");
  tec_kernel_plan kp;
  const tec_status st = tec_conv_plan(d, epi, knobs, &kp);
  if (st) return st;
  *bytes = (size_t)kp.workspace_bytes;
  return TEC_OK;
}

tec_status tec_depthwise_fused(const tec_conv_desc* d, const tec_epilogue* epi,
                               const tec_knobs* knobs, const void* x_packed,
                               const void* w_packed, void* y, int32_t out_dtype,
                               int32_t* err_flag, void* stream) {
  Plan pl{};
  tec_status st = make_plan(d, &pl);
  if (st) return st;
  if (!d->depthwise) return fail(TEC_E_LOWERING, "not a depthwise descriptor");
  EpilogueParams ep;
  st = build_epilogue(epi, d->compute == TEC_COMPUTE_I8, &ep);
  if (st) return st;
  if (epi_requant(ep) || ep.res_i8)
    return fail(TEC_E_LOWERING, "depthwise: no requantize / i8-residual epilogue");
  DepthwiseParams p{};
  p.n = (int32_t)d->n; p.h = (int32_t)d->h; p.w = (int32_t)d->w; p.c = (int32_t)d->c;
  p.oh = (int32_t)pl.oh; p.ow = (int32_t)pl.ow;
  p.r = (int32_t)d->r; p.s = (int32_t)d->s;
  p.sh = (int32_t)d->stride_h; p.sw = (int32_t)d->stride_w;
  p.ph = (int32_t)d->pad_h; p.pw = (int32_t)d->pad_w;
  p.in_type = pl.act == TEC_DT_BF16 ? kBF16 : pl.act == TEC_DT_I8 ? kI8 : kF32;
  p.out_type = out_dtype == TEC_DT_BF16 ? kBF16 : out_dtype == TEC_DT_I32 ? kI32 : kF32;
  p.x = x_packed;
  p.wt = w_packed;
  p.y = y;
  p.err = err_flag;
  p.epi = ep;
  // knob unroll: 0 auto (TMA-tiled kernel when it applies), 8 TMA-tiled,
  // 2/4 column-streaming kernel with that many outputs per thread, 1 generic.
  const int tw = knobs && knobs->unroll ? (int)knobs->unroll : 0;
  if (tw == 0 || tw == 8) {
    const int prog = epi && fast_program(ep) ? (ep.n_ops == 0 ? 0 : ep.n_ops == 1 ? 1 : 2) : -1;
    DwTmaShape t{};
    if (prog >= 0 && (p.in_type == kBF16 || p.in_type == kF32) && dw_tma_plan(p, &t)) {
      const DriverFns& fns = driver_fns();
      const int es = p.in_type == kBF16 ? 2 : 4;
      CUtensorMap tm{};
      cuuint64_t dims[4] = {(cuuint64_t)d->c, (cuuint64_t)d->w, (cuuint64_t)d->h, (cuuint64_t)d->n};
      cuuint64_t strides[3] = {(cuuint64_t)(d->c * es), (cuuint64_t)(d->c * es * d->w),
                               (cuuint64_t)(d->c * es * d->w * d->h)};
      cuuint32_t box[4] = {(cuuint32_t)t.cb, (cuuint32_t)t.cols_in, (cuuint32_t)t.rows_in,
                           (cuuint32_t)t.ni};
      cuuint32_t estr[4] = {1, 1, 1, 1};
      CUresult r = fns.ok ? fns.tiled(&tm, es == 2 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16
                                                   : CU_TENSOR_MAP_DATA_TYPE_FLOAT32,
                                      4, const_cast<void*>(x_packed), dims, strides, box, estr,
                                      CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                      CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                                      CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE)
                          : CUDA_ERROR_NOT_INITIALIZED;
      if (r == CUDA_SUCCESS) {
        int dev = 0;
        cudaGetDevice(&dev);
        if (plan_only(TEC_KERNEL_DW_TMA, t.cb, t.th, 2, 0, 2 * t.buf_bytes + 128, 0, 0, 1, 1))
          return TEC_OK;
        const int e = launch_dw_tma(p, tm, t, prog, sm_count(dev), (cudaStream_t)stream);
        if (e == 0) return TEC_OK;
        if (e != -1) return cuda_fail(e, "depthwise (TMA) launch");
      }
    }
    if (tw == 8) return fail(TEC_E_LOWERING, "TMA depthwise kernel does not apply to this layer");
  }
  if (plan_only(TEC_KERNEL_DW_DIRECT, 0, tw == 0 ? 4 : tw, 0, 0, 0, 0, 0, 1, 1)) return TEC_OK;
  const int e = launch_depthwise(p, tw == 0 ? 4 : tw, (cudaStream_t)stream);
  if (e == -1)
    return fail(TEC_E_LOWERING, "depthwise: unsupported dtype pair or C not a multiple of the vector width");
  if (e) return cuda_fail(e, "depthwise launch");
  return TEC_OK;
}

// ------------------------------------------------------------ pooling
namespace {
int32_t elem_type_of(int32_t dt) {
  return dt == TEC_DT_BF16 ? kBF16 : dt == TEC_DT_I8 ? kI8 : dt == TEC_DT_I32 ? kI32 : kF32;
}
tec_status pool_check(const tec_pool_desc* d, bool window) {
  if (!d) return fail(TEC_E_INTERNAL, "null descriptor");
  if (d->n <= 0 || d->c <= 0 || d->h <= 0 || d->w <= 0)
    return fail(TEC_E_SHAPE_MISMATCH, "pool: non-positive input shape");
  if (window) {
    if (d->r <= 0 || d->s <= 0 || d->stride_h <= 0 || d->stride_w <= 0 || d->pad_h < 0 ||
        d->pad_w < 0)
      return fail(TEC_E_SHAPE_MISMATCH, "max_pool2d: bad window/stride/padding");
    if (d->h + 2 * d->pad_h < d->r || d->w + 2 * d->pad_w < d->s)
      return fail(TEC_E_SHAPE_MISMATCH, "max_pool2d: window larger than padded input");
    if (d->pad_h >= d->r || d->pad_w >= d->s)
      return fail(TEC_E_SHAPE_MISMATCH, "max_pool2d: padding must be smaller than the window");
  }
  if (d->n * d->c * d->h * d->w > (int64_t)1 << 40)
    return fail(TEC_E_SHAPE_MISMATCH, "pool: tensor too large");
  return TEC_OK;
}
}  // namespace

tec_status tec_conv_plan(const tec_conv_desc* d, const tec_epilogue* epi,
                         const tec_knobs* knobs, tec_kernel_plan* out) {
  if (!out) return fail(TEC_E_INTERNAL, "null plan");
  *out = tec_kernel_plan{};
  cudaFree(nullptr);  // tensor-map encoding needs a current context
  tec_conv_layout lay;
  tec_status st = tec_conv_layout_of(d, &lay);
  if (st) return st;
  // Operand pointers only feed tensor-map encodes here (nothing launches):
  // any aligned address works.
  static char dummy[256] __attribute__((aligned(256)));
  tec_epilogue e{};
  if (epi) {
    e = *epi;
    if (e.bias) e.bias = dummy;
    if (e.residual) e.residual = dummy;
    if (e.mul_operand) e.mul_operand = dummy;
  }
  const bool rq = epi && epi->n_ops > 0 && epi->ops[epi->n_ops - 1] == TEC_EPI_REQUANTIZE;
  const int32_t out_t = d->compute == TEC_COMPUTE_I8 ? (rq ? TEC_DT_I8 : TEC_DT_I32)
                        : d->compute == TEC_COMPUTE_BF16 ? TEC_DT_BF16 : TEC_DT_F32;
  g_plan = out;
  st = tec_conv2d_fused(d, epi ? &e : nullptr, knobs, dummy, dummy, dummy, out_t, nullptr, nullptr);
  g_plan = nullptr;
  return st;
}

tec_status tec_pool_infer(const tec_pool_desc* d, int64_t out_shape[4]) {
  tec_status st = pool_check(d, true);
  if (st) return st;
  out_shape[0] = d->n;
  out_shape[1] = d->c;
  out_shape[2] = (d->h + 2 * d->pad_h - d->r) / d->stride_h + 1;
  out_shape[3] = (d->w + 2 * d->pad_w - d->s) / d->stride_w + 1;
  return TEC_OK;
}

tec_status tec_max_pool2d(const tec_pool_desc* d, const void* x, void* y, void* stream) {
  int64_t os[4];
  tec_status st = tec_pool_infer(d, os);
  if (st) return st;
  if (d->dtype != d->out_dtype) return fail(TEC_E_LOWERING, "max_pool2d keeps the dtype");
  if (!x || !y) return fail(TEC_E_INTERNAL, "null buffer");
  PoolParams p{};
  p.n = (int32_t)d->n; p.h = (int32_t)d->h; p.w = (int32_t)d->w; p.c = (int32_t)d->c;
  p.oh = (int32_t)os[2]; p.ow = (int32_t)os[3];
  p.r = (int32_t)d->r; p.s = (int32_t)d->s;
  p.sh = (int32_t)d->stride_h; p.sw = (int32_t)d->stride_w;
  p.ph = (int32_t)d->pad_h; p.pw = (int32_t)d->pad_w;
  p.type = p.out_type = elem_type_of(d->dtype);
  p.x = x; p.y = y;
  // bf16 3x3 windows: TMA-tiled kernel (NaN out-of-bounds fill, skipped by
  // the max), the depthwise tile planner sizes the halo tiles.
  if (p.type == kBF16 && p.r == 3 && p.s == 3 && p.sh == p.sw && (p.sw == 1 || p.sw == 2) &&
      p.pw <= 1 && p.ph <= 1) {
    DepthwiseParams q{};
    q.n = p.n; q.h = p.h; q.w = p.w; q.c = p.c; q.oh = p.oh; q.ow = p.ow;
    q.r = 3; q.s = 3; q.sh = p.sh; q.sw = p.sw; q.ph = p.ph; q.pw = p.pw;
    q.in_type = q.out_type = kBF16;
    q.x = x; q.y = y;
    DwTmaShape t{};
    const DriverFns& fns = driver_fns();
    if (fns.ok && dw_tma_plan(q, &t)) {
      CUtensorMap tm{};
      cuuint64_t dims[4] = {(cuuint64_t)d->c, (cuuint64_t)d->w, (cuuint64_t)d->h, (cuuint64_t)d->n};
      cuuint64_t strides[3] = {(cuuint64_t)(d->c * 2), (cuuint64_t)(d->c * 2 * d->w),
                               (cuuint64_t)(d->c * 2 * d->w * d->h)};
      cuuint32_t box[4] = {(cuuint32_t)t.cb, (cuuint32_t)t.cols_in, (cuuint32_t)t.rows_in,
                           (cuuint32_t)t.ni};
      cuuint32_t estr[4] = {1, 1, 1, 1};
      CUresult r = fns.tiled(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(x), dims,
                             strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                             CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                             CU_TENSOR_MAP_FLOAT_OOB_FILL_NAN_REQUEST_ZERO_FMA);
      if (r == CUDA_SUCCESS) {
        int dev = 0;
        cudaGetDevice(&dev);
        const int e = launch_pool_tma(q, tm, t, sm_count(dev), (cudaStream_t)stream);
        if (e == 0) return TEC_OK;
        if (e != -1) return cuda_fail(e, "max_pool2d (TMA) launch");
      }
    }
  }
  const int e = launch_max_pool(p, (cudaStream_t)stream);
  if (e == -1) return fail(TEC_E_LOWERING, "max_pool2d: channels x element size must be a multiple of 16 B");
  if (e) return cuda_fail(e, "max_pool2d launch");
  return TEC_OK;
}

tec_status tec_global_avg_pool(const tec_pool_desc* d, const void* x, void* y, void* stream) {
  tec_status st = pool_check(d, false);
  if (st) return st;
  if (!x || !y) return fail(TEC_E_INTERNAL, "null buffer");
  PoolParams p{};
  p.n = (int32_t)d->n; p.h = (int32_t)d->h; p.w = (int32_t)d->w; p.c = (int32_t)d->c;
  p.oh = p.ow = 1;
  p.scale = (float)(1.0 / (double)(d->h * d->w));  // scale attr rounded to float (R/src/ops.cpp:260-281)
  p.type = elem_type_of(d->dtype);
  p.out_type = elem_type_of(d->out_dtype);
  p.x = x; p.y = y;
  const int e = launch_global_avg_pool(p, (cudaStream_t)stream);
  if (e == -1) return fail(TEC_E_LOWERING, "global_avg_pool: f32/bf16 only, channels x element size a multiple of 16 B");
  if (e) return cuda_fail(e, "global_avg_pool launch");
  return TEC_OK;
}

tec_status tec_elementwise(const tec_elem_prog* d, const void* x, void* y, int32_t* err_flag,
                           void* stream) {
  if (!d) return fail(TEC_E_INTERNAL, "null elementwise program");
  if (d->n_ops < 0 || d->n_ops > TEC_MAX_ELEM_OPS)
    return fail(TEC_E_LOWERING, "elementwise: 0.." + std::to_string(TEC_MAX_ELEM_OPS) + " members");
  if (d->count < 0) return fail(TEC_E_SHAPE_MISMATCH, "elementwise: negative count");
  const int32_t sd = d->src_dtype, dd = d->dst_dtype;
  auto known = [](int32_t t) { return t == TEC_DT_F32 || t == TEC_DT_I32 || t == TEC_DT_I8; };
  if (!known(sd) || !known(dd)) return fail(TEC_E_LOWERING, "elementwise: f32 / i32 / i8 data only");
  ElemProg p{};
  p.n_ops = d->n_ops;
  p.in_type = elem_type_of(sd);
  p.out_type = elem_type_of(dd);
  p.count = d->count;
  // walk the chain's value type (graph.py infer) so a bad program fails here
  int32_t t = sd;
  for (int k = 0; k < d->n_ops; ++k) {
    const int32_t kind = d->kind[k];
    p.kind[k] = kind;
    const std::string at = "elementwise member " + std::to_string(k) + ": ";
    if (kind == TEC_ELEM_CAST) {
      const int32_t to = d->cast_to[k];
      const bool ok = (t == TEC_DT_I8 && (to == TEC_DT_I32 || to == TEC_DT_F32 || to == TEC_DT_I8)) ||
                      (t == TEC_DT_I32 && (to == TEC_DT_F32 || to == TEC_DT_I32)) ||
                      (t == TEC_DT_F32 && to == TEC_DT_F32);
      if (!ok) return fail(TEC_E_LOWERING, at + "unsupported cast");
      p.cast_to_f[k] = to == TEC_DT_F32 && t != TEC_DT_F32;
      t = to;
    } else if (kind == TEC_ELEM_SCALE) {
      const double c = d->scale[k];
      if (t == TEC_DT_F32) {
        p.fscale[k] = (float)c;  // the factor rounded to float (R/src/ops.cpp:260-281)
      } else {
        if (c != std::floor(c)) return fail(TEC_E_SHAPE_MISMATCH, at + "integer scale requires an integral factor");
        if (std::fabs(c) >= 4294967296.0) return fail(TEC_E_LOWERING, at + "|integral scale| >= 2^32");
        if (t == TEC_DT_I8) return fail(TEC_E_LOWERING, at + "scale of i8 data (cast to i32 first)");
        p.mult[k] = (int64_t)c;
      }
    } else if (kind == TEC_ELEM_RELU) {
    } else if (kind == TEC_ELEM_REQUANTIZE) {
      if (t != TEC_DT_I32) return fail(TEC_E_SHAPE_MISMATCH, at + "requantize wants i32 data");
      if (d->mult[k] < 1 || d->mult[k] >= (int64_t(1) << 31) || d->shift[k] < 0 || d->shift[k] > 62)
        return fail(TEC_E_SHAPE_MISMATCH, at + "requantize needs 1 <= multiplier < 2^31, 0 <= shift <= 62");
      p.mult[k] = d->mult[k];
      p.shift[k] = d->shift[k];
      t = TEC_DT_I8;
    } else {
      return fail(TEC_E_LOWERING, at + "unknown kind " + std::to_string(kind));
    }
  }
  if (t != dd) return fail(TEC_E_SHAPE_MISMATCH, "elementwise: the chain ends in dtype " +
                                                     std::to_string(t) + ", y is " + std::to_string(dd));
  p.out_f = dd == TEC_DT_F32;
  if (d->count == 0) return TEC_OK;
  if (!x || !y) return fail(TEC_E_INTERNAL, "null buffer");
  if ((reinterpret_cast<uintptr_t>(x) | reinterpret_cast<uintptr_t>(y)) & 15)
    return fail(TEC_E_LOWERING, "elementwise: x / y must be 16-byte aligned");
  int dev = 0;
  cudaGetDevice(&dev);
  const int e = launch_elementwise(p, x, y, err_flag, sm_count(dev), (cudaStream_t)stream);
  if (e) return cuda_fail(e, "elementwise launch");
  return TEC_OK;
}

tec_status tec_eval_fused_conv(const tec_conv_desc* d, const tec_epilogue* epi,
                               const tec_knobs* knobs, const void* x,
                               const void* w, void* y, int device) {
  Plan pl{};
  tec_status st = make_plan(d, &pl);
  if (st) return st;
  const bool integer = d->compute == TEC_COMPUTE_I8;
  EpilogueParams probe;
  st = build_epilogue(epi, integer, &probe);
  if (st) return st;
  TEC_CUDA(cudaSetDevice(device));
  HostWorkspace& ws = workspace(device);
  std::lock_guard<std::mutex> lock(ws.mu);
  // Every exit -- errors included -- waits for the call's copy and compute
  // streams, so no DMA into the caller's host buffers outlives the call.
  struct Drain {
    HostWorkspace& w;
    ~Drain() {
      for (cudaStream_t t : {w.stream, w.h2d, w.d2h})
        if (t) cudaStreamSynchronize(t);
    }
  } drain{ws};
  if (!ws.stream) TEC_CUDA(cudaStreamCreateWithFlags(&ws.stream, cudaStreamNonBlocking));
  cudaStream_t s = ws.stream;

  const int in_es = integer ? 1 : 4;
  const int acc_t = integer ? TEC_DT_I32 : TEC_DT_F32;
  const int64_t x_elems = d->n * d->c * d->h * d->w;
  const int64_t w_elems = d->depthwise ? d->c * d->r * d->s : d->k * d->c * d->r * d->s;
  const int64_t y_elems = d->n * d->k * pl.oh * pl.ow;
  tec_conv_layout lay;
  st = tec_conv_layout_of(d, &lay);
  if (st) return st;

  if ((st = ensure(&ws.x_src, x_elems * in_es))) return st;
  if ((st = ensure(&ws.w_src, w_elems * in_es))) return st;
  if ((st = ensure(&ws.x_pack, lay.act_bytes))) return st;
  if ((st = ensure(&ws.w_pack, lay.wt_bytes))) return st;
  if ((st = ensure(&ws.y_nhwc, y_elems * 4))) return st;
  if ((st = ensure(&ws.y_nchw, y_elems * 4))) return st;
  if ((st = ensure(&ws.err, 4))) return st;
  TEC_CUDA(cudaMemcpyAsync(ws.w_src.p, w, w_elems * in_es, cudaMemcpyHostToDevice, s));
  TEC_CUDA(cudaMemsetAsync(ws.err.p, 0, 4, s));

  tec_epilogue dev_epi;
  std::memset(&dev_epi, 0, sizeof(dev_epi));
  if (epi) {
    dev_epi = *epi;
    if (epi->bias) {
      if ((st = ensure(&ws.bias, d->k * 4))) return st;
      TEC_CUDA(cudaMemcpyAsync(ws.bias.p, epi->bias, d->k * 4, cudaMemcpyHostToDevice, s));
      dev_epi.bias = ws.bias.p;
    }
    // Same-shape operands arrive NCHW; the kernels read them NHWC.
    const void* srcs[2] = {epi->residual, epi->mul_operand};
    DevBuf* raw[2] = {&ws.res_src, &ws.mul_src};
    DevBuf* pk[2] = {&ws.res_pack, &ws.mul_pack};
    const void** dst[2] = {&dev_epi.residual, &dev_epi.mul_operand};
    for (int i = 0; i < 2; ++i) {
      if (!srcs[i]) continue;
      if ((st = ensure(raw[i], y_elems * 4))) return st;
      if ((st = ensure(pk[i], y_elems * 4))) return st;
      TEC_CUDA(cudaMemcpyAsync(raw[i]->p, srcs[i], y_elems * 4, cudaMemcpyHostToDevice, s));
      st = tec_nchw_to_nhwc(raw[i]->p, acc_t, pk[i]->p, acc_t, d->n, d->k, pl.oh, pl.ow, s);
      if (st) return st;
      *dst[i] = pk[i]->p;
    }
  }
  // Pipelined host path: without same-shape operands the batch is cut into
  // chunks of whole images and H2D of chunk i+1, pack/conv/unpack of chunk i
  // and D2H of chunk i-1 overlap on three streams (PCIe is full duplex). Each
  // image's result is independent of the chunking (every output sums its K
  // in the same order; tests check batch linearity bit for bit).
  const bool same_shape_ops = epi && (epi->residual || epi->mul_operand);
  const int64_t x_img = x_elems / d->n * in_es;
  static const int64_t chunk_bytes = [] {
    const char* e = std::getenv("TEC_SM100_CHUNK_KB");  // tuning override
    return e ? std::max<int64_t>(64, std::atoll(e)) << 10 : int64_t(6) << 20;
  }();
  // sized by the larger direction (the stem's output is 5x its input): the
  // first chunk's upload and the last chunk's download are the exposed ends
  const int64_t io_bytes = std::max<int64_t>(x_elems * in_es, y_elems * 4);
  int64_t chunks = std::min<int64_t>(d->n, std::max<int64_t>(1, io_bytes / chunk_bytes));
  chunks = std::min<int64_t>(chunks, 64);
  if (!same_shape_ops && chunks > 1 && lay.act_bytes % d->n == 0) {
    if (!ws.h2d) TEC_CUDA(cudaStreamCreateWithFlags(&ws.h2d, cudaStreamNonBlocking));
    if (!ws.d2h) TEC_CUDA(cudaStreamCreateWithFlags(&ws.d2h, cudaStreamNonBlocking));
    while ((int64_t)ws.ev.size() < 2 * chunks) {
      cudaEvent_t e;
      TEC_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
      ws.ev.push_back(e);
    }
    if ((st = tec_weight_pretransform(d, ws.w_src.p, ws.w_pack.p, s))) return st;
    const int64_t per = (d->n + chunks - 1) / chunks;
    const int64_t a_img = lay.act_bytes / d->n, y_img = y_elems / d->n * 4;
    // the raw x copy above is replaced by per-chunk copies on the H2D stream
    for (int64_t c = 0, n0 = 0; n0 < d->n; ++c, n0 += per) {
      const int64_t nb = std::min<int64_t>(per, d->n - n0);
      tec_conv_desc dc = *d;
      dc.n = nb;
      uint8_t* xs = static_cast<uint8_t*>(ws.x_src.p) + n0 * x_img;
      TEC_CUDA(cudaMemcpyAsync(xs, static_cast<const uint8_t*>(x) + n0 * x_img, nb * x_img,
                               cudaMemcpyHostToDevice, ws.h2d));
      TEC_CUDA(cudaEventRecord(ws.ev[2 * c], ws.h2d));
      TEC_CUDA(cudaStreamWaitEvent(s, ws.ev[2 * c], 0));
      uint8_t* xp = static_cast<uint8_t*>(ws.x_pack.p) + n0 * a_img;
      uint8_t* yn = static_cast<uint8_t*>(ws.y_nhwc.p) + n0 * y_img;
      uint8_t* yc = static_cast<uint8_t*>(ws.y_nchw.p) + n0 * y_img;
      if ((st = tec_activation_pack(&dc, xs, xp, s))) return st;
      st = tec_conv2d_fused(&dc, epi ? &dev_epi : nullptr, knobs, xp, ws.w_pack.p, yn, acc_t,
                            static_cast<int32_t*>(ws.err.p), s);
      if (st) return st;
      if ((st = tec_output_unpack(yn, acc_t, yc, acc_t, nb, d->k, pl.oh, pl.ow, s))) return st;
      TEC_CUDA(cudaEventRecord(ws.ev[2 * c + 1], s));
      TEC_CUDA(cudaStreamWaitEvent(ws.d2h, ws.ev[2 * c + 1], 0));
      TEC_CUDA(cudaMemcpyAsync(static_cast<uint8_t*>(y) + n0 * y_img, yc, nb * y_img,
                               cudaMemcpyDeviceToHost, ws.d2h));
    }
    int32_t err_host = 0;
    TEC_CUDA(cudaMemcpyAsync(&err_host, ws.err.p, 4, cudaMemcpyDeviceToHost, s));
    TEC_CUDA(cudaStreamSynchronize(s));
    TEC_CUDA(cudaStreamSynchronize(ws.d2h));
    if (err_host)
      return fail(TEC_E_FOLD_OVERFLOW, "value out of range for i32 in the fused epilogue");
    return TEC_OK;
  }
  // Weights first: the conv kernel reads them BEFORE griddepcontrol.wait
  // (they are parameters), so the kernel right before it must not be the
  // one producing them -- the activation pack sits in between.
  if ((st = tec_weight_pretransform(d, ws.w_src.p, ws.w_pack.p, s))) return st;
  TEC_CUDA(cudaMemcpyAsync(ws.x_src.p, x, x_elems * in_es, cudaMemcpyHostToDevice, s));
  if ((st = tec_activation_pack(d, ws.x_src.p, ws.x_pack.p, s))) return st;
  st = tec_conv2d_fused(d, epi ? &dev_epi : nullptr, knobs, ws.x_pack.p, ws.w_pack.p,
                        ws.y_nhwc.p, acc_t, static_cast<int32_t*>(ws.err.p), s);
  if (st) return st;
  if ((st = tec_output_unpack(ws.y_nhwc.p, acc_t, ws.y_nchw.p, acc_t, d->n, d->k, pl.oh,
                              pl.ow, s)))
    return st;
  int32_t err_host = 0;
  TEC_CUDA(cudaMemcpyAsync(y, ws.y_nchw.p, y_elems * 4, cudaMemcpyDeviceToHost, s));
  TEC_CUDA(cudaMemcpyAsync(&err_host, ws.err.p, 4, cudaMemcpyDeviceToHost, s));
  TEC_CUDA(cudaStreamSynchronize(s));
  if (err_host)
    return fail(TEC_E_FOLD_OVERFLOW, "value out of range for i32 in the fused epilogue");
  return TEC_OK;
}

tec_status tec_measure(const tec_conv_desc* d, const tec_epilogue* epi,
                       const tec_knobs* knobs, int device, int warmup, int reps,
                       int flush_l2, double* median_us) {
  Plan pl{};
  tec_status st = make_plan(d, &pl);
  if (st) return st;
  TEC_CUDA(cudaSetDevice(device));
  tec_conv_layout lay;
  if ((st = tec_conv_layout_of(d, &lay))) return st;
  const bool integer = d->compute == TEC_COMPUTE_I8;
  const bool rq = epi && epi->n_ops > 0 && epi->ops[epi->n_ops - 1] == TEC_EPI_REQUANTIZE;
  const int32_t out_t = integer ? (rq ? TEC_DT_I8 : TEC_DT_I32)
                        : d->compute == TEC_COMPUTE_F32 || d->compute == TEC_COMPUTE_F32TC
                            ? TEC_DT_F32 : TEC_DT_BF16;
  void *x = nullptr, *w = nullptr, *y = nullptr, *b = nullptr, *r = nullptr, *fl = nullptr;
  const size_t flush_bytes = 256ull << 20;
  cudaStream_t s;
  TEC_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  TEC_CUDA(cudaMalloc(&x, lay.act_bytes));
  TEC_CUDA(cudaMalloc(&w, lay.wt_bytes));
  TEC_CUDA(cudaMalloc(&y, lay.out_elems * 4));
  TEC_CUDA(cudaMalloc(&b, d->k * 4));
  TEC_CUDA(cudaMalloc(&r, lay.out_elems * 4));
  if (flush_l2) TEC_CUDA(cudaMalloc(&fl, flush_bytes));
  TEC_CUDA(cudaMemsetAsync(x, 1, lay.act_bytes, s));
  TEC_CUDA(cudaMemsetAsync(w, 1, lay.wt_bytes, s));
  TEC_CUDA(cudaMemsetAsync(b, 0, d->k * 4, s));
  TEC_CUDA(cudaMemsetAsync(r, 0, lay.out_elems * 4, s));
  tec_epilogue e{};
  if (epi) {
    e = *epi;
    if (e.bias) e.bias = b;
    if (e.residual) e.residual = r;
    if (e.mul_operand) e.mul_operand = r;
  }
  // Event timestamps here advance in ~2 us steps, too coarse for one launch
  // of a 10-30 us kernel: time `reps` back-to-back (flush, launch) pairs and
  // subtract the same number of flushes timed alone; three such batches,
  // median. The host enqueues each launch while the GPU runs the flush, so
  // host planning time stays outside the measurement.
  std::vector<float> times;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int i = 0; i < warmup && st == TEC_OK; ++i)
    st = tec_conv2d_fused(d, epi ? &e : nullptr, knobs, x, w, y, out_t, nullptr, s);
  if (st == TEC_OK && cudaStreamSynchronize(s) != cudaSuccess)
    st = fail(TEC_E_CUDA, "measure: kernel failed");
  const int n = std::max(1, reps);
  auto batch = [&](bool with_conv, float* us) -> tec_status {
    cudaEventRecord(e0, s);
    for (int i = 0; i < n; ++i) {
      if (flush_l2) cudaMemsetAsync(fl, i & 0xff, flush_bytes, s);
      if (with_conv) {
        tec_status t = tec_conv2d_fused(d, epi ? &e : nullptr, knobs, x, w, y, out_t, nullptr, s);
        if (t) return t;
      }
    }
    cudaEventRecord(e1, s);
    if (cudaEventSynchronize(e1) != cudaSuccess) return fail(TEC_E_CUDA, "measure: kernel failed");
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    *us = ms * 1000.f;
    return TEC_OK;
  };
  for (int trial = 0; trial < 3 && st == TEC_OK; ++trial) {
    float t_all = 0.f, t_flush = 0.f;
    st = batch(true, &t_all);
    if (st == TEC_OK && flush_l2) st = batch(false, &t_flush);
    if (st == TEC_OK) times.push_back(std::max(0.f, t_all - t_flush) / n);
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(x); cudaFree(w); cudaFree(y); cudaFree(b); cudaFree(r);
  if (fl) cudaFree(fl);
  cudaStreamDestroy(s);
  if (st) return st;
  if (times.empty()) return fail(TEC_E_INTERNAL, "no repetitions");
  std::sort(times.begin(), times.end());
  *median_us = times[times.size() / 2];
  return TEC_OK;
}

}  // extern "C"

// ------------------------------------------------------- native launch plans
struct tec_plan {
  std::vector<tec_step> steps;
  cudaGraph_t graph = nullptr;
  cudaGraphExec_t exec = nullptr;
  // the plan's own split-K scratch (steps run in order on one stream, so
  // they share it; zero-filled once, left zeroed by every launch)
  void* ws = nullptr;
  size_t ws_bytes = 0;
  int32_t* err = nullptr;  // integer range overflow flag shared by every step
};

namespace {
tec_status run_step(const tec_plan* p, const tec_step& s, void* stream) {
  switch (s.kind) {
    case TEC_STEP_CONV:
      return tec_conv2d_fused_ws(&s.conv, &s.epi, &s.knobs, s.src, s.w, s.dst, s.dst_dtype,
                                 p->err, p->ws, p->ws_bytes, stream);
    case TEC_STEP_DEPTHWISE:
      return tec_depthwise_fused(&s.conv, &s.epi, &s.knobs, s.src, s.w, s.dst, s.dst_dtype,
                                 p->err, stream);
    case TEC_STEP_ELEMWISE:
      return tec_elementwise(&s.elem, s.src, s.dst, p->err, stream);
    case TEC_STEP_MAX_POOL:
      return tec_max_pool2d(&s.pool, s.src, s.dst, stream);
    case TEC_STEP_AVG_POOL:
      return tec_global_avg_pool(&s.pool, s.src, s.dst, stream);
    case TEC_STEP_PACK:
      return tec_activation_pack(&s.conv, s.src, s.dst, stream);
    case TEC_STEP_UNPACK:
      return tec_output_unpack(s.src, s.src_dtype, s.dst, s.dst_dtype, s.n, s.c, s.h, s.w_, stream);
    case TEC_STEP_TO_NHWC:
      return tec_nchw_to_nhwc(s.src, s.src_dtype, s.dst, s.dst_dtype, s.n, s.c, s.h, s.w_, stream);
    case TEC_STEP_PACK_NHWC:
      return tec_activation_pack_nhwc(&s.conv, s.src, s.dst, stream);
    default:
      return fail(TEC_E_INTERNAL, "unknown plan step kind " + std::to_string(s.kind));
  }
}

tec_status run_steps(const tec_plan* p, void* stream) {
  for (size_t i = 0; i < p->steps.size(); ++i) {
    tec_status st = run_step(p, p->steps[i], stream);
    if (st) {
      g_last_error = "plan step " + std::to_string(i) + ": " + g_last_error;
      return st;
    }
  }
  return TEC_OK;
}
}  // namespace

extern "C" {
tec_status tec_plan_create(const tec_step* steps, int32_t n_steps, tec_plan** out) {
  if (!out || (n_steps > 0 && !steps) || n_steps < 0) return fail(TEC_E_INTERNAL, "bad plan arguments");
  auto* p = new tec_plan;
  p->steps.assign(steps, steps + n_steps);
  for (int32_t i = 0; i < n_steps; ++i) {
    if (steps[i].kind != TEC_STEP_CONV && steps[i].kind != TEC_STEP_DEPTHWISE) continue;
    tec_kernel_plan kp;
    tec_status st = tec_conv_plan(&steps[i].conv, &steps[i].epi, &steps[i].knobs, &kp);
    if (st) {
      delete p;
      g_last_error = "plan step " + std::to_string(i) + ": " + g_last_error;
      return st;
    }
    p->ws_bytes = std::max(p->ws_bytes, (size_t)kp.workspace_bytes);
  }
  if (cudaMalloc(reinterpret_cast<void**>(&p->err), sizeof(int32_t)) != cudaSuccess ||
      cudaMemset(p->err, 0, sizeof(int32_t)) != cudaSuccess) {
    if (p->err) cudaFree(p->err);
    delete p;
    return fail(TEC_E_CUDA, "plan error flag allocation failed");
  }
  if (p->ws_bytes) {
    if (cudaMalloc(&p->ws, p->ws_bytes) != cudaSuccess ||
        cudaMemset(p->ws, 0, p->ws_bytes) != cudaSuccess) {
      if (p->ws) cudaFree(p->ws);
      cudaFree(p->err);
      delete p;
      return fail(TEC_E_CUDA, "plan workspace allocation failed");
    }
  }
  *out = p;
  return TEC_OK;
}

tec_status tec_plan_run(tec_plan* p, void* stream) {
  if (!p) return fail(TEC_E_INTERNAL, "null plan");
  if (p->exec) {
    TEC_CUDA(cudaGraphLaunch(p->exec, (cudaStream_t)stream));
    return TEC_OK;
  }
  return run_steps(p, stream);
}

tec_status tec_plan_capture(tec_plan* p, void* stream) {
  if (!p) return fail(TEC_E_INTERNAL, "null plan");
  if (p->exec) {
    cudaGraphExecDestroy(p->exec);
    cudaGraphDestroy(p->graph);
    p->exec = nullptr;
    p->graph = nullptr;
  }
  cudaStream_t s = (cudaStream_t)stream;
  tec_status st = run_steps(p, stream);  // eager pass: attributes, split-K workspace
  if (st) return st;
  TEC_CUDA(cudaStreamSynchronize(s));
  TEC_CUDA(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
  st = run_steps(p, stream);
  cudaGraph_t g = nullptr;
  const cudaError_t ce = cudaStreamEndCapture(s, &g);
  if (st) {
    if (g) cudaGraphDestroy(g);
    return st;
  }
  if (ce != cudaSuccess) return cuda_fail(ce, "cudaStreamEndCapture");
  cudaGraphExec_t exec = nullptr;
  const cudaError_t ie = cudaGraphInstantiate(&exec, g, 0);
  if (ie != cudaSuccess) {
    cudaGraphDestroy(g);
    return cuda_fail(ie, "cudaGraphInstantiate");
  }
  p->graph = g;
  p->exec = exec;
  return TEC_OK;
}

tec_status tec_plan_run_steps(tec_plan* p, int32_t first, int32_t count, void* stream) {
  if (!p || first < 0 || count < 0 || (size_t)first + (size_t)count > p->steps.size())
    return fail(TEC_E_INTERNAL, "plan step range out of bounds");
  for (int32_t i = first; i < first + count; ++i) {
    tec_status st = run_step(p, p->steps[i], stream);
    if (st) {
      g_last_error = "plan step " + std::to_string(i) + ": " + g_last_error;
      return st;
    }
  }
  return TEC_OK;
}

int32_t tec_plan_size(const tec_plan* p) { return p ? (int32_t)p->steps.size() : 0; }

tec_status tec_plan_status(tec_plan* p, void* stream) {
  if (!p) return fail(TEC_E_INTERNAL, "null plan");
  cudaStream_t s = (cudaStream_t)stream;
  int32_t h = 0;
  TEC_CUDA(cudaMemcpyAsync(&h, p->err, sizeof(h), cudaMemcpyDeviceToHost, s));
  TEC_CUDA(cudaMemsetAsync(p->err, 0, sizeof(int32_t), s));
  TEC_CUDA(cudaStreamSynchronize(s));
  if (h) return fail(TEC_E_FOLD_OVERFLOW, "value out of range for i32 in a plan step");
  return TEC_OK;
}

void tec_plan_destroy(tec_plan* p) {
  if (!p) return;
  if (p->exec) cudaGraphExecDestroy(p->exec);
  if (p->graph) cudaGraphDestroy(p->graph);
  if (p->ws) cudaFree(p->ws);
  if (p->err) cudaFree(p->err);
  delete p;
}
}  // extern "C"
