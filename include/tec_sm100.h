/* tec_sm100.h -- C ABI of the B200 (sm_100a) backend for the fused
 * conv2d / depthwise_conv2d operator path of the reference "tec"
 * (/root/reference/proj, the arXiv 1802.04799 re-creation).
 *
 * Plain C: pointers, sizes, int/double scalars. No exceptions cross this
 * boundary; every call returns a tec_status and the message of the last
 * failure on the calling thread is available from tec_last_error().
 *
 * Which reference interface each entry point replaces (R = reference/proj):
 *
 *   tec_eval_fused_conv      eval_graph_node(fused [conv2d, scale?, bias_add?,
 *                            add?, mul?, relu?]) R/src/graph.cpp:209-225, and
 *                            eval_operator("conv2d"/"depthwise_conv2d")
 *                            R/src/ops.cpp:517-531 -- host DenseTensor-style
 *                            NCHW buffers in, NCHW out (the OperatorDef::
 *                            native_eval hook, R/include/tec/ops.hpp:63-65)
 *   tec_conv_infer           infer_conv R/src/ops.cpp:163-192 (same checks,
 *                            same ShapeMismatch code)
 *   tec_conv2d_fused /       the lowered + executed fused node for
 *   tec_depthwise_fused      target="sm100" (LowerOptions::target,
 *                            R/include/tec/lower.hpp:26-33): device buffers,
 *                            kernel-native layouts, caller's stream
 *   tec_weight_pretransform  the weight side of apply_layouts/fold_constants
 *                            (R/src/graph_passes.cpp:41-178): OIHW -> KRSC
 *   tec_activation_pack /    layout_transform (R/src/ops.cpp:419-489) at
 *   tec_output_unpack        graph boundaries: NCHW <-> packed NHWC
 *   tec_measure              measure_program / measure for target "sm100"
 *                            (R/src/tune.cpp:295-351): on-device timing
 *
 * Status codes: 0 = OK, otherwise 1 + (int)tec::ErrorCode
 * (R/include/tec/error.hpp:25-47, order is stable), plus TEC_E_CUDA for
 * device/runtime failures that have no reference counterpart.
 */
#ifndef TEC_SM100_H_
#define TEC_SM100_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TEC_SM100_API_VERSION 1

typedef int32_t tec_status;
enum {
  TEC_OK = 0,
  TEC_E_UNKNOWN_OPERATOR = 1,
  TEC_E_SHAPE_MISMATCH = 2,
  TEC_E_FOLD_OVERFLOW = 3,
  TEC_E_UNBOUND_AXIS = 4,
  TEC_E_DUPLICATE_INTRINSIC = 5,
  TEC_E_INVALID_FACTOR = 6,
  TEC_E_ILLEGAL_REORDER = 7,
  TEC_E_ILLEGAL_ANNOTATION = 8,
  TEC_E_ILLEGAL_BIND = 9,
  TEC_E_BIND_CONFLICT = 10,
  TEC_E_ILLEGAL_COMPUTE_AT = 11,
  TEC_E_SCOPE = 12,
  TEC_E_CAPACITY = 13,
  TEC_E_TENSORIZE_MISMATCH = 14,
  TEC_E_LOWERING = 15,
  TEC_E_BOUNDS = 16,
  TEC_E_DEADLOCK = 17,
  TEC_E_RACE = 18,
  TEC_E_NOT_ENOUGH_DATA = 19,
  TEC_E_IO = 20,
  TEC_E_INTERNAL = 21,
  TEC_E_CUDA = 64
};

/* Element types. The first three mirror tec::DType (R/include/tec/dtype.hpp:27). */
typedef enum {
  TEC_DT_F32 = 0,
  TEC_DT_I32 = 1,
  TEC_DT_I8 = 2,
  TEC_DT_BF16 = 3
} tec_dtype;

/* Arithmetic an operator runs with:
 *   BF16   : tcgen05 kind::f16 -- inputs rounded to bf16, exact products,
 *            f32 tensor-core accumulation (stated tolerance)
 *   F32TC  : f32 on tcgen05 kind::f16 -- every f32 operand split exactly into
 *            three bf16 planes (h + m + l), six products, the hh term folded
 *            into round-to-nearest f32 registers every 256 K elements: within
 *            the reference comparator's 1e-4 of evaluate_reference (dense
 *            conv; depthwise runs the exact F32 kernel)
 *   I8     : tcgen05 kind::i8 -- s8 x s8 -> s32 (bit-exact i8 path)
 *   F32    : f32 parity path -- SIMT, the reference's exact reduction
 *            order and rounding: bit-identical to evaluate_reference      */
typedef enum {
  TEC_COMPUTE_BF16 = 1,
  TEC_COMPUTE_F32TC = 2,
  TEC_COMPUTE_I8 = 3,
  TEC_COMPUTE_F32 = 4
} tec_compute;

/* Fused member ops, listed in member order (R/src/graph.cpp:209-222). */
typedef enum {
  TEC_EPI_SCALE = 1,  /* x * c            R/src/ops.cpp:260-281 */
  TEC_EPI_BIAS = 2,   /* x + b[oc]        R/src/ops.cpp:282-305 */
  TEC_EPI_ADD = 3,    /* x + r            R/src/ops.cpp:216-223 */
  TEC_EPI_MUL = 4,    /* x * r            R/src/ops.cpp:224-231 */
  TEC_EPI_RELU = 5,   /* max(x, 0)        R/src/ops.cpp:250-259 */
  /* int8 graphs (graph.py "requantize", not in the reference
   * registry): i32 -> i8 clamp((x * rq_mult + 2^(rq_shift-1)) >> rq_shift,
   * -128, 127). I8 compute only, the LAST member; y is then i8
   * (out_dtype TEC_DT_I8) and K a multiple of 16. */
  TEC_EPI_REQUANTIZE = 6
} tec_epi_op;

#define TEC_MAX_EPILOGUE 8

/* Logical operator shape: NCHW data, OIHW weights (R/src/ops.cpp:118-119),
 * symmetric padding (R/src/ops.cpp:125). Depthwise: k == c, weights [C,1,r,s]. */
typedef struct {
  int64_t n, c, h, w;
  int64_t k, r, s;
  int64_t stride_h, stride_w, pad_h, pad_w;
  int32_t depthwise;
  int32_t compute; /* tec_compute */
} tec_conv_desc;

typedef struct {
  int32_t n_ops;
  int32_t ops[TEC_MAX_EPILOGUE]; /* tec_epi_op, member order */
  double scale[TEC_MAX_EPILOGUE]; /* attr "scale" of each SCALE op */
  const void* bias;        /* BIAS operand: [K], f32 (i32 for I8)        */
  const void* residual;    /* ADD operand: output-shaped                  */
  const void* mul_operand; /* MUL operand: output-shaped                  */
  /* int8 graphs. Zero-initialised = unused. */
  int64_t rq_mult;         /* REQUANTIZE multiplier, 1 <= m < 2^31         */
  int32_t rq_shift;        /* REQUANTIZE shift, 0 <= s <= 62               */
  int32_t residual_i8;     /* 1: the ADD operand is an i8 tensor entering  */
  int64_t residual_scale;  /*    as scale(cast(r, i32), residual_scale)    */
                           /*    (|residual_scale| <= 2^24: no overflow)   */
} tec_epilogue;

/* Schedule knobs (Config = map<string,int64>, R/include/tec/autotune.hpp:43),
 * 0 = let the library choose. Mapping to the paper's primitives:
 *   tile_n   split/tile of the output-channel axis -> CTA tile N (64/128/256)
 *   tile_m   split/tile of the pixel axis -> CTA tile M (128)
 *   stages   cache_read(shared) depth -> smem ring stages
 *   acc_bufs virtual_thread -> TMEM accumulator buffers (2)
 *   grid     bind(blockIdx) extent -> persistent CTAs (<= #SMs)
 *   vec      vectorize width of the depthwise kernel (channels per thread)
 *   raster   reorder of the tile loop (0 = N fastest)
 *   tile_k   A-operand strategy: 1 im2col TMA, 2 shifted-window halo
 *   split_k  rfactor of the reduction over CTAs (-1: stream-K, f32tc)
 *   cluster_n 2 = two CTAs per cluster: the halo path multicasts weight
 *            tiles; the im2col path runs CTA pairs (tcgen05 cta_group::2,
 *            M = 256, each CTA loading half of the weight rows)
 *   cta_pair reserved (0)                                              */
typedef struct {
  int64_t tile_m, tile_n, tile_k, stages, cta_pair, cluster_m, cluster_n;
  int64_t raster, swizzle, split_k, vec, unroll, acc_bufs, grid;
} tec_knobs;

/* Kernel-native layouts chosen for a desc (sizes in bytes). */
typedef struct {
  int64_t oh, ow;          /* output spatial dims                          */
  int64_t cp;              /* stored channels of the packed activation     */
  int32_t act_dtype;       /* element type of packed activation/weights    */
  int32_t acc_dtype;       /* f32 or i32                                   */
  int64_t act_bytes;       /* packed NHWC activation                       */
  int64_t wt_bytes;        /* packed weights                               */
  int64_t out_elems;       /* n*k*oh*ow                                     */
} tec_conv_layout;

int tec_api_version(void);
const char* tec_last_error(void);
int tec_device_sm_count(int device);

/* infer_conv: output NCHW shape, or TEC_E_SHAPE_MISMATCH. */
tec_status tec_conv_infer(const tec_conv_desc* d, int64_t out_shape[4]);
tec_status tec_conv_layout_of(const tec_conv_desc* d, tec_conv_layout* out);

/* ---- device-level path (device pointers, caller's cudaStream_t) ---- */
/* NCHW f32 (or i8 for I8) -> packed NHWC activation. */
tec_status tec_activation_pack(const tec_conv_desc* d, const void* x_nchw,
                               void* x_packed, void* stream);
/* OIHW f32 (or i8) -> packed weights (KRSC, or [R][S][C] for depthwise). */
tec_status tec_weight_pretransform(const tec_conv_desc* d, const void* w_oihw,
                                   void* w_packed, void* stream);
/* tec_weight_pretransform with batch-norm folding (SURVEY 8f.4,
 * graph.py fold_batch_norm): packs w[k][c][r][s] * scale[k] (each product
 * rounded to f32 once -- graph.py bn_fold_weight), scale = the device f32
 * vector gamma / sqrt(var + eps). F32 / F32TC / BF16 weights (not I8). */
tec_status tec_weight_pretransform_bn(const tec_conv_desc* d, const void* w_oihw,
                                      const float* scale, void* w_packed, void* stream);
/* f32 NHWC [n*h*w][c] (an f32tc layer's output) -> the packed input of an
 * f32tc dense conv (its three exact bf16 planes), without the NCHW detour. */
tec_status tec_activation_pack_nhwc(const tec_conv_desc* d, const void* x_nhwc_f32,
                                    void* x_packed, void* stream);
/* NCHW (f32 / i32) -> NHWC in out_dtype (residual/mul operands). */
tec_status tec_nchw_to_nhwc(const void* src, int32_t src_dtype, void* dst,
                            int32_t dst_dtype, int64_t n, int64_t c,
                            int64_t h, int64_t w, void* stream);
/* NHWC [n*h*w][c] (f32/bf16/i32) -> NCHW (f32 or i32). */
tec_status tec_output_unpack(const void* y_nhwc, int32_t y_dtype, void* y_nchw,
                             int32_t dst_dtype, int64_t n, int64_t c,
                             int64_t h, int64_t w, void* stream);

/* Fused conv: y (NHWC [N*OH*OW][K], out_dtype f32/bf16, or i32 for I8)
 * = epilogue(conv(x_packed, w_packed)). Epilogue operands are device
 * pointers: bias [K] (f32 / i32), residual & mul NHWC in out_dtype.
 * err_flag (device int32, may be NULL) is OR-ed with 1 on i32 overflow. */
tec_status tec_conv2d_fused(const tec_conv_desc* d, const tec_epilogue* epi,
                            const tec_knobs* knobs, const void* x_packed,
                            const void* w_packed, void* y, int32_t out_dtype,
                            int32_t* err_flag, void* stream);
tec_status tec_depthwise_fused(const tec_conv_desc* d, const tec_epilogue* epi,
                               const tec_knobs* knobs, const void* x_packed,
                               const void* w_packed, void* y,
                               int32_t out_dtype, int32_t* err_flag,
                               void* stream);
/* Device scratch a tec_conv2d_fused_ws launch of this desc + knobs needs
 * (split-K partial tiles + tile counters; 0 for every other schedule). */
tec_status tec_workspace_bytes(const tec_conv_desc* d, const tec_epilogue* epi,
                               const tec_knobs* knobs, size_t* bytes);
/* tec_conv2d_fused on a CALLER-OWNED workspace of >= tec_workspace_bytes
 * bytes, zero-filled before its first use (every launch leaves its counter
 * region zeroed; one workspace may serve launches of different shapes).
 * Nothing is allocated on this path; a workspace may be shared by launches
 * that are ordered on one stream. CapacityError if ws_bytes is too small.
 * (tec_conv2d_fused without a workspace uses a grow-only internal scratch
 * per (device, stream), never freed while the library is loaded.) */
tec_status tec_conv2d_fused_ws(const tec_conv_desc* d, const tec_epilogue* epi,
                               const tec_knobs* knobs, const void* x_packed,
                               const void* w_packed, void* y, int32_t out_dtype,
                               int32_t* err_flag, void* ws, size_t ws_bytes,
                               void* stream);

/* ---- lowering (target "sm100"): the kernel a descriptor + knobs lower to,
 * without launching (LowerOptions::target, R/include/tec/lower.hpp:26-33;
 * capacity checks replace check_target). LoweringError when no kernel fits. */
typedef enum {
  TEC_KERNEL_IM2COL = 1,     /* conv_tc.cu: TMA im2col implicit GEMM      */
  TEC_KERNEL_HALO = 2,       /* conv_halo.cu: shifted-window implicit GEMM */
  TEC_KERNEL_F32_EXACT = 3,  /* conv_f32_exact.cu: SIMT, reference order  */
  TEC_KERNEL_DW_TMA = 4,     /* depthwise_tma.cu                           */
  TEC_KERNEL_DW_DIRECT = 5,  /* depthwise.cu                               */
  TEC_KERNEL_F32TC = 6,      /* conv_f32tc.cu: split-bf16 f32 on tcgen05    */
  TEC_KERNEL_F32TC_HALO = 7  /* conv_f32tc.cu, shifted-window (stride 1)    */
} tec_kernel_family;

typedef struct {
  int32_t family;                    /* tec_kernel_family */
  int32_t tile_m, tile_n, stages;    /* rows / output channels per tile; stages
                                        (halo: 1 streamed, 2 resident weights) */
  int32_t split_k, cluster;          /* K splits; CTAs sharing weights       */
  int32_t grid;                      /* persistent CTAs (0: data-dependent)  */
  int32_t smem_bytes, tmem_cols;     /* per-CTA on-chip budget used          */
  int32_t tma_store;                 /* 1: TMA-store epilogue                */
  int64_t workspace_bytes;           /* device scratch the launch needs (split-K
                                        partials + tile counters); 0 = none  */
} tec_kernel_plan;

tec_status tec_conv_plan(const tec_conv_desc* d, const tec_epilogue* epi,
                         const tec_knobs* knobs, tec_kernel_plan* out);

/* ---- graph operators around the conv path (ResNet-18 graph).
 * The reference has no pooling operator; these are new registered ops
 * whose semantics oracle/tec_oracle.c restates (see pool.cu). NHWC device
 * tensors; dtype/out_dtype are tec_dtype. */
typedef struct {
  int64_t n, c, h, w;                      /* input, logical NCHW dims   */
  int64_t r, s;                            /* window (max_pool2d)        */
  int64_t stride_h, stride_w, pad_h, pad_w;
  int32_t dtype, out_dtype;
} tec_pool_desc;

/* max_pool2d: y NHWC [n][oh][ow][c], oh = (h + 2ph - r)/sh + 1; padded taps
 * are skipped. dtype == out_dtype (f32, bf16, i32, i8); c*elem % 16 == 0. */
tec_status tec_max_pool2d(const tec_pool_desc* d, const void* x, void* y, void* stream);
/* global_avg_pool == scale(sum(sum(x, W), H), 1/(h*w)) in float:
 * y [n][c] (f32 or bf16) from x NHWC (f32 or bf16). */
tec_status tec_global_avg_pool(const tec_pool_desc* d, const void* x, void* y, void* stream);
tec_status tec_pool_infer(const tec_pool_desc* d, int64_t out_shape[4]);

/* ---- unary integer graph operators around the int8 conv path (int8
 * ResNet-18 end to end). Not in the reference registry (like
 * the pools): new registered ops (graph.py "cast", "requantize"; the
 * reference's own "scale" and "relu") whose semantics elementwise.cu states
 * and tests/graph_oracle.py restates. A program is the member chain of one
 * fused elementwise node, applied per element in member order:
 *   CAST        i8 -> i32 exact; i8 | i32 -> f32 (round to nearest)
 *   SCALE       integer data: x * c, integral |c| < 2^32, int64 product with
 *               the i32 range check (DenseTensor::set_i) -> err flag, which
 *               the caller reports as TEC_E_FOLD_OVERFLOW; f32 data: x * (float)c
 *   RELU        max(x, 0)
 *   REQUANTIZE  i32 -> i8: clamp((x * mult + 2^(shift-1)) >> shift, -128, 127),
 *               1 <= mult < 2^31, 0 <= shift <= 62 (ties toward +inf)
 * x / y: device buffers, 16-byte aligned; count elements (any layout). */
typedef enum {
  TEC_ELEM_CAST = 1,
  TEC_ELEM_SCALE = 2,
  TEC_ELEM_RELU = 3,
  TEC_ELEM_REQUANTIZE = 4
} tec_elem_kind;

#define TEC_MAX_ELEM_OPS 4
typedef struct {
  int32_t n_ops;
  int32_t kind[TEC_MAX_ELEM_OPS];   /* tec_elem_kind                         */
  int32_t shift[TEC_MAX_ELEM_OPS];  /* REQUANTIZE                            */
  int32_t cast_to[TEC_MAX_ELEM_OPS];/* CAST: target tec_dtype                */
  int64_t mult[TEC_MAX_ELEM_OPS];   /* REQUANTIZE multiplier                 */
  double scale[TEC_MAX_ELEM_OPS];   /* SCALE factor                          */
  int32_t src_dtype, dst_dtype;     /* tec_dtype of x and y                  */
  int64_t count;
} tec_elem_prog;

/* Validates the program against the dtypes (a chain whose value type does
 * not end in dst_dtype, a REQUANTIZE of non-integer data, ... are
 * TEC_E_LOWERING) and launches it. err_flag (device int32, may be null) is
 * set to 1 on an i32 range overflow. */
tec_status tec_elementwise(const tec_elem_prog* p, const void* x, void* y,
                           int32_t* err_flag, void* stream);

/* ---- native launch plans: the executor's run loop (evaluate_graph for
 * target sm100, R/src/graph.cpp:227-256). A compiled graph is a list of
 * steps on caller-owned device buffers; the plan runs them in order or
 * captures them ONCE into a CUDA graph and replays that. */
typedef enum {
  TEC_STEP_CONV = 1,       /* tec_conv2d_fused                              */
  TEC_STEP_MAX_POOL = 2,   /* tec_max_pool2d                                */
  TEC_STEP_AVG_POOL = 3,   /* tec_global_avg_pool                           */
  TEC_STEP_PACK = 4,       /* tec_activation_pack(conv, src -> dst)         */
  TEC_STEP_UNPACK = 5,     /* tec_output_unpack(src, src_dtype -> dst)      */
  TEC_STEP_TO_NHWC = 6,    /* tec_nchw_to_nhwc(src, src_dtype -> dst)       */
  TEC_STEP_DEPTHWISE = 7,  /* tec_depthwise_fused                           */
  TEC_STEP_PACK_NHWC = 8,  /* tec_activation_pack_nhwc(conv, src -> dst)    */
  TEC_STEP_ELEMWISE = 9    /* tec_elementwise(elem, src -> dst)             */
} tec_step_kind;

typedef struct {
  int32_t kind;            /* tec_step_kind */
  int32_t src_dtype, dst_dtype;
  tec_conv_desc conv;      /* CONV, DEPTHWISE, PACK */
  tec_epilogue epi;        /* CONV, DEPTHWISE (device operand pointers)     */
  tec_knobs knobs;         /* CONV, DEPTHWISE */
  tec_pool_desc pool;      /* MAX_POOL, AVG_POOL */
  const void* src;         /* input (x / NCHW source)                       */
  const void* w;           /* CONV, DEPTHWISE: packed weights               */
  void* dst;               /* output                                        */
  int64_t n, c, h, w_;     /* UNPACK / TO_NHWC logical NCHW dims            */
  tec_elem_prog elem;      /* ELEMWISE */
} tec_step;

typedef struct tec_plan tec_plan;
/* Copies the steps; LoweringError if a conv step has no kernel. */
tec_status tec_plan_create(const tec_step* steps, int32_t n_steps, tec_plan** out);
/* Enqueues the plan on `stream`: the captured CUDA graph when there is one,
 * otherwise every step in order. */
tec_status tec_plan_run(tec_plan* plan, void* stream);
/* Runs the steps once eagerly (first-use setup), then captures them into a
 * CUDA graph that later tec_plan_run calls replay. */
tec_status tec_plan_capture(tec_plan* plan, void* stream);
/* Runs steps [first, first + count) eagerly (per-launch profiling). */
tec_status tec_plan_run_steps(tec_plan* plan, int32_t first, int32_t count, void* stream);
int32_t tec_plan_size(const tec_plan* plan);
/* Integer range overflow raised by any step since the last call (the plan
 * owns one device flag that its conv and elementwise steps share):
 * synchronizes `stream`, clears the flag, returns TEC_E_FOLD_OVERFLOW if it
 * was set (the reference throws at the member that overflows). */
tec_status tec_plan_status(tec_plan* plan, void* stream);
void tec_plan_destroy(tec_plan* plan);

/* ---- host-level path: eval_graph_node / native_eval for target sm100 ----
 * x: NCHW f32 (i8 for I8); w: OIHW f32 (i8); epilogue operands NCHW f32
 * (i32); y: NCHW f32 (i32). All HOST pointers; copies included. */
tec_status tec_eval_fused_conv(const tec_conv_desc* d, const tec_epilogue* epi,
                               const tec_knobs* knobs, const void* x,
                               const void* w, void* y, int device);

/* On-device timing of one fused-conv configuration with synthetic data:
 * CUDA events around `reps` launches after `warmup`, L2 flushed between
 * reps when flush_l2 != 0; writes the median in microseconds. */
tec_status tec_measure(const tec_conv_desc* d, const tec_epilogue* epi,
                       const tec_knobs* knobs, int device, int warmup,
                       int reps, int flush_l2, double* median_us);

#ifdef __cplusplus
}
#endif
#endif /* TEC_SM100_H_ */
