"""ctypes binding of the C ABI in include/tec_sm100.h (libtec_sm100.so).

The shared library is built in-tree (paper_1802_04799_b200/lib/) by
``make -C paper_1802_04799_b200`` / ``__graft_entry__.build()``. There is
no fallback: if the library is missing, importing the compute entry points
raises -- the product path never silently degrades to CPU code.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "lib", "libtec_sm100.so")

# Status codes: 1 + tec::ErrorCode (R/include/tec/error.hpp:25-47).
ERROR_NAMES = [
    "UnknownOperator", "ShapeMismatch", "FoldOverflow", "UnboundAxis",
    "DuplicateIntrinsic", "InvalidFactor", "IllegalReorder",
    "IllegalAnnotation", "IllegalBind", "BindConflict", "IllegalComputeAt",
    "ScopeError", "CapacityError", "TensorizeMismatch", "LoweringError",
    "BoundsError", "DeadlockError", "RaceError", "NotEnoughData", "IOError",
    "Internal",
]
TEC_E_CUDA = 64

DT_F32, DT_I32, DT_I8, DT_BF16 = 0, 1, 2, 3
COMPUTE_BF16, COMPUTE_F32TC, COMPUTE_I8, COMPUTE_F32 = 1, 2, 3, 4
EPI_SCALE, EPI_BIAS, EPI_ADD, EPI_MUL, EPI_RELU, EPI_REQUANTIZE = 1, 2, 3, 4, 5, 6
MAX_EPILOGUE = 8


class TecError(RuntimeError):
    """Mirror of tec::Error: carries the stable error code."""

    def __init__(self, status: int, msg: str):
        self.status = status
        if 1 <= status <= len(ERROR_NAMES):
            self.code = ERROR_NAMES[status - 1]
        elif status == TEC_E_CUDA:
            self.code = "CudaError"
        else:
            self.code = f"status{status}"
        super().__init__(f"{self.code}: {msg}")


class ConvDesc(C.Structure):
    _fields_ = [(n, C.c_int64) for n in
                ("n", "c", "h", "w", "k", "r", "s", "stride_h", "stride_w",
                 "pad_h", "pad_w")] + [("depthwise", C.c_int32),
                                       ("compute", C.c_int32)]


class Epilogue(C.Structure):
    _fields_ = [("n_ops", C.c_int32),
                ("ops", C.c_int32 * MAX_EPILOGUE),
                ("scale", C.c_double * MAX_EPILOGUE),
                ("bias", C.c_void_p),
                ("residual", C.c_void_p),
                ("mul_operand", C.c_void_p),
                ("rq_mult", C.c_int64),
                ("rq_shift", C.c_int32),
                ("residual_i8", C.c_int32),
                ("residual_scale", C.c_int64)]


class Knobs(C.Structure):
    _fields_ = [(n, C.c_int64) for n in
                ("tile_m", "tile_n", "tile_k", "stages", "cta_pair",
                 "cluster_m", "cluster_n", "raster", "swizzle", "split_k",
                 "vec", "unroll", "acc_bufs", "grid")]


class PoolDesc(C.Structure):
    """tec_pool_desc (include/tec_sm100.h)."""
    _fields_ = [(f, C.c_int64) for f in ("n", "c", "h", "w", "r", "s", "stride_h", "stride_w",
                                         "pad_h", "pad_w")] + \
               [("dtype", C.c_int32), ("out_dtype", C.c_int32)]


class KernelPlan(C.Structure):
    """tec_kernel_plan (include/tec_sm100.h)."""
    _fields_ = [(f, C.c_int32) for f in ("family", "tile_m", "tile_n", "stages", "split_k",
                                         "cluster", "grid", "smem_bytes", "tmem_cols",
                                         "tma_store")] + [("workspace_bytes", C.c_int64)]


class ConvLayout(C.Structure):
    _fields_ = [("oh", C.c_int64), ("ow", C.c_int64), ("cp", C.c_int64),
                ("act_dtype", C.c_int32), ("acc_dtype", C.c_int32),
                ("act_bytes", C.c_int64), ("wt_bytes", C.c_int64),
                ("out_elems", C.c_int64)]


STEP_CONV, STEP_MAX_POOL, STEP_AVG_POOL, STEP_PACK, STEP_UNPACK, STEP_TO_NHWC, STEP_DEPTHWISE, \
    STEP_PACK_NHWC, STEP_ELEMWISE = 1, 2, 3, 4, 5, 6, 7, 8, 9

ELEM_CAST, ELEM_SCALE, ELEM_RELU, ELEM_REQUANTIZE = 1, 2, 3, 4
MAX_ELEM_OPS = 4


class ElemProg(C.Structure):
    """tec_elem_prog (include/tec_sm100.h): a unary member chain."""
    _fields_ = [("n_ops", C.c_int32), ("kind", C.c_int32 * MAX_ELEM_OPS),
                ("shift", C.c_int32 * MAX_ELEM_OPS), ("cast_to", C.c_int32 * MAX_ELEM_OPS),
                ("mult", C.c_int64 * MAX_ELEM_OPS), ("scale", C.c_double * MAX_ELEM_OPS),
                ("src_dtype", C.c_int32), ("dst_dtype", C.c_int32), ("count", C.c_int64)]


class Step(C.Structure):
    """tec_step (include/tec_sm100.h): one launch of a native plan."""
    _fields_ = [("kind", C.c_int32), ("src_dtype", C.c_int32), ("dst_dtype", C.c_int32),
                ("conv", ConvDesc), ("epi", Epilogue), ("knobs", Knobs), ("pool", PoolDesc),
                ("src", C.c_void_p), ("w", C.c_void_p), ("dst", C.c_void_p),
                ("n", C.c_int64), ("c", C.c_int64), ("h", C.c_int64), ("w_", C.c_int64),
                ("elem", ElemProg)]


# Every symbol include/tec_sm100.h declares, with its ctypes signature.
_P = C.c_void_p
_DESC = C.POINTER(ConvDesc)
_EPI = C.POINTER(Epilogue)
_KN = C.POINTER(Knobs)
SIGNATURES = {
    "tec_api_version": (C.c_int, []),
    "tec_last_error": (C.c_char_p, []),
    "tec_device_sm_count": (C.c_int, [C.c_int]),
    "tec_conv_infer": (C.c_int32, [_DESC, C.POINTER(C.c_int64)]),
    "tec_conv_layout_of": (C.c_int32, [_DESC, C.POINTER(ConvLayout)]),
    "tec_activation_pack": (C.c_int32, [_DESC, _P, _P, _P]),
    "tec_activation_pack_nhwc": (C.c_int32, [_DESC, _P, _P, _P]),
    "tec_weight_pretransform": (C.c_int32, [_DESC, _P, _P, _P]),
    "tec_nchw_to_nhwc": (C.c_int32, [_P, C.c_int32, _P, C.c_int32, C.c_int64,
                                     C.c_int64, C.c_int64, C.c_int64, _P]),
    "tec_output_unpack": (C.c_int32, [_P, C.c_int32, _P, C.c_int32, C.c_int64,
                                      C.c_int64, C.c_int64, C.c_int64, _P]),
    "tec_conv2d_fused": (C.c_int32, [_DESC, _EPI, _KN, _P, _P, _P, C.c_int32,
                                     _P, _P]),
    "tec_depthwise_fused": (C.c_int32, [_DESC, _EPI, _KN, _P, _P, _P,
                                        C.c_int32, _P, _P]),
    "tec_workspace_bytes": (C.c_int32, [_DESC, _EPI, _KN, C.POINTER(C.c_size_t)]),
    "tec_conv2d_fused_ws": (C.c_int32, [_DESC, _EPI, _KN, _P, _P, _P, C.c_int32, _P, _P,
                                        C.c_size_t, _P]),
    "tec_eval_fused_conv": (C.c_int32, [_DESC, _EPI, _KN, _P, _P, _P, C.c_int]),
    "tec_measure": (C.c_int32, [_DESC, _EPI, _KN, C.c_int, C.c_int, C.c_int,
                                C.c_int, C.POINTER(C.c_double)]),
    "tec_pool_infer": (C.c_int32, [C.POINTER(PoolDesc), C.POINTER(C.c_int64)]),
    "tec_conv_plan": (C.c_int32, [_DESC, _EPI, _KN, C.POINTER(KernelPlan)]),
    "tec_max_pool2d": (C.c_int32, [C.POINTER(PoolDesc), _P, _P, _P]),
    "tec_global_avg_pool": (C.c_int32, [C.POINTER(PoolDesc), _P, _P, _P]),
    "tec_plan_create": (C.c_int32, [C.POINTER(Step), C.c_int32, C.POINTER(C.c_void_p)]),
    "tec_plan_run": (C.c_int32, [_P, _P]),
    "tec_plan_capture": (C.c_int32, [_P, _P]),
    "tec_plan_run_steps": (C.c_int32, [_P, C.c_int32, C.c_int32, _P]),
    "tec_plan_size": (C.c_int32, [_P]),
    "tec_plan_status": (C.c_int32, [_P, _P]),
    "tec_elementwise": (C.c_int32, [C.POINTER(ElemProg), _P, _P, _P, _P]),
    "tec_weight_pretransform_bn": (C.c_int32, [_DESC, _P, _P, _P, _P]),
    "tec_plan_destroy": (None, [_P]),
}

_lib = None


def load() -> C.CDLL:
    """Load libtec_sm100.so (raises if it has not been built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(
            f"{LIB_PATH} is missing: build it with `make -C {_HERE}` "
            "(or __graft_entry__.build()); there is no CPU fallback")
    lib = C.CDLL(LIB_PATH)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def check(status: int) -> None:
    if status != 0:
        msg = load().tec_last_error().decode(errors="replace")
        raise TecError(status, msg)
