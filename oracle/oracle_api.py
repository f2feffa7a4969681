"""TEST INFRASTRUCTURE ONLY: Python access to the two checkers.

* ``fused_conv``      -> oracle/_build/libtec_oracle.so, the plain-C
  restatement (oracle/tec_oracle.c) of make_conv + evaluate_reference +
  fused members (R/src/ops.cpp:120-305, R/src/texpr.cpp:178-262,
  R/src/graph.cpp:209-222).
* ``load_tensor`` / ``save_tensor`` -> the reference's on-disk tensor format
  (R/src/io.cpp:111-127), used by the golden fixtures.
* ``same_values``     -> DenseTensor::same_values (R/src/tensor.cpp:56-72).
* ``ref_driver``      -> path of the reference binary (oracle/_ref), when
  it has been built (build container, or shipped to the GPU box).
"""
from __future__ import annotations

import ctypes as C
import json
import os
import subprocess
from typing import Optional, Sequence

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
PORT_LIB = os.path.join(HERE, "_build", "libtec_oracle.so")
REF_DRIVER = os.path.join(HERE, "_ref", "ref_driver")

SCALE, BIAS, ADD, MUL, RELU = 1, 2, 3, 4, 5
_EPI = {"scale": SCALE, "bias_add": BIAS, "add": ADD, "mul": MUL, "relu": RELU}


class _Epi(C.Structure):
    _fields_ = [("op", C.c_int32), ("scale", C.c_double),
                ("operand", C.c_void_p)]


class _Conv(C.Structure):
    _fields_ = [(n, C.c_int64) for n in
                ("n", "c", "h", "w", "oc", "kh", "kw", "sh", "sw", "ph",
                 "pw")] + [("depthwise", C.c_int32)]


_lib = None


def build_port() -> None:
    subprocess.run(["make", "-s", "-C", HERE, "port"], check=True)


def _load():
    global _lib
    if _lib is None:
        if not os.path.exists(PORT_LIB):
            build_port()
        lib = C.CDLL(PORT_LIB)
        for fn in (lib.tec_oracle_fused_conv_f32, lib.tec_oracle_fused_conv_i8):
            fn.restype = C.c_int
            fn.argtypes = [C.POINTER(_Conv), C.c_void_p, C.c_void_p,
                           C.POINTER(_Epi), C.c_int, C.c_void_p, C.c_int]
        i64 = C.c_int64
        lib.tec_oracle_max_pool2d_f32.restype = C.c_int
        lib.tec_oracle_max_pool2d_f32.argtypes = [C.c_void_p] + [i64] * 10 + [C.c_void_p]
        lib.tec_oracle_global_avg_pool_f32.restype = C.c_int
        lib.tec_oracle_global_avg_pool_f32.argtypes = [C.c_void_p] + [i64] * 4 + [C.c_void_p]
        _lib = lib
    return _lib


def max_pool2d(x: np.ndarray, kernel=(3, 3), strides=(2, 2), padding=(1, 1)) -> np.ndarray:
    """max_pool2d on NCHW f32 (tec_oracle.c); padded taps never win."""
    x = np.ascontiguousarray(x, dtype=np.float32)
    n, c, h, w = x.shape
    (r, s), (sh, sw), (ph, pw) = kernel, strides, padding
    oh, ow = (h + 2 * ph - r) // sh + 1, (w + 2 * pw - s) // sw + 1
    y = np.empty((n, c, oh, ow), np.float32)
    st = _load().tec_oracle_max_pool2d_f32(x.ctypes.data, n, c, h, w, r, s, sh, sw, ph, pw,
                                           y.ctypes.data)
    if st:
        raise OracleError(st)
    return y


def global_avg_pool(x: np.ndarray) -> np.ndarray:
    """scale(sum(sum(x, axis=3), axis=2), 1/(H*W)) in float: [N, C]."""
    x = np.ascontiguousarray(x, dtype=np.float32)
    n, c, h, w = x.shape
    y = np.empty((n, c), np.float32)
    _load().tec_oracle_global_avg_pool_f32(x.ctypes.data, n, c, h, w, y.ctypes.data)
    return y


class OracleError(RuntimeError):
    def __init__(self, status):
        self.status = status
        super().__init__(f"oracle status {status}")


def out_shape(op, x_shape, w_shape, strides=(1, 1), padding=(0, 0)):
    n, _, h, w = x_shape
    k, _, r, s = w_shape
    return (n, k, (h + 2 * padding[0] - r) // strides[0] + 1,
            (w + 2 * padding[1] - s) // strides[1] + 1)


def fused_conv(op: str, x: np.ndarray, w: np.ndarray, strides=(1, 1),
               padding=(0, 0), epilogue: Sequence[tuple] = (),
               threads: Optional[int] = None) -> np.ndarray:
    """Reference-order evaluation of [conv, epilogue...]; f32 or i8 -> i32."""
    lib = _load()
    integer = x.dtype == np.int8
    x = np.ascontiguousarray(x)
    w = np.ascontiguousarray(w)
    d = _Conv(n=x.shape[0], c=x.shape[1], h=x.shape[2], w=x.shape[3],
              oc=w.shape[0], kh=w.shape[2], kw=w.shape[3], sh=strides[0],
              sw=strides[1], ph=padding[0], pw=padding[1],
              depthwise=1 if op == "depthwise_conv2d" else 0)
    shp = out_shape(op, x.shape, w.shape, strides, padding)
    y = np.empty(shp, np.int32 if integer else np.float32)
    epis = (_Epi * max(1, len(epilogue)))()
    keep = []
    for i, item in enumerate(epilogue):
        epis[i].op = _EPI[item[0]]
        if item[0] == "scale":
            epis[i].scale = float(item[1])
        elif item[0] != "relu":
            a = np.ascontiguousarray(item[1])
            keep.append(a)
            epis[i].operand = a.ctypes.data
    fn = lib.tec_oracle_fused_conv_i8 if integer else lib.tec_oracle_fused_conv_f32
    st = fn(C.byref(d), x.ctypes.data, w.ctypes.data, epis, len(epilogue),
            y.ctypes.data, threads or os.cpu_count() or 1)
    if st:
        raise OracleError(st)
    return y


def same_values(a: np.ndarray, b: np.ndarray, rel_tol: float) -> bool:
    """DenseTensor::same_values (R/src/tensor.cpp:56-72)."""
    if a.shape != b.shape or a.dtype != b.dtype:
        return False
    if a.dtype.kind in "iu":
        return bool(np.array_equal(a, b))
    a64 = a.astype(np.float64)
    b64 = b.astype(np.float64)
    if np.isnan(a64).any() or np.isnan(b64).any():
        return False
    denom = np.maximum(np.maximum(np.abs(a64), np.abs(b64)), 1.0)
    return bool(np.all(np.abs(a64 - b64) <= rel_tol * denom))


def max_rel_err(a: np.ndarray, b: np.ndarray) -> float:
    a64 = a.astype(np.float64)
    b64 = b.astype(np.float64)
    denom = np.maximum(np.maximum(np.abs(a64), np.abs(b64)), 1.0)
    return float(np.max(np.abs(a64 - b64) / denom)) if a.size else 0.0


_NP = {"f32": np.float32, "i32": np.int32, "i8": np.int8}


def load_tensor(d: str, name: str) -> np.ndarray:
    """load_tensor (R/src/io.cpp:121-127)."""
    with open(os.path.join(d, name + ".json")) as f:
        m = json.load(f)
    dt = _NP[m["dtype"]]
    raw = np.fromfile(os.path.join(d, name + ".bin"), dtype=dt)
    return raw.reshape(m["shape"])


def save_tensor(d: str, name: str, a: np.ndarray) -> None:
    """save_tensor (R/src/io.cpp:111-119): raw row-major bytes + a JSON header."""
    dt = {np.dtype(np.float32): "f32", np.dtype(np.int32): "i32", np.dtype(np.int8): "i8"}[a.dtype]
    np.ascontiguousarray(a).tofile(os.path.join(d, name + ".bin"))
    with open(os.path.join(d, name + ".json"), "w") as f:
        json.dump({"dtype": dt, "name": name, "shape": list(a.shape)}, f)


def bf16_round(a: np.ndarray) -> np.ndarray:
    """Round-to-nearest-even onto bf16, returned as f32 (what the bf16 path
    feeds the tensor cores)."""
    u = np.ascontiguousarray(a, dtype=np.float32).view(np.uint32)
    r = ((u + 0x7FFF + ((u >> 16) & 1)) & 0xFFFF0000).astype(np.uint32)
    return r.view(np.float32)
