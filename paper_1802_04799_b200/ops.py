"""Host-side mirror of the reference operator API for the fused-conv path.

Reference interface (R = /root/reference/proj) and what stands in for it:

  eval_operator(op, inputs, attrs)      R/src/ops.cpp:517-531
      -> conv2d / depthwise_conv2d on the sm_100a kernels
  eval_graph_node(node, inputs)         R/src/graph.cpp:209-225
      -> one fused kernel for a fused [conv, scale?, bias_add?, add?, mul?,
         relu?] node (the reference runs members one by one)
  infer_type (infer_conv)               R/src/ops.cpp:163-192

Tensors are numpy arrays in the reference's DenseTensor layout (row-major
NCHW / OIHW); dtypes f32 / i8 / i32 as tec::DType. Errors raise TecError
carrying the reference's ErrorCode name.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import Any, Dict, List, Optional, Sequence

import numpy as np

from . import _abi
from ._abi import (COMPUTE_BF16, COMPUTE_F32, COMPUTE_F32TC, COMPUTE_I8, EPI_ADD,
                   EPI_BIAS, EPI_MUL, EPI_RELU, EPI_SCALE, TecError)

AttrMap = Dict[str, Any]

_COMPUTE_NAMES = {"bf16": COMPUTE_BF16, "f32tc": COMPUTE_F32TC,
                  "fp32": COMPUTE_F32, "f32": COMPUTE_F32, "i8": COMPUTE_I8}
_EPI_OPS = {"scale": EPI_SCALE, "bias_add": EPI_BIAS, "add": EPI_ADD,
            "mul": EPI_MUL, "relu": EPI_RELU}


# The graph node type is the reference mirror in graph.py (graph.hpp:38-47).
from .graph import GraphNode  # noqa: E402


def _pair(attrs: AttrMap, key: str, dflt: Sequence[int]) -> List[int]:
    v = list(attrs.get(key, dflt))
    if len(v) != 2:
        raise TecError(2, "conv2d strides/padding must be pairs")
    return [int(a) for a in v]


def conv_desc(op: str, x_shape, w_shape, attrs: AttrMap,
              compute: int, out_shape: Optional[list] = None) -> _abi.ConvDesc:
    """Builds the C descriptor with infer_conv's checks (ops.cpp:163-192);
    `out_shape`, when given, receives the NCHW output shape the C ABI
    inferred (the one source of truth for buffer sizes)."""
    if op not in ("conv2d", "depthwise_conv2d"):
        raise TecError(1, f"no sm100 kernel for operator '{op}'")
    if len(x_shape) != 4 or len(w_shape) != 4:
        raise TecError(2, f"{op} wants NCHW data, OIHW weights")
    dw = op == "depthwise_conv2d"
    strides = _pair(attrs, "strides", (1, 1))
    padding = _pair(attrs, "padding", (0, 0))
    n, c, h, w = (int(v) for v in x_shape)
    k, wc, r, s = (int(v) for v in w_shape)
    if dw:
        if k != c or wc != 1:
            raise TecError(2, f"{op} weights must be [C,1,kh,kw] with C={c}")
    elif wc != c:
        raise TecError(2, f"{op}: weight input-channel dim {wc} != data channels {c}")
    d = _abi.ConvDesc(n=n, c=c, h=h, w=w, k=k, r=r, s=s,
                      stride_h=strides[0], stride_w=strides[1],
                      pad_h=padding[0], pad_w=padding[1],
                      depthwise=1 if dw else 0, compute=compute)
    out = (C.c_int64 * 4)()
    _abi.check(_abi.load().tec_conv_infer(C.byref(d), out))
    if out_shape is not None:
        out_shape[:] = [int(v) for v in out]
    return d


def _compute_for(dtype: np.dtype, compute: Optional[str]) -> int:
    if dtype == np.int8:
        if compute not in (None, "i8"):
            raise TecError(2, "i8 operands run on the i8 path only")
        return COMPUTE_I8
    if dtype != np.float32:
        raise TecError(2, f"unsupported operand dtype {dtype}")
    if compute is None:
        return COMPUTE_F32  # bit-exact f32 parity path by default
    if compute not in _COMPUTE_NAMES or compute == "i8":
        raise TecError(15, f"unknown compute mode '{compute}'")
    return _COMPUTE_NAMES[compute]


def fused_conv(op: str, x: np.ndarray, w: np.ndarray, attrs: AttrMap,
               epilogue: Sequence[tuple] = (), *, compute: Optional[str] = None,
               knobs: Optional[Dict[str, int]] = None, device: int = 0) -> np.ndarray:
    """conv (+ epilogue members in order) through tec_eval_fused_conv.

    epilogue items: ("scale", c) | ("bias_add", b[K]) | ("add", r) |
    ("mul", r) | ("relu",) with r in the output's NCHW shape.
    """
    if x.dtype != w.dtype:
        raise TecError(2, f"{op} operand dtypes differ")
    cm = _compute_for(x.dtype, compute)
    shape: list = []
    d = conv_desc(op, x.shape, w.shape, attrs, cm, shape)
    acc = np.int32 if cm == COMPUTE_I8 else np.float32
    out_shape = tuple(shape)
    epi = _abi.Epilogue()
    keep = []
    if len(epilogue) > _abi.MAX_EPILOGUE:
        raise TecError(15, "too many fused epilogue members")
    for i, item in enumerate(epilogue):
        name = item[0]
        if name not in _EPI_OPS:
            raise TecError(1, f"'{name}' cannot be fused into a conv epilogue")
        epi.ops[i] = _EPI_OPS[name]
        if name == "scale":
            epi.scale[i] = float(item[1])
        elif name == "bias_add":
            b = np.ascontiguousarray(item[1])
            if b.shape != (d.k,) or b.dtype != acc:
                raise TecError(2, "bias must be rank-1 matching dim 1")
            keep.append(b)
            epi.bias = b.ctypes.data
        elif name in ("add", "mul"):
            r = np.ascontiguousarray(item[1])
            if r.shape != out_shape or r.dtype != acc:
                raise TecError(2, f"{name} operand types differ")
            keep.append(r)
            if name == "add":
                epi.residual = r.ctypes.data
            else:
                epi.mul_operand = r.ctypes.data
    epi.n_ops = len(epilogue)
    names = [it[0] for it in epilogue]
    for op in ("bias_add", "add", "mul"):
        if names.count(op) > 1:  # one operand slot each in tec_epilogue
            raise TecError(15, f"more than one '{op}' member in one fused conv")
    kn = _abi.Knobs(**(knobs or {}))
    x = np.ascontiguousarray(x)
    w = np.ascontiguousarray(w)
    y = np.empty(out_shape, dtype=acc)
    _abi.check(_abi.load().tec_eval_fused_conv(
        C.byref(d), C.byref(epi), C.byref(kn), x.ctypes.data, w.ctypes.data,
        y.ctypes.data, device))
    return y


def eval_operator(op: str, inputs: Sequence[np.ndarray], attrs: AttrMap = None,
                  **kw) -> np.ndarray:
    """eval_operator (R/src/ops.cpp:517-531) for the conv operators."""
    attrs = attrs or {}
    if len(inputs) != 2:
        raise TecError(2, f"{op} expects 2 inputs, got {len(inputs)}")
    return fused_conv(op, inputs[0], inputs[1], attrs, (), **kw)


def epilogue_of(node: GraphNode, inputs: Sequence[np.ndarray]):
    """Maps a fused node's members to (conv member, epilogue items).

    The member list must be exactly what fuse_pass builds for this path
    (R/src/graph_passes.cpp:219-248): a complex-out-fusable conv first,
    then injective members each consuming the previous member's result.
    """
    env = {nid: t for nid, t in zip(node.inputs, inputs)}
    ms = node.members
    if not ms or ms[0].op not in ("conv2d", "depthwise_conv2d"):
        raise TecError(15, "fused node is not a conv-rooted group")
    conv = ms[0]
    items = []
    prev = conv.id
    for m in ms[1:]:
        if m.op not in _EPI_OPS:
            raise TecError(15, f"member '{m.op}' has no sm100 epilogue")
        others = [i for i in m.inputs if i != prev]
        if prev not in m.inputs or len(others) != len(m.inputs) - 1:
            raise TecError(15, "fused members are not a single chain")
        if m.op == "relu":
            items.append(("relu",))
        elif m.op == "scale":
            items.append(("scale", float(m.attrs.get("scale", 1.0))))
        else:
            if len(others) != 1 or others[0] not in env:
                raise TecError(15, f"member {m.id} reads an internal tensor")
            if m.op == "bias_add":
                ax = int(m.attrs.get("axis", 1))
                if ax != 1:
                    raise TecError(15, "bias_add must broadcast over channels")
            items.append((m.op, env[others[0]]))
        prev = m.id
    return conv, [env[conv.inputs[0]], env[conv.inputs[1]]], items


def eval_graph_node(node: GraphNode, inputs: Sequence[np.ndarray],
                    **kw) -> np.ndarray:
    """eval_graph_node (R/src/graph.cpp:209-225): ONE kernel per fused node."""
    if node.op != "fused":
        return eval_operator(node.op, inputs, node.attrs, **kw)
    conv, (x, w), items = epilogue_of(node, inputs)
    return fused_conv(conv.op, x, w, conv.attrs, items, **kw)
