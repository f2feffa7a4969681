"""TEST INFRASTRUCTURE ONLY: evaluate_graph (R/src/graph.cpp:227-256) over a
fused graph with the oracle restatement (oracle/tec_oracle.c) as the
arithmetic, to check the device executor.

mode "f32": the reference's own numerics (bit-identical to the reference's
evaluate_graph -- pinned by tests/test_graph.py against tests/golden/graphs).
mode "bf16": emulates the executor's bf16 pipeline exactly where it is
deterministic -- conv/matmul operands rounded to bf16, f32 accumulation in
the reference order, every activation rounded to bf16 (graph outputs of
the head -- matmul, pools -- kept in f32, executor.f32_output) -- so the only remaining difference to the device is the
tensor core's accumulation order.
mode "i8": int8 graphs -- the conv itself through the oracle
restatement (i8 x i8 -> i32, bit-identical to the reference), then every
member of the fused node evaluated one by one in member order, as
evaluate_graph does (R/src/graph.cpp:209-222): integer members in int64 with
the i32 range check (DenseTensor::set_i, R/include/tec/tensor.hpp:63-69),
plus the two int8-graph ops the reference registry lacks, restated here from
their definition in paper_1802_04799_b200/csrc/elementwise.cu:
  cast(x, dtype)                   value conversion;
  requantize(x, multiplier, shift) clamp((x*m + 2^(shift-1)) >> shift, -128, 127).
"""
from __future__ import annotations

from typing import Dict

import numpy as np

from oracle.oracle_api import bf16_round, fused_conv, global_avg_pool, max_pool2d
from paper_1802_04799_b200.executor import f32_output


def _epilogue(members, env, prev):
    items = []
    for m in members:
        others = [i for i in m.inputs if i != prev]
        if m.op == "relu":
            items.append(("relu",))
        elif m.op == "scale":
            items.append(("scale", float(m.attrs.get("scale", 1.0))))
        else:
            items.append((m.op, env[others[0]]))
        prev = m.id
    return items


class Overflow(Exception):
    """An i32 range overflow (the reference throws FoldOverflow)."""


def _i32(v):
    if v.size and (v.min() < -2 ** 31 or v.max() > 2 ** 31 - 1):
        raise Overflow()
    return v.astype(np.int32)


def _int_member(m, env):
    """One member of an integer fused node (R/src/ops.cpp semantics)."""
    x = env[m.inputs[0]]
    op = m.op
    if op == "bias_add":
        b = env[m.inputs[1]].astype(np.int64)
        return _i32(x.astype(np.int64) + b.reshape(1, -1, *([1] * (x.ndim - 2))))
    if op in ("add", "mul"):
        y = env[m.inputs[1]].astype(np.int64)
        return _i32(x.astype(np.int64) + y if op == "add" else x.astype(np.int64) * y)
    if op == "relu":
        return np.where(x < 0, 0, x).astype(x.dtype)
    if op == "scale":
        c = float(m.attrs.get("scale", 1.0))
        assert c == int(c)
        return _i32(x.astype(np.int64) * int(c))
    if op == "cast":
        return x.astype({"i8": np.int8, "i32": np.int32, "f32": np.float32}[m.attrs.get("dtype", "i32")])
    if op == "requantize":
        t = x.astype(np.int64) * int(m.attrs.get("multiplier", 1))
        sh = int(m.attrs.get("shift", 0))
        if sh > 0:
            t = (t + (1 << (sh - 1))) >> sh
        return np.clip(t, -128, 127).astype(np.int8)
    raise NotImplementedError(op)


def _evaluate_int(g, feeds, params):
    env = {}
    env.update({k: np.asarray(v) for k, v in feeds.items()})
    env.update({k: np.asarray(v) for k, v in params.items()})
    for n in g.nodes:
        if n.op == "input":
            continue
        ms = n.members if n.op == "fused" else [n]
        local = dict(env)
        for m in ms:
            if m.op in ("conv2d", "depthwise_conv2d"):
                st = tuple(m.attrs.get("strides", (1, 1)))
                pd = tuple(m.attrs.get("padding", (0, 0)))
                local[m.id] = fused_conv(m.op, local[m.inputs[0]], local[m.inputs[1]], st, pd, [])
            elif m.op == "max_pool2d":
                x = local[m.inputs[0]]  # i8 / i32 values are exact in f32
                local[m.id] = max_pool2d(x, tuple(m.attrs.get("kernel", (3, 3))),
                                         tuple(m.attrs.get("strides", (2, 2))),
                                         tuple(m.attrs.get("padding", (1, 1)))).astype(x.dtype)
            else:
                local[m.id] = _int_member(m, local)
        env[n.id] = local[ms[-1].id]
    return {o: env[o] for o in g.outputs}


def evaluate(g, feeds: Dict[str, np.ndarray], params: Dict[str, np.ndarray],
             mode: str = "f32") -> Dict[str, np.ndarray]:
    """g: a fuse_pass'ed ComputeGraph (paper_1802_04799_b200.graph)."""
    if mode == "i8":
        return _evaluate_int(g, feeds, params)
    rnd = bf16_round if mode == "bf16" else (lambda a: a)
    outs = set(g.outputs)
    env = {}
    env.update({k: np.asarray(v, np.float32) for k, v in feeds.items()})
    env.update({k: np.asarray(v, np.float32) for k, v in params.items()})
    cons = g.consumers()
    gap_src = {}
    for n in g.nodes:
        if n.op == "input":
            continue
        if n.op == "fused" or n.op in ("conv2d", "depthwise_conv2d", "matmul"):
            ms = n.members if n.op == "fused" else [n]
            root = ms[0]
            x, w = env[root.inputs[0]], env[root.inputs[1]]
            local = dict(env)
            items = _epilogue(ms[1:], local, root.id)
            if root.op == "matmul":
                xx = x.reshape(x.shape[0], -1, 1, 1)
                ww = np.ascontiguousarray(w.T)[:, :, None, None]
                y = fused_conv("conv2d", rnd(xx), rnd(ww), (1, 1), (0, 0),
                               _reshape_items(items)).reshape(x.shape[0], -1)
            else:
                st = tuple(root.attrs.get("strides", (1, 1)))
                pd = tuple(root.attrs.get("padding", (0, 0)))
                y = fused_conv(root.op, rnd(x), rnd(w), st, pd, items)
        elif n.op in ("bn_fold_weight", "bn_fold_bias"):
            # parameters: kept in f32 (the device folds before packing)
            env[n.id] = _bn_fold(n, [env[i] for i in n.inputs])
            continue
        elif n.op == "const":
            env[n.id] = np.asarray(n.data, np.float32)
            continue
        elif n.op == "max_pool2d":
            y = max_pool2d(env[n.inputs[0]], tuple(n.attrs.get("kernel", (3, 3))),
                           tuple(n.attrs.get("strides", (2, 2))),
                           tuple(n.attrs.get("padding", (1, 1))))
        elif n.op == "global_avg_pool":
            x = env[n.inputs[0]]
            y = global_avg_pool(x).reshape(x.shape[0], x.shape[1], 1, 1)
        elif n.op == "flatten":
            y = env[n.inputs[0]].reshape(n.out_type.shape)
        elif n.op == "sum":
            # only as the reference composition scale(sum(sum(x, 3), 2))
            if int(n.attrs.get("axis", -1)) == 3:
                gap_src[n.id] = n.inputs[0]
                y = None
            else:
                gap_src[n.id] = gap_src[n.inputs[0]]
                y = None
        elif n.op == "scale" and n.inputs[0] in gap_src:
            y = global_avg_pool(env[gap_src[n.inputs[0]]])
        else:
            raise NotImplementedError(n.op)
        if y is not None and (n.id not in outs or not f32_output(n)):
            y = rnd(y)
        env[n.id] = y
    del cons
    return {o: env[o] for o in g.outputs}


def _bn_fold(n, ins):
    """fold_batch_norm's parameter ops, restated: s = gamma / sqrt(var + eps)
    and every product / sum rounded to f32 once."""
    f32 = np.float32
    eps = f32(float(n.attrs.get("eps", 1e-5)))
    if n.op == "bn_fold_weight":
        w, g, v = (np.asarray(a, f32) for a in ins)
        s = (g / np.sqrt(v + eps)).astype(f32)
        return (w * s[:, None, None, None]).astype(f32)
    b, g, beta, mu, v = (np.asarray(a, f32) for a in ins)
    s = (g / np.sqrt(v + eps)).astype(f32)
    return (((b - mu).astype(f32) * s).astype(f32) + beta).astype(f32)


def _reshape_items(items):
    out = []
    for it in items:
        if it[0] in ("add", "mul"):
            out.append((it[0], it[1].reshape(it[1].shape[0], -1, 1, 1)))
        else:
            out.append(it)
    return out
