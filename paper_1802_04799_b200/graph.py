"""Compute-graph API of the reference (R/include/tec/graph.hpp,
R/include/tec/graph_passes.hpp), restated for the sm100 executor.

Reference -> here:
  GraphNode / ComputeGraph          graph.hpp:38-59     -> GraphNode / ComputeGraph
  ComputeGraph::validate            graph.cpp:83-119    -> ComputeGraph.validate
  graph_from_json / graph_to_json   graph.cpp:121-207   -> same names, same JSON
                                                           (base64 const payloads)
  fuse_pass                         graph_passes.cpp:196-283 -> fuse_pass
  plan_memory / check_memory_plan   graph_passes.cpp:285-358 -> plan_memory /
      check_memory_plan (same greedy best-fit; an optional byte-size function
      and alignment let the device executor plan its bf16 arena)
  evaluate_graph                    graph.cpp:227-256   -> executor.DeviceGraph
      (the device executor; there is no host evaluator in the product)

Operator registry (R/src/ops.cpp:196-488): the reference ops keep their
fusion pattern and type rule. The ResNet-18 graph adds three
ops the reference lacks: max_pool2d and global_avg_pool (opaque: they never
join a fused group, so conv -> bias_add -> relu stays one node) and flatten
(injective; [N,C,1,1] -> [N,C], an alias on the device).
"""
from __future__ import annotations

import base64
import copy
import json
from dataclasses import dataclass, field
from typing import Callable, Dict, List, Optional, Sequence, Tuple

import numpy as np

from ._abi import TecError

# ErrorCode numbering of R/include/tec/error.hpp (status = 1 + code).
E_SHAPE, E_IO, E_NOT_ENOUGH_DATA, E_INTERNAL = 2, 20, 19, 21

INJECTIVE, REDUCTION, COMPLEX, OPAQUE = "injective", "reduction", "complex_out_fusable", "opaque"

DTYPE_BYTES = {"f32": 4, "i32": 4, "i8": 1, "bf16": 2}
NP_DTYPE = {"f32": "<f4", "i32": "<i4", "i8": "i1"}


def _fail(code: int, msg: str):
    raise TecError(code, msg)


@dataclass
class TensorType:
    shape: List[int] = field(default_factory=list)
    dtype: str = "f32"

    def validate(self):
        if self.dtype not in DTYPE_BYTES:
            _fail(E_SHAPE, f"unknown dtype {self.dtype}")
        if any(d <= 0 for d in self.shape):
            _fail(E_SHAPE, f"non-positive dim in {self.shape}")

    def rank(self) -> int:
        return len(self.shape)

    def num_elements(self) -> int:
        n = 1
        for d in self.shape:
            n *= d
        return n

    def num_bytes(self, dtype_bytes: Optional[Dict[str, int]] = None) -> int:
        return self.num_elements() * (dtype_bytes or DTYPE_BYTES)[self.dtype]

    def __str__(self):
        return f"{self.dtype}[{','.join(map(str, self.shape))}]"


@dataclass
class GraphNode:
    """graph.hpp:38-47. op is "input", "const", an operator, or "fused"."""
    id: str
    op: str
    inputs: List[str] = field(default_factory=list)
    attrs: Dict[str, object] = field(default_factory=dict)
    out_type: TensorType = field(default_factory=TensorType)
    data: Optional[np.ndarray] = None
    members: List["GraphNode"] = field(default_factory=list)


# ------------------------------------------------------------ type rules
def _ints(attrs, key, dflt):
    v = attrs.get(key, dflt)
    return [int(x) for x in (v if isinstance(v, (list, tuple)) else [v, v])]


def _same_binary(name):
    def f(ins, attrs):
        if len(ins) != 2:
            _fail(E_SHAPE, f"{name} expects 2 inputs")
        if ins[0].shape != ins[1].shape or ins[0].dtype != ins[1].dtype:
            _fail(E_SHAPE, f"{name} operands differ: {ins[0]} vs {ins[1]}")
        return copy.deepcopy(ins[0])
    return f


def _unary(name, float_only):
    def f(ins, attrs):
        if len(ins) != 1:
            _fail(E_SHAPE, f"{name} expects 1 input")
        if float_only and ins[0].dtype != "f32":
            _fail(E_SHAPE, f"{name} requires f32 input")
        return copy.deepcopy(ins[0])
    return f


def _scale(ins, attrs):
    c = float(attrs.get("scale", 1.0))
    if ins[0].dtype != "f32" and c != np.floor(c):
        _fail(E_SHAPE, "integer scale requires an integral factor")
    return copy.deepcopy(ins[0])


def _bias_add(ins, attrs):
    ax = int(attrs.get("axis", 1 if ins[0].rank() >= 2 else 0))
    if ax < 0 or ax >= ins[0].rank():
        _fail(E_SHAPE, "bias_add axis out of range")
    if ins[1].rank() != 1 or ins[1].shape[0] != ins[0].shape[ax]:
        _fail(E_SHAPE, f"bias must be rank-1 matching dim {ax}")
    if ins[0].dtype != ins[1].dtype:
        _fail(E_SHAPE, "bias dtype differs from data")
    return copy.deepcopy(ins[0])


def _sum(ins, attrs):
    ax = int(attrs.get("axis", ins[0].rank() - 1))
    if ax < 0 or ax >= ins[0].rank():
        _fail(E_SHAPE, "sum axis out of range")
    shape = [d for i, d in enumerate(ins[0].shape) if i != ax] or [1]
    return TensorType(shape, ins[0].dtype)


def _matmul(ins, attrs):
    a, b = ins
    if a.rank() != 2 or b.rank() != 2 or a.shape[1] != b.shape[0]:
        _fail(E_SHAPE, f"matmul wants [M,K]x[K,N], got {a} x {b}")
    if a.dtype != b.dtype:
        _fail(E_SHAPE, "matmul operand dtypes differ")
    return TensorType([a.shape[0], b.shape[1]], "i32" if a.dtype == "i8" else a.dtype)


def _conv(depthwise):
    name = "depthwise_conv2d" if depthwise else "conv2d"

    def f(ins, attrs):  # infer_conv, R/src/ops.cpp:163-192
        if len(ins) != 2:
            _fail(E_SHAPE, f"{name} expects 2 inputs")
        dt, wt = ins
        if dt.rank() != 4 or wt.rank() != 4:
            _fail(E_SHAPE, f"{name} wants NCHW data, OIHW weights")
        if dt.dtype != wt.dtype:
            _fail(E_SHAPE, f"{name} operand dtypes differ")
        st, pd = _ints(attrs, "strides", [1, 1]), _ints(attrs, "padding", [0, 0])
        if len(st) != 2 or len(pd) != 2:
            _fail(E_SHAPE, f"{name} strides/padding must be pairs")
        c = dt.shape[1]
        if depthwise:
            if wt.shape[0] != c or wt.shape[1] != 1:
                _fail(E_SHAPE, f"{name} weights must be [C,1,kh,kw] with C={c}")
        elif wt.shape[1] != c:
            _fail(E_SHAPE, f"{name}: weight input-channel dim {wt.shape[1]} != data channels {c}")
        oh = (dt.shape[2] + 2 * pd[0] - wt.shape[2]) // st[0] + 1
        ow = (dt.shape[3] + 2 * pd[1] - wt.shape[3]) // st[1] + 1
        if oh <= 0 or ow <= 0:
            _fail(E_SHAPE, f"{name}: window larger than input")
        return TensorType([dt.shape[0], wt.shape[0], oh, ow], "i32" if dt.dtype == "i8" else dt.dtype)
    return f


def _max_pool2d(ins, attrs):
    x = ins[0]
    if x.rank() != 4:
        _fail(E_SHAPE, "max_pool2d wants NCHW data")
    k = _ints(attrs, "kernel", [3, 3])
    st, pd = _ints(attrs, "strides", [2, 2]), _ints(attrs, "padding", [1, 1])
    if pd[0] >= k[0] or pd[1] >= k[1]:
        _fail(E_SHAPE, "max_pool2d: padding must be smaller than the window")
    oh = (x.shape[2] + 2 * pd[0] - k[0]) // st[0] + 1
    ow = (x.shape[3] + 2 * pd[1] - k[1]) // st[1] + 1
    if oh <= 0 or ow <= 0:
        _fail(E_SHAPE, "max_pool2d: window larger than input")
    return TensorType([x.shape[0], x.shape[1], oh, ow], x.dtype)


def _global_avg_pool(ins, attrs):
    x = ins[0]
    if x.rank() != 4 or x.dtype != "f32":
        _fail(E_SHAPE, "global_avg_pool wants f32 NCHW data")
    return TensorType([x.shape[0], x.shape[1], 1, 1], x.dtype)


def _flatten(ins, attrs):
    x = ins[0]
    if x.rank() < 2:
        _fail(E_SHAPE, "flatten wants rank >= 2")
    return TensorType([x.shape[0], int(np.prod(x.shape[1:]))], x.dtype)


def _layout_transform(ins, attrs):
    src, dst = attrs.get("src_layout", "row_major"), attrs.get("dst_layout", "row_major")
    x = ins[0]
    if src == "row_major" and dst == "tiled4x4":
        if x.rank() != 2:
            _fail(E_SHAPE, "tiled4x4 layout applies to rank-2 tensors")
        return TensorType([(x.shape[0] + 3) // 4, (x.shape[1] + 3) // 4, 4, 4], x.dtype)
    if src == "tiled4x4" and dst == "row_major":
        h, w = int(attrs.get("height", 0)), int(attrs.get("width", 0))
        if x.rank() != 4 or h <= 0 or w <= 0:
            _fail(E_SHAPE, "tiled4x4 -> row_major needs a rank-4 source and height/width")
        return TensorType([h, w], x.dtype)
    if {src, dst} == {"row_major", "nhwc"}:
        # a physical relayout of a rank-4 activation (NCHW <-> NHWC); the
        # type keeps the LOGICAL NCHW shape (logical shapes are
        # NCHW, kernels run NHWC)
        if x.rank() != 4:
            _fail(E_SHAPE, "nhwc layout applies to rank-4 tensors")
        return copy.deepcopy(x)
    if src == dst:
        return copy.deepcopy(x)
    _fail(E_SHAPE, f"unsupported layout pair {src} -> {dst}")


def _cast(ins, attrs):
    """cast(x, dtype): i8 -> i32 | f32, i32 -> f32 (and the identity). Not in
    the reference registry: the int8 graph's shortcut operand (elementwise.cu)."""
    to = attrs.get("dtype", "i32")
    frm = ins[0].dtype
    if (frm, to) not in (("i8", "i32"), ("i8", "f32"), ("i32", "f32"), ("i8", "i8"),
                         ("i32", "i32"), ("f32", "f32")):
        _fail(E_SHAPE, f"cast {frm} -> {to} is not supported")
    return TensorType(list(ins[0].shape), to)


def _requantize(ins, attrs):
    """requantize(x: i32) -> i8 = clamp((x * multiplier + 2^(shift-1)) >> shift,
    -128, 127). Not in the reference registry: the int8 graph's per-layer
    output rescale (elementwise.cu states the arithmetic)."""
    if ins[0].dtype != "i32":
        _fail(E_SHAPE, "requantize wants i32 data")
    m, sh = attrs.get("multiplier", 1), attrs.get("shift", 0)
    if int(m) != m or int(sh) != sh or not (1 <= int(m) < 2 ** 31) or not (0 <= int(sh) <= 62):
        _fail(E_SHAPE, "requantize needs an integer 1 <= multiplier < 2^31 and 0 <= shift <= 62")
    return TensorType(list(ins[0].shape), "i8")


def _per_channel(name, n_vec, data_first=True):
    """Ops over a rank-4 x (NCHW, channel axis 1) and n_vec [C] vectors."""
    def f(ins, attrs):
        x = ins[0]
        if x.rank() != 4 and data_first:
            _fail(E_SHAPE, f"{name} wants NCHW data")
        c = x.shape[0] if not data_first else x.shape[1]
        for v in ins[1:1 + n_vec]:
            if v.rank() != 1 or v.shape[0] != c or v.dtype != "f32":
                _fail(E_SHAPE, f"{name}: per-channel operands must be f32 [{c}]")
        if x.dtype != "f32":
            _fail(E_SHAPE, f"{name} wants f32 data")
        if float(attrs.get("eps", 1e-5)) < 0:
            _fail(E_SHAPE, f"{name}: eps must be >= 0")
        return copy.deepcopy(x)
    return f


# name -> (pattern, arity, infer)
OPS: Dict[str, Tuple[str, int, Callable]] = {
    "add": (INJECTIVE, 2, _same_binary("add")),
    "mul": (INJECTIVE, 2, _same_binary("mul")),
    "exp": (INJECTIVE, 1, _unary("exp", True)),
    "sqrt": (INJECTIVE, 1, _unary("sqrt", True)),
    "relu": (INJECTIVE, 1, _unary("relu", False)),
    "scale": (INJECTIVE, 1, _scale),
    "bias_add": (INJECTIVE, 2, _bias_add),
    "sum": (REDUCTION, 1, _sum),
    "matmul": (COMPLEX, 2, _matmul),
    "conv2d": (COMPLEX, 2, _conv(False)),
    "depthwise_conv2d": (COMPLEX, 2, _conv(True)),
    "sort": (OPAQUE, 1, _unary("sort", False)),
    "layout_transform": (INJECTIVE, 1, _layout_transform),
    # ResNet-18 graph ops (not in the reference registry)
    "max_pool2d": (OPAQUE, 1, _max_pool2d),
    "global_avg_pool": (OPAQUE, 1, _global_avg_pool),
    "flatten": (INJECTIVE, 1, _flatten),
    # int8 graph ops (not in the reference registry)
    "cast": (INJECTIVE, 1, _cast),
    "requantize": (INJECTIVE, 1, _requantize),
    # inference batch norm and its folded form (fold_batch_norm; not in the
    # reference registry): s = gamma / sqrt(var + eps) per channel, every
    # operation rounded to f32 separately (no FMA)
    #   batch_norm(x, gamma, beta, mean, var) = (x - mean) * s + beta
    #   bn_fold_weight(w[K,C,R,S], gamma, var) = w * s[k]
    #   bn_fold_bias(b, gamma, beta, mean, var) = (b - mean) * s + beta
    "batch_norm": (INJECTIVE, 5, _per_channel("batch_norm", 4)),
    "bn_fold_weight": (INJECTIVE, 3, _per_channel("bn_fold_weight", 2, data_first=False)),
    "bn_fold_bias": (INJECTIVE, 5, _per_channel("bn_fold_bias", 4, data_first=False)),
}


def op_def(name: str):
    if name not in OPS:
        _fail(E_SHAPE, f"unknown operator '{name}'")
    return OPS[name]


def _infer_node(n: GraphNode, in_types: List[TensorType]) -> TensorType:
    """graph.cpp:48-81."""
    if n.op in ("input", "const"):
        n.out_type.validate()
        return n.out_type
    if n.op == "fused":
        if not n.members:
            _fail(E_SHAPE, f"fused node {n.id} has no members")
        env = dict(zip(n.inputs, in_types))
        last = None
        for m in n.members:
            mt = []
            for i in m.inputs:
                if i not in env:
                    _fail(E_SHAPE, f"fused member {m.id} reads unknown tensor {i}")
                mt.append(env[i])
            last = op_def(m.op)[2](mt, m.attrs)
            env[m.id] = last
        return last
    pat, arity, infer = op_def(n.op)
    if len(n.inputs) != arity:
        _fail(E_SHAPE, f"{n.op} node {n.id} has {len(n.inputs)} inputs, expected {arity}")
    return infer(in_types, n.attrs)


@dataclass
class ComputeGraph:
    nodes: List[GraphNode] = field(default_factory=list)  # topologically ordered
    outputs: List[str] = field(default_factory=list)

    def find(self, nid: str) -> Optional[GraphNode]:
        for n in self.nodes:
            if n.id == nid:
                return n
        return None

    def node(self, nid: str) -> GraphNode:
        n = self.find(nid)
        if n is None:
            _fail(E_SHAPE, f"graph has no node '{nid}'")
        return n

    def consumers(self) -> Dict[str, List[str]]:
        out: Dict[str, List[str]] = {}
        for n in self.nodes:
            for i in n.inputs:
                out.setdefault(i, []).append(n.id)
        return out

    def validate(self) -> None:
        """graph.cpp:83-119: unique ids, topological references, outputs,
        re-inferred types checked against declared ones."""
        types: Dict[str, TensorType] = {}
        for n in self.nodes:
            if n.id in types:
                _fail(E_SHAPE, f"duplicate node id '{n.id}'")
            ins = []
            for i in n.inputs:
                if i not in types:
                    _fail(E_SHAPE, f"node {n.id} references '{i}' before its definition")
                ins.append(types[i])
            t = _infer_node(n, ins)
            if n.out_type.shape and (n.out_type.shape != t.shape or n.out_type.dtype != t.dtype):
                _fail(E_SHAPE, f"node {n.id} declares {n.out_type} but computes {t}")
            n.out_type = copy.deepcopy(t)
            if n.op == "const" and n.data is not None and \
                    list(n.data.shape) != t.shape:
                _fail(E_SHAPE, f"const {n.id} payload shape {list(n.data.shape)}, declared {t}")
            types[n.id] = t
        if not self.outputs:
            _fail(E_SHAPE, "graph declares no outputs")
        for o in self.outputs:
            if o not in types:
                _fail(E_SHAPE, f"output '{o}' is not a node")


# ------------------------------------------------------------- JSON I/O
def _node_from_json(j: dict) -> GraphNode:
    n = GraphNode(id=j["id"], op=j["op"], inputs=list(j.get("inputs", [])),
                  attrs=dict(j.get("attrs", {})))
    if "shape" in j:
        n.out_type = TensorType([int(d) for d in j["shape"]], j.get("dtype", "f32"))
    elif n.op in ("input", "const"):
        _fail(E_IO, f"node {n.id} needs an explicit shape")
    if j.get("data"):
        raw = base64.b64decode(j["data"])
        n.data = np.frombuffer(raw, dtype=NP_DTYPE[n.out_type.dtype]).reshape(n.out_type.shape).copy()
    for m in j.get("members", []):
        n.members.append(_node_from_json(m))
    return n


def _node_to_json(n: GraphNode) -> dict:
    j = {"id": n.id, "op": n.op, "inputs": list(n.inputs)}
    if n.attrs:
        j["attrs"] = {k: (list(v) if isinstance(v, tuple) else v) for k, v in n.attrs.items()}
    if n.out_type.shape:
        j["shape"] = list(n.out_type.shape)
        j["dtype"] = n.out_type.dtype
    if n.data is not None:
        j["data"] = base64.b64encode(
            np.ascontiguousarray(n.data, dtype=NP_DTYPE[n.out_type.dtype]).tobytes()).decode()
    if n.members:
        j["members"] = [_node_to_json(m) for m in n.members]
    return j


def graph_from_json(j) -> ComputeGraph:
    """graph.cpp:189-198 (accepts a dict or JSON text)."""
    if isinstance(j, (str, bytes)):
        try:
            j = json.loads(j)
        except ValueError:
            _fail(E_IO, "malformed graph JSON")
    if not isinstance(j.get("nodes"), list):
        _fail(E_IO, "graph JSON needs a 'nodes' array")
    g = ComputeGraph([_node_from_json(n) for n in j["nodes"]], list(j.get("outputs", [])))
    g.validate()
    return g


def graph_to_json(g: ComputeGraph) -> dict:
    return {"nodes": [_node_to_json(n) for n in g.nodes], "outputs": list(g.outputs)}


# ------------------------------------------------------------- fuse_pass
def fuse_pass(g: ComputeGraph) -> ComputeGraph:
    """graph_passes.cpp:196-283: reverse-topological greedy grouping with
    union-find; a producer joins the single group consuming all its uses
    when injective -> {injective, reduction} or complex -> injective (the
    group's anchor becomes complex). Outputs and opaque ops never move."""
    n = len(g.nodes)
    index_of = {nd.id: i for i, nd in enumerate(g.nodes)}
    outputs = set(g.outputs)

    def pattern_of(nd):
        if nd.op in ("input", "const", "fused"):
            return None
        return op_def(nd.op)[0]

    parent = list(range(n))

    def find(x):
        while parent[x] != x:
            parent[x] = parent[parent[x]]
            x = parent[x]
        return x

    anchor = [pattern_of(nd) or OPAQUE for nd in g.nodes]
    cons = g.consumers()
    for i in range(n - 1, -1, -1):
        u = g.nodes[i]
        pu = pattern_of(u)
        if pu is None or pu == OPAQUE or u.id in outputs:
            continue
        cids = cons.get(u.id, [])
        if not cids:
            continue
        groups = {find(index_of[c]) for c in cids}
        if len(groups) != 1:
            continue
        group = groups.pop()
        if group == find(i):
            continue
        ga = anchor[group]
        nxt = ga
        if pu == INJECTIVE and ga in (INJECTIVE, REDUCTION):
            merge = True
        elif pu == COMPLEX and ga == INJECTIVE:
            merge, nxt = True, COMPLEX
        else:
            merge = False
        if not merge:
            continue
        parent[find(i)] = find(group)
        anchor[find(i)] = nxt

    groups: Dict[int, List[int]] = {}
    for i in range(n):
        groups.setdefault(find(i), []).append(i)
    out = ComputeGraph([], list(g.outputs))
    for i in range(n):
        members = groups[find(i)]
        if members[-1] != i:
            continue
        if len(members) == 1:
            out.nodes.append(copy.deepcopy(g.nodes[i]))
            continue
        internal = {g.nodes[m].id for m in members}
        fused = GraphNode(id=g.nodes[i].id, op="fused", out_type=copy.deepcopy(g.nodes[i].out_type))
        for m in members:
            fused.members.append(copy.deepcopy(g.nodes[m]))
            for inp in g.nodes[m].inputs:
                if inp not in internal and inp not in fused.inputs:
                    fused.inputs.append(inp)
        out.nodes.append(fused)
    out.validate()
    return out


# ----------------------------------------------------------- plan_memory
@dataclass
class MemoryPlan:
    slot_of: Dict[str, int] = field(default_factory=dict)
    slot_bytes: List[int] = field(default_factory=list)
    total_bytes: int = 0
    naive_bytes: int = 0
    slot_offset: List[int] = field(default_factory=list)  # arena offsets (device plan)


def plan_memory(g: ComputeGraph, nbytes: Optional[Callable[[GraphNode], int]] = None,
                align: int = 1) -> MemoryPlan:
    """graph_passes.cpp:285-329: greedy best-fit slot reuse in execution
    order; a producer stays live through its last consumer (no in-place
    update); inputs, consts and graph outputs own their storage.
    `nbytes` (default: the reference's num_bytes) and `align` let the device
    executor plan its own arena with the same algorithm."""
    outputs = set(g.outputs)
    size = nbytes or (lambda nd: nd.out_type.num_bytes())
    remaining: Dict[str, int] = {}
    for nd in g.nodes:
        for i in nd.inputs:
            remaining[i] = remaining.get(i, 0) + 1
    plan = MemoryPlan()
    free: List[Tuple[int, int]] = []  # sorted (bytes, slot)
    for nd in g.nodes:
        if nd.op in ("input", "const"):
            continue
        if nd.id not in outputs:
            need = size(nd)
            need = (need + align - 1) // align * align
            plan.naive_bytes += need
            pick = next((k for k, (b, s) in enumerate(free) if b >= need), None)
            if pick is not None:
                slot = free.pop(pick)[1]
            else:
                slot = len(plan.slot_bytes)
                plan.slot_bytes.append(need)
            plan.slot_of[nd.id] = slot
        seen = set()
        for i in nd.inputs:
            remaining[i] -= 1
            if remaining[i] == 0 and i in plan.slot_of and i not in seen:
                s = plan.slot_of[i]
                free.append((plan.slot_bytes[s], s))
                free.sort()
                seen.add(i)
    off = 0
    for b in plan.slot_bytes:
        plan.slot_offset.append(off)
        off += b
    plan.total_bytes = off
    return plan


def check_memory_plan(g: ComputeGraph, plan: MemoryPlan,
                      nbytes: Optional[Callable[[GraphNode], int]] = None) -> None:
    """graph_passes.cpp:331-358: replay; no operand clobbered before it is
    read, no slot too small, no node writing its own operand's slot."""
    size = nbytes or (lambda nd: nd.out_type.num_bytes())
    content: Dict[int, str] = {}
    for nd in g.nodes:
        if nd.op in ("input", "const"):
            continue
        for i in nd.inputs:
            if i not in plan.slot_of:
                continue
            if content.get(plan.slot_of[i]) != i:
                _fail(E_INTERNAL, f"memory plan clobbers '{i}' before node '{nd.id}' reads it")
        if nd.id in plan.slot_of:
            s = plan.slot_of[nd.id]
            if plan.slot_bytes[s] < size(nd):
                _fail(E_INTERNAL, f"slot too small for '{nd.id}'")
            for i in nd.inputs:
                if plan.slot_of.get(i) == s:
                    _fail(E_INTERNAL, f"node '{nd.id}' would overwrite its own operand")
            content[s] = nd.id


# ------------------------------------------------------- tensor artifacts
def save_tensor(directory: str, name: str, arr: np.ndarray, dtype: Optional[str] = None) -> None:
    """save_tensor (R/src/io.cpp:111-119): <name>.json manifest {name, shape,
    dtype} + <name>.bin raw little-endian payload (i8 one byte/element)."""
    import os
    dtype = dtype or {np.dtype(np.float32): "f32", np.dtype(np.int32): "i32",
                      np.dtype(np.int8): "i8"}.get(arr.dtype)
    if dtype not in NP_DTYPE:
        _fail(E_IO, f"cannot save dtype {arr.dtype}")
    os.makedirs(directory, exist_ok=True)
    with open(os.path.join(directory, name + ".json"), "w") as f:
        json.dump({"name": name, "shape": [int(d) for d in arr.shape], "dtype": dtype}, f, indent=2)
        f.write("\n")
    with open(os.path.join(directory, name + ".bin"), "wb") as f:
        f.write(np.ascontiguousarray(arr, dtype=NP_DTYPE[dtype]).tobytes())


def load_tensor(directory: str, name: str) -> np.ndarray:
    """load_tensor (R/src/io.cpp:121-127); IOError on a missing or
    malformed manifest / a payload of the wrong size."""
    import os
    try:
        with open(os.path.join(directory, name + ".json")) as f:
            man = json.load(f)
        with open(os.path.join(directory, name + ".bin"), "rb") as f:
            raw = f.read()
    except (OSError, ValueError) as e:
        _fail(E_IO, f"cannot load tensor '{name}' from {directory}: {e}")
    dt = man.get("dtype", "f32")
    if dt not in NP_DTYPE:
        _fail(E_IO, f"unknown dtype '{dt}' in {name}.json")
    shape = [int(d) for d in man["shape"]]
    a = np.frombuffer(raw, dtype=NP_DTYPE[dt])
    if a.size != int(np.prod(shape)):
        _fail(E_IO, f"{name}.bin holds {a.size} elements, manifest says {shape}")
    return a.reshape(shape).astype({"f32": np.float32, "i32": np.int32, "i8": np.int8}[dt])


# ------------------------------------------------------- fold_constants
E_FOLD_OVERFLOW = 3
_I32 = (np.iinfo(np.int32).min, np.iinfo(np.int32).max)


def _check_i32(v: np.ndarray, what: str) -> np.ndarray:
    if v.size and (v.min() < _I32[0] or v.max() > _I32[1]):
        _fail(E_FOLD_OVERFLOW, f"value out of range for i32 folding {what}")
    return v


def _libm_expf(x: np.ndarray) -> np.ndarray:
    """std::exp on float (the reference's kExp, R/src/expr.cpp:155-156) via
    the C library itself, so folded results match it bit for bit."""
    import ctypes
    import ctypes.util
    lib = ctypes.CDLL(ctypes.util.find_library("m") or "libm.so.6")
    lib.expf.restype = ctypes.c_float
    lib.expf.argtypes = [ctypes.c_float]
    flat = np.ascontiguousarray(x, dtype=np.float32).ravel()
    return np.array([lib.expf(float(v)) for v in flat], dtype=np.float32).reshape(x.shape)


def bn_scale(gamma: np.ndarray, var: np.ndarray, eps: float) -> np.ndarray:
    """s = gamma / sqrt(var + eps), each step rounded to f32."""
    g, v = np.asarray(gamma, np.float32), np.asarray(var, np.float32)
    return (g / np.sqrt(v + np.float32(eps))).astype(np.float32)


def bn_eval(op: str, ins: List[np.ndarray], eps: float) -> np.ndarray:
    """The batch-norm ops' f32 semantics (see OPS)."""
    if op == "bn_fold_weight":
        w, g, v = ins
        s = bn_scale(g, v, eps)
        return (np.asarray(w, np.float32) * s.reshape(-1, *([1] * (w.ndim - 1)))).astype(np.float32)
    x, g, b, m, v = ins
    s = bn_scale(g, v, eps)
    shp = (1, -1, 1, 1) if op == "batch_norm" else (-1,)
    x = np.asarray(x, np.float32)
    y = (x - np.asarray(m, np.float32).reshape(shp)).astype(np.float32)
    y = (y * s.reshape(shp)).astype(np.float32)
    return (y + np.asarray(b, np.float32).reshape(shp)).astype(np.float32)


def _fold_eval(n: GraphNode, ins: List[np.ndarray]) -> np.ndarray:
    """Compile-time evaluation of one node whose inputs are all constants.
    Elementwise / reduction / layout ops follow the reference's host
    semantics (float ops rounded per operation, integer ops in 64 bits with
    the i32 range check, R/src/expr.cpp:95-167); conv / matmul / pool nodes
    run through the device executor's bit-exact f32 path."""
    op = n.op
    isf = ins[0].dtype == np.float32 if ins else True
    if op in ("add", "mul"):
        a, b = ins
        if isf:
            return (a + b) if op == "add" else (a * b)
        v = (a.astype(np.int64) + b) if op == "add" else (a.astype(np.int64) * b)
        return _check_i32(v, n.id).astype(a.dtype if a.dtype == np.int32 else np.int32)
    if op == "relu":
        x = ins[0]
        return np.where(x < 0, np.zeros_like(x), x)
    if op in ("batch_norm", "bn_fold_weight", "bn_fold_bias"):
        return bn_eval(op, ins, float(n.attrs.get("eps", 1e-5)))
    if op == "cast":
        return ins[0].astype({"i8": np.int8, "i32": np.int32, "f32": np.float32}[n.attrs.get("dtype", "i32")])
    if op == "requantize":
        m, sh = int(n.attrs.get("multiplier", 1)), int(n.attrs.get("shift", 0))
        t = ins[0].astype(np.int64) * m
        if sh > 0:
            t = (t + (1 << (sh - 1))) >> sh
        return np.clip(t, -128, 127).astype(np.int8)
    if op == "exp":
        return _libm_expf(ins[0])
    if op == "sqrt":
        return np.sqrt(ins[0].astype(np.float32))
    if op == "scale":
        c = float(n.attrs.get("scale", 1.0))
        if isf:
            return ins[0] * np.float32(c)
        return _check_i32(ins[0].astype(np.int64) * int(c), n.id).astype(np.int32)
    if op == "bias_add":
        x, b = ins
        ax = int(n.attrs.get("axis", 1 if x.ndim >= 2 else 0))
        shape = [1] * x.ndim
        shape[ax] = -1
        if isf:
            return x + b.reshape(shape)
        return _check_i32(x.astype(np.int64) + b.reshape(shape), n.id).astype(np.int32)
    if op == "sum":
        x = ins[0]
        ax = int(n.attrs.get("axis", x.ndim - 1))
        if isf:  # sequential accumulation from 0, rounded per add
            acc = np.zeros(np.delete(x.shape, ax), np.float32)
            for i in range(x.shape[ax]):
                acc = acc + np.take(x, i, axis=ax)
            out = acc
        else:
            out = _check_i32(x.astype(np.int64).sum(axis=ax), n.id).astype(np.int32)
        return out.reshape(n.out_type.shape)
    if op == "layout_transform":
        x = ins[0]
        src, dst = n.attrs.get("src_layout", "row_major"), n.attrs.get("dst_layout", "row_major")
        if src == dst:
            return x.copy()
        if src == "row_major":
            h, w = x.shape
            out = np.zeros(n.out_type.shape, x.dtype)
            for i in range(h):
                for j in range(w):
                    out[i // 4, j // 4, i % 4, j % 4] = x[i, j]
            return out
        h, w = n.out_type.shape
        return np.array([[x[i // 4, j // 4, i % 4, j % 4] for j in range(w)] for i in range(h)],
                        dtype=x.dtype)
    # conv / matmul / fused / pools: one-node graph on the device (f32 exact)
    from .executor import DeviceGraph
    names = [f"__c{i}" for i in range(len(ins))]
    nodes = [GraphNode(nm, "input", out_type=TensorType(list(a.shape),
                                                        {np.dtype(np.float32): "f32",
                                                         np.dtype(np.int32): "i32",
                                                         np.dtype(np.int8): "i8"}[a.dtype]))
             for nm, a in zip(names, ins)]
    node = copy.deepcopy(n)
    node.inputs = names
    if node.op == "fused":
        ren = dict(zip(n.inputs, names))
        for m in node.members:
            m.inputs = [ren.get(i, i) for i in m.inputs]
    g = ComputeGraph(nodes + [node], [node.id])
    g.validate()
    dg = DeviceGraph(g, compute="f32")
    dg.bind_params({k: v for k, v in zip(names, ins) if k in dg.param_names})
    return dg.run({k: v for k, v in zip(names, ins) if k in dg.feed_names})[node.id]


def _strip_dead(g: ComputeGraph) -> ComputeGraph:
    live = set(g.outputs)
    for n in reversed(g.nodes):
        if n.id in live:
            live.update(n.inputs)
    return ComputeGraph([n for n in g.nodes if n.id in live], list(g.outputs))


def fold_constants(g: ComputeGraph) -> ComputeGraph:
    """graph_passes.cpp:41-73: nodes whose inputs are all constants are
    evaluated and replaced by const nodes; unreferenced nodes are dropped.
    Folding through a const without payload is NotEnoughData; integer
    overflow is FoldOverflow."""
    out = ComputeGraph([], list(g.outputs))
    consts: Dict[str, GraphNode] = {}
    for n in g.nodes:
        copy_n = copy.deepcopy(n)
        foldable = n.op not in ("input", "const") and n.inputs and \
            all(i in consts for i in n.inputs)
        if foldable:
            ins = []
            for i in n.inputs:
                c = consts[i]
                if c.data is None:
                    _fail(E_NOT_ENOUGH_DATA, f"cannot fold through const '{i}' with no data")
                ins.append(c.data)
            v = np.ascontiguousarray(_fold_eval(n, ins))
            copy_n = GraphNode(n.id, "const", out_type=TensorType(list(v.shape), n.out_type.dtype),
                               data=v)
        out.nodes.append(copy_n)
        if copy_n.op == "const":
            consts[copy_n.id] = copy_n
    out = _strip_dead(out)
    out.validate()
    return out


# -------------------------------------------------------- apply_layouts
_LAYOUT_ELEMWISE = ("add", "mul", "exp", "sqrt", "relu", "scale")


# Ops that run on NHWC activations on the device (the "nhwc" preference):
# the conv / pool kernels and the per-element ops around them.
_NHWC_OPS = ("conv2d", "depthwise_conv2d", "max_pool2d", "global_avg_pool", "bias_add", "add",
             "mul", "relu", "scale", "cast", "requantize", "fused")
_SUFFIX = {"tiled4x4": "#t", "nhwc": "#h"}


def apply_layouts(g: ComputeGraph, prefs: Dict[str, str]) -> ComputeGraph:
    """graph_passes.cpp:84-178: realise per-node layout preferences by
    inserting layout_transform nodes; graph outputs stay row-major by
    contract. Preferences: "row_major", "tiled4x4" (the reference's: rank-2
    elementwise ops) and "nhwc" (the B200 pass, see nhwc_layout_pass:
    rank-4 device ops). A node with a non-row-major preference runs as
    "<id>#t" / "<id>#h"; a transform of producer X into a layout is
    "X#t" / "X#h", back to row-major "X#r"; an output's final transform
    takes over the output's id."""
    for nid, pf in prefs.items():
        if pf not in ("row_major", "tiled4x4", "nhwc"):
            _fail(E_SHAPE, f"unknown layout preference '{pf}'")
        if pf == "row_major":
            continue
        n = g.node(nid)
        if pf == "tiled4x4":
            if n.op not in _LAYOUT_ELEMWISE:
                _fail(E_SHAPE, f"tiled4x4 preference on '{nid}' ({n.op}): only elementwise ops can carry it")
            if n.out_type.rank() != 2:
                _fail(E_SHAPE, f"tiled4x4 preference on '{nid}' needs a rank-2 tensor")
        else:
            if n.op not in _NHWC_OPS:
                _fail(E_SHAPE, f"nhwc preference on '{nid}' ({n.op}): not a device NHWC op")
            if n.out_type.rank() != 4:
                _fail(E_SHAPE, f"nhwc preference on '{nid}' needs a rank-4 tensor")
    pref_of = lambda i: prefs.get(i, "row_major")  # noqa: E731
    out = ComputeGraph([], list(g.outputs))
    rm_type = {n.id: n.out_type for n in g.nodes}
    realized: Dict[Tuple[str, str], str] = {}
    made_in: Dict[str, str] = {}  # node id -> the layout it was computed in
    for n in g.nodes:
        pf = pref_of(n.id)
        run_id = n.id + _SUFFIX.get(pf, "")
        c = copy.deepcopy(n)
        c.id = run_id
        c.out_type = TensorType()
        if n.op in ("input", "const"):
            c.out_type = copy.deepcopy(n.out_type)
            out.nodes.append(c)
            realized[(n.id, "row_major")] = n.id
            made_in[n.id] = "row_major"
            continue
        new_inputs = []
        # weights (operand 1 of a conv, also inside a fused node) and
        # per-channel vectors stay row-major: they are parameters, packed
        # once by tec_weight_pretransform
        weights = {m.inputs[1] for m in (n.members or [n])
                   if m.op in ("conv2d", "depthwise_conv2d") and len(m.inputs) > 1}
        for pos, i in enumerate(c.inputs):
            want = pf if rm_type[i].rank() == 4 or pf == "tiled4x4" else "row_major"
            if pf == "nhwc" and i in weights:
                want = "row_major"
            key = (i, want)
            if key in realized:
                new_inputs.append(realized[key])
                continue
            rt = rm_type[i]
            src_l = made_in[i]
            if want != "row_major":
                tr = GraphNode(i + _SUFFIX[want], "layout_transform", [realized[(i, src_l)]],
                               {"src_layout": "row_major", "dst_layout": want})
                if (i, "row_major") not in realized:
                    _fail(E_SHAPE, f"no row-major form of '{i}' to transform")
                tr.inputs = [realized[(i, "row_major")]]
            else:
                attrs = {"src_layout": src_l, "dst_layout": "row_major"}
                if src_l == "tiled4x4":
                    attrs.update({"height": rt.shape[0], "width": rt.shape[1]})
                tr = GraphNode(i + "#r", "layout_transform", [realized[(i, src_l)]], attrs)
            realized[key] = tr.id
            new_inputs.append(tr.id)
            out.nodes.append(tr)
        c.inputs = new_inputs
        if c.members:  # a fused node reads its operands by the outer ids
            ren = dict(zip(n.inputs, new_inputs))
            for m in c.members:
                m.inputs = [ren.get(x, x) for x in m.inputs]
        out.nodes.append(c)
        realized[(n.id, pf)] = run_id
        made_in[n.id] = pf
    for o in out.outputs:
        if (o, "row_major") in realized:
            continue
        rt = rm_type[o]
        src_l = made_in[o]
        attrs = {"src_layout": src_l, "dst_layout": "row_major"}
        if src_l == "tiled4x4":
            attrs.update({"height": rt.shape[0], "width": rt.shape[1]})
        out.nodes.append(GraphNode(o, "layout_transform", [realized[(o, src_l)]], attrs))
        realized[(o, "row_major")] = o
    out = _strip_dead(out)
    out.validate()
    return out


def nhwc_layout_pass(g: ComputeGraph) -> ComputeGraph:
    """The B200 layout pass: every rank-4 device op runs NHWC
    (apply_layouts with an "nhwc" preference on each), so layout_transform
    nodes appear exactly where an activation crosses between the reference
    NCHW layout and the kernels' NHWC one -- graph inputs feeding the
    network, rank-4 graph outputs, and row-major consumers (the matmul
    head). The executor realises each transform inside a neighbouring
    launch (the conv's input pack, the output unpack) or as a no-op when
    the two layouts coincide ([N, C, 1, 1])."""
    prefs = {n.id: "nhwc" for n in g.nodes
             if n.op in _NHWC_OPS and n.out_type.rank() == 4
             and not (n.op == "fused" and n.members[0].op == "matmul")}
    return apply_layouts(g, prefs)


def fold_batch_norm(g: ComputeGraph) -> ComputeGraph:
    """BN folding: conv2d(x, W) [-> bias_add(., B)] ->
    batch_norm(., gamma, beta, mean, var) becomes
    conv2d(x, bn_fold_weight(W, gamma, var)) -> bias_add(., bn_fold_bias(B,
    gamma, beta, mean, var)) (B = zeros when there was no bias_add). The
    fold nodes depend on parameters only: fold_constants evaluates them at
    compile time when they are consts, and the device executor runs them
    inside tec_weight_pretransform_bn when they are bound parameters."""
    cons = g.consumers()
    outs = set(g.outputs)
    by_id = {n.id: n for n in g.nodes}
    rewrite: Dict[str, Tuple[str, Optional[str]]] = {}  # bn id -> (conv id, bias_add id)
    for n in g.nodes:
        if n.op != "batch_norm":
            continue
        src = by_id[n.inputs[0]]
        bias = None
        if src.op == "bias_add" and len(cons.get(src.id, [])) == 1 and src.id not in outs:
            bias, src = src, by_id[src.inputs[0]]
        if src.op != "conv2d" or len(cons.get(src.id, [])) != 1 or src.id in outs:
            continue
        if by_id[src.inputs[1]].op not in ("input", "const"):
            continue
        rewrite[n.id] = (src.id, bias.id if bias else None)
    if not rewrite:
        return copy.deepcopy(g)
    conv_of = {c: bn for bn, (c, _) in rewrite.items()}
    bias_of = {b: bn for bn, (_, b) in rewrite.items() if b}
    out = ComputeGraph([], list(g.outputs))
    for bn_node in g.nodes:
        # everything is emitted where the batch_norm was: its parameters
        # and the conv's operands all precede it
        if bn_node.id not in rewrite:
            if bn_node.id not in conv_of and bn_node.id not in bias_of:
                out.nodes.append(copy.deepcopy(bn_node))
            continue
        n = by_id[rewrite[bn_node.id][0]]
        if True:
            bn = bn_node
            eps = {"eps": float(bn.attrs.get("eps", 1e-5))}
            _, gm, bt, mu, vr = bn.inputs
            wf = GraphNode(n.id + "#bnw", "bn_fold_weight", [n.inputs[1], gm, vr], dict(eps))
            out.nodes.append(wf)
            b_in = by_id[rewrite[bn.id][1]].inputs[1] if rewrite[bn.id][1] else None
            if b_in is None:
                z = GraphNode(n.id + "#b0", "const",
                              out_type=TensorType([by_id[n.inputs[1]].out_type.shape[0]], "f32"))
                z.data = np.zeros(z.out_type.shape, np.float32)
                out.nodes.append(z)
                b_in = z.id
            # the fold nodes precede the conv, so fuse_pass groups the conv
            # with its epilogue only (a parameter computation never joins it)
            bf = GraphNode(n.id + "#bnb", "bn_fold_bias", [b_in, gm, bt, mu, vr], dict(eps))
            out.nodes.append(bf)
            c = copy.deepcopy(n)
            c.inputs = [n.inputs[0], wf.id]
            out.nodes.append(c)
            # the bias_add takes over the batch_norm's id (its consumers)
            out.nodes.append(GraphNode(bn.id, "bias_add", [c.id, bf.id]))
    out.validate()
    return out
