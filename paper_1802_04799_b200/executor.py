"""Device graph executor: evaluate_graph (R/src/graph.cpp:227-256) for
target sm100 -- SURVEY 8f.1.

The reference runs a fused node member by member with every intermediate in
a std::map (R/src/graph.cpp:209-225). Here a graph is compiled ONCE into a
list of kernel launches on device buffers:

  * fuse_pass (graph.py, R/src/graph_passes.cpp:196-283) groups
    [conv2d|depthwise_conv2d|matmul, scale?, bias_add?, add?, mul?, relu?]
    into one node -> ONE fused kernel (tec_conv2d_fused / tec_depthwise_fused;
    matmul runs as a 1x1 conv over a 1x1 image);
  * max_pool2d / global_avg_pool -> tec_max_pool2d / tec_global_avg_pool;
    the reference composition scale(sum(sum(x, 3), 2)) is recognised as a
    global average pool; flatten of an [N,C,1,1] tensor is an alias;
  * intermediates live in ONE arena laid out by plan_memory
    (R/src/graph_passes.cpp:285-329, same greedy best-fit, device byte
    sizes, 256-B aligned slots); graph inputs and outputs own their buffers;
  * weights are pre-transformed once (bind_params); activations stay in the
    kernels' NHWC layout between nodes -- a layout change (NHWC <-> the
    packed input of the next conv) is inserted only where a consumer needs
    one (the stem's space-to-depth pack; the f32 parity path's NCHW input);
  * the launch list is a native plan (tec_plan_create, tec_sm100_abi.cpp):
    an array of tec_step records the C++ runtime walks, or captures once
    into a CUDA graph (tec_plan_capture) and replays -- no Python per
    launch.

Compute modes: "bf16" (activations bf16 NHWC, f32 accumulate; graph outputs
f32), "f32" (the bit-exact SIMT path: every conv equals the reference's
evaluate_graph bit for bit), "f32tc" (f32 on the tensor cores) and "i8"
(int8 graphs: i8 activations NHWC, i32 accumulate, bit-exact).
Members of a fused conv node that the conv epilogue cannot apply become
elementwise launches (tec_elementwise) around the conv:
  * a side chain -- unary members feeding an add / mul operand, e.g. the
    int8 shortcut scale(cast(y, i32)) -- runs BEFORE the conv into a shared
    operand buffer;
  * the tail of the main chain from the first non-epilogue member on (e.g.
    requantize, i32 -> i8) runs AFTER it, reading the conv's i32 result from
    a shared scratch buffer.
Integer range overflow in any step is reported by run() as FoldOverflow
(tec_plan_status). Unsupported nodes raise LoweringError -- there is no CPU
fallback.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import Callable, Dict, List, Optional

import numpy as np
import torch

from . import _abi
from ._abi import TecError
from .graph import (ComputeGraph, GraphNode, bn_eval, bn_scale, check_memory_plan,
                    fold_batch_norm, fuse_pass, nhwc_layout_pass, plan_memory)

E_LOWERING, E_IO, E_SHAPE = 15, 20, 2
_EPI = {"scale": _abi.EPI_SCALE, "bias_add": _abi.EPI_BIAS, "add": _abi.EPI_ADD,
        "mul": _abi.EPI_MUL, "relu": _abi.EPI_RELU}
_ELEM = {"cast": _abi.ELEM_CAST, "scale": _abi.ELEM_SCALE, "relu": _abi.ELEM_RELU,
         "requantize": _abi.ELEM_REQUANTIZE}
_DT = {"f32": _abi.DT_F32, "i32": _abi.DT_I32, "i8": _abi.DT_I8}
_BN_FOLD = ("bn_fold_weight", "bn_fold_bias")
_TORCH = {_abi.DT_F32: torch.float32, _abi.DT_BF16: torch.bfloat16,
          _abi.DT_I32: torch.int32, _abi.DT_I8: torch.int8}
_BYTES = {_abi.DT_F32: 4, _abi.DT_BF16: 2, _abi.DT_I32: 4, _abi.DT_I8: 1}
ALIGN = 256


@dataclass
class DevTensor:
    """A device tensor of the executor. shape is the LOGICAL (reference)
    shape; layout "nhwc" stores [N][H][W][C] (rank-2 [N][C] counts as nhwc
    with H = W = 1), "nchw" the reference row-major order."""
    buf: torch.Tensor
    shape: List[int]
    dtype: int
    layout: str = "nhwc"

    def ptr(self) -> int:
        return self.buf.data_ptr()

    @property
    def nchw4(self):
        s = self.shape
        return (s[0], s[1], s[2], s[3]) if len(s) == 4 else (s[0], s[1], 1, 1)


def _resolve_aliases(g: ComputeGraph) -> ComputeGraph:
    """The executor's view of a fused, layout-annotated graph: nodes that
    only re-view a buffer are removed and their consumers read the
    underlying tensor, so plan_memory sees the true lifetimes.
      * layout_transform row_major <-> nhwc (nhwc_layout_pass): realised by
        the consuming launch (see DevTensor.layout);
      * flatten of an [N, C, 1, 1] tensor: same bytes in NHWC;
      * sum(axis=3) -> sum(axis=2) -> scale(1/(H*W)), each with a single
        consumer: one global_avg_pool node (the reference composition).
    The result is internal (node types are kept, not re-validated)."""
    import copy
    outs = set(g.outputs)
    # an output's final NHWC -> row-major transform: the producer itself
    # takes the output id (outputs own their buffers; the unpack happens in
    # output())
    ren: Dict[str, str] = {}
    kinds = {n.id: n.op for n in g.nodes}
    for n in g.nodes:
        if (n.id in outs and n.op == "layout_transform" and
                {n.attrs.get("src_layout"), n.attrs.get("dst_layout")} == {"row_major", "nhwc"}
                and kinds[n.inputs[0]] not in ("input", "const") and n.inputs[0] not in outs):
            ren[n.inputs[0]] = n.id
    if ren:
        g2 = ComputeGraph([], list(g.outputs))
        for n in g.nodes:
            if n.id in outs and n.op == "layout_transform" and n.inputs[0] in ren:
                continue
            m = copy.deepcopy(n)
            m.id = ren.get(m.id, m.id)
            m.inputs = [ren.get(i, i) for i in m.inputs]
            for mm in m.members:
                mm.inputs = [ren.get(i, i) for i in mm.inputs]
            g2.nodes.append(m)
        g = g2
    cons = g.consumers()
    alias: Dict[str, str] = {}
    gap_of: Dict[str, str] = {}   # scale node id -> pooled input id
    dropped = set()
    for a in g.nodes:
        if a.op != "sum" or int(a.attrs.get("axis", -1)) != 3 or a.id in outs:
            continue
        x = g.node(a.inputs[0]).out_type
        ca = cons.get(a.id, [])
        if x.rank() != 4 or len(ca) != 1:
            continue
        b = g.node(ca[0])
        cb = cons.get(b.id, [])
        if b.op != "sum" or int(b.attrs.get("axis", -1)) != 2 or b.id in outs or len(cb) != 1:
            continue
        c = g.node(cb[0])
        if c.op != "scale" or float(c.attrs.get("scale", 1.0)) != 1.0 / (x.shape[2] * x.shape[3]):
            continue
        gap_of[c.id] = a.inputs[0]
        dropped |= {a.id, b.id}
    shapes = {n.id: n.out_type.shape for n in g.nodes}
    for n in g.nodes:
        if (n.op == "layout_transform" and n.id not in outs and
                {n.attrs.get("src_layout"), n.attrs.get("dst_layout")} == {"row_major", "nhwc"}):
            # realised by the consumer (a conv's input pack reads NCHW, the
            # pools convert on demand) or a no-op: DevTensor tracks the
            # physical layout
            alias[n.id] = alias.get(n.inputs[0], n.inputs[0])
            dropped.add(n.id)
            continue
        if n.op == "flatten" and n.id not in outs:
            src = n.inputs[0]
            sh = shapes[src]
            if len(sh) == 4 and sh[2] * sh[3] == 1:
                alias[n.id] = alias.get(src, src)
                dropped.add(n.id)
    out = ComputeGraph([], list(g.outputs))
    for n in g.nodes:
        if n.id in dropped:
            continue
        m = copy.deepcopy(n)
        if m.id in gap_of:
            m.op, m.inputs, m.attrs = "global_avg_pool", [gap_of[m.id]], {}
        m.inputs = [alias.get(i, i) for i in m.inputs]
        for mm in m.members:
            mm.inputs = [alias.get(i, i) for i in mm.inputs]
        out.nodes.append(m)
    return out


def f32_output(n: GraphNode) -> bool:
    """Graph outputs kept in f32 in bf16 mode (see DeviceGraph._node_dtype)."""
    root = n.members[0] if n.op == "fused" else n
    return root.op in ("matmul", "global_avg_pool", "scale")


def split_conv_members(n: GraphNode):
    """A conv-rooted fused node's members (graph.cpp:209-222 order) as
    (root, main, sides, tail):
      main  -- the chain from the root the conv epilogue applies;
      sides -- unary chains (first input, last member id, members) that
               compute an add / mul operand of the main chain from a
               tensor outside the node (fuse_pass pulls them in);
      tail  -- main-chain members from the first one the epilogue cannot
               apply on (all unary elementwise)."""
    ms = n.members if n.op == "fused" else [n]
    root = ms[0]
    if root.op not in ("conv2d", "depthwise_conv2d", "matmul"):
        raise TecError(E_LOWERING, f"fused node '{n.id}' is not conv/matmul-rooted")
    ids = {m.id for m in ms}
    main, sides, side_of, prev = [], [], {}, root.id
    for m in ms[1:]:
        if prev in m.inputs:
            main.append(m)
            prev = m.id
            continue
        if m.op not in _ELEM or len(m.inputs) != 1:
            raise TecError(E_LOWERING, f"fused member '{m.id}' ({m.op}) is off the conv chain")
        src = m.inputs[0]
        if src in side_of:  # extends a side chain
            k = side_of.pop(src)
            first, _, members = sides[k]
            sides[k] = (first, m.id, members + [m])
        elif src in ids:
            raise TecError(E_LOWERING, f"fused member '{m.id}' reads an interior value")
        else:
            sides.append((src, m.id, [m]))
            k = len(sides) - 1
        side_of[m.id] = k
    cut = next((i for i, m in enumerate(main) if m.op not in _EPI), len(main))
    head, tail = main[:cut], main[cut:]
    for m in tail:
        if m.op not in _ELEM or len(m.inputs) != 1:
            raise TecError(E_LOWERING, f"member '{m.op}' has no sm100 epilogue")
    return root, head, sides, tail


def _i8_shortcut_scale(members) -> Optional[int]:
    """c for a side chain [cast(i32)] (c = 1) or [cast(i32), scale(c)] with an
    integral |c| <= 2^24 (no i32 overflow for any i8 value), else None."""
    if not members or members[0].op != "cast" or members[0].attrs.get("dtype", "i32") != "i32":
        return None
    if len(members) == 1:
        return 1
    if len(members) != 2 or members[1].op != "scale":
        return None
    c = float(members[1].attrs.get("scale", 1.0))
    if c != int(c) or abs(c) > 2 ** 24:
        return None
    return int(c)


class DeviceGraph:
    def __init__(self, g: ComputeGraph, compute: str = "bf16", device: int = 0,
                 knobs: Optional[Dict[str, dict]] = None):
        if compute not in ("bf16", "f32", "f32tc", "i8"):
            raise TecError(E_LOWERING, f"executor compute mode '{compute}' (bf16 | f32 | f32tc | i8)")
        self.lib = _abi.load()
        self.dev = torch.device("cuda", device)
        self.compute = compute
        # f32tc: every conv on the tensor cores at f32 (conv_f32tc.cu), f32
        # NHWC activations between layers, each conv's input packed into its
        # three bf16 planes by a layout step
        self.cmode = {"bf16": _abi.COMPUTE_BF16, "f32": _abi.COMPUTE_F32,
                      "f32tc": _abi.COMPUTE_F32TC, "i8": _abi.COMPUTE_I8}[compute]
        self.act_dt = {"bf16": _abi.DT_BF16, "i8": _abi.DT_I8}.get(compute, _abi.DT_F32)
        self.in_dtype = "i8" if compute == "i8" else "f32"  # graph input / weight dtype
        self.knobs = knobs or {}
        # BN folded into conv weights / biases (parameters, bind time), then
        # the reference's fusion
        self.fused = fuse_pass(fold_batch_norm(g))
        # the B200 layout pass: NHWC placement made explicit in the graph
        self.laid = nhwc_layout_pass(self.fused)
        self.g = _resolve_aliases(self.laid)
        self.outputs = list(self.g.outputs)
        self._classify_inputs()
        self.steps: List[_abi.Step] = []
        self.tensors: Dict[str, DevTensor] = {}
        self.params: Dict[str, torch.Tensor] = {}
        self.param_prep: List[Callable[[int], None]] = []
        self.feeds: Dict[str, DevTensor] = {}
        self.keep: list = []
        self._plan()
        self._compile()
        self._native = None
        self._captured = False
        self._make_plan()

    def _make_plan(self):
        arr = (_abi.Step * max(len(self.steps), 1))(*self.steps)
        h = C.c_void_p()
        with torch.cuda.device(self.dev):
            _abi.check(self.lib.tec_plan_create(arr, len(self.steps), C.byref(h)))
        self._native = h

    def __del__(self):
        h = getattr(self, "_native", None)
        if h is not None and h.value:
            self.lib.tec_plan_destroy(h)
            self._native = None

    # ------------------------------------------------------------ analysis
    def _classify_inputs(self):
        """Graph inputs used only as a weight / bias operand are parameters
        (uploaded and transformed once); the rest are per-run feeds."""
        uses: Dict[str, set] = {}
        for n in self.g.nodes:
            members = n.members if n.op == "fused" else [n]
            for m in members:
                for pos, i in enumerate(m.inputs):
                    role = "data"
                    if m.op in ("conv2d", "depthwise_conv2d", "matmul") and pos == 1:
                        role = "weight"
                    elif m.op == "bias_add" and pos == 1:
                        role = "bias"
                    elif m.op in _BN_FOLD:
                        role = "param"  # folded into a weight / bias at bind time
                    uses.setdefault(i, set()).add(role)
        self.param_names, self.feed_names = [], []
        cons = self.g.consumers()
        for n in self.g.nodes:
            if n.op == "const":
                if cons.get(n.id) and all(self.g.node(c).op == "bn_fold_bias" for c in cons[n.id]):
                    continue  # fold_batch_norm's zero bias
                raise TecError(E_LOWERING, "const nodes: bind them as parameters (inputs)")
            if n.op != "input":
                continue
            u = uses.get(n.id, set())
            if u and (u <= {"weight", "param"} or u <= {"bias", "param"}):
                self.param_names.append(n.id)
            else:
                self.feed_names.append(n.id)

    def _node_dtype(self, n: GraphNode) -> int:
        """bf16 mode: every activation is bf16 (a conv's add/mul operand
        must share its output dtype); graph outputs of the head (matmul-
        rooted nodes, pools) are produced in f32."""
        if n.out_type.dtype in ("i32", "i8"):
            return _DT[n.out_type.dtype]
        return _abi.DT_F32 if n.id in self.outputs and f32_output(n) else self.act_dt

    def _dev_bytes(self, n: GraphNode) -> int:
        return n.out_type.num_elements() * _BYTES[self._node_dtype(n)]

    def _plan(self):
        self.plan = plan_memory(self.g, nbytes=self._dev_bytes, align=ALIGN)
        check_memory_plan(self.g, self.plan, nbytes=self._dev_bytes)
        self.arena = torch.empty(max(self.plan.total_bytes, ALIGN), dtype=torch.uint8,
                                 device=self.dev)
        # shared buffers of the elementwise launches around fused convs
        # (steps run in order on one stream, so one of each suffices)
        tail_b, side_b = 0, 0
        for n in self.g.nodes:
            if n.op == "fused" and n.members[0].op in ("conv2d", "depthwise_conv2d", "matmul"):
                _, _, sides, tail = split_conv_members(n)
                if tail:
                    tail_b = max(tail_b, n.out_type.num_elements() * 4)
                for _, last, _ in sides:
                    side_b = max(side_b, n.out_type.num_elements() * 4)
        self.tail_buf = torch.empty(max(tail_b, ALIGN), dtype=torch.uint8, device=self.dev)
        self.side_buf = torch.empty(max(side_b, ALIGN), dtype=torch.uint8, device=self.dev)

    def _out_buffer(self, n: GraphNode, dtype: int, nelem: int) -> torch.Tensor:
        nbytes = nelem * _BYTES[dtype]
        if n.id in self.plan.slot_of:
            off = self.plan.slot_offset[self.plan.slot_of[n.id]]
            raw = self.arena[off:off + nbytes]
        else:
            raw = torch.empty(nbytes, dtype=torch.uint8, device=self.dev)
        return raw.view(_TORCH[dtype])

    def _scratch(self, nbytes: int) -> torch.Tensor:
        t = torch.empty(max(nbytes, 16), dtype=torch.uint8, device=self.dev)
        self.keep.append(t)
        return t

    # ------------------------------------------------------------- compile
    def _compile(self):
        for n in self.g.nodes:
            if n.op == "input":
                if n.id in self.feed_names:
                    shape = list(n.out_type.shape)
                    dt = _DT[n.out_type.dtype]
                    buf = torch.empty(int(np.prod(shape)), dtype=_TORCH[dt], device=self.dev)
                    t = DevTensor(buf, shape, dt, "nchw")
                    self.feeds[n.id] = t
                    self.tensors[n.id] = t
                continue
            if n.op == "fused" or n.op in ("conv2d", "depthwise_conv2d", "matmul"):
                self._compile_conv(n)
            elif n.op == "max_pool2d":
                self._compile_maxpool(n)
            elif n.op == "global_avg_pool":
                self._compile_avgpool(n, self.tensors[n.inputs[0]])
            elif n.op in _ELEM or (n.op == "fused" and n.members[0].op in _ELEM):
                self._compile_elemwise(n)
            elif n.op in _BN_FOLD or n.op == "const":
                continue  # parameter derivations: computed in bind_params (see _bind_weight)
            elif n.op == "layout_transform":
                # an output's final NHWC -> NCHW transform: output() unpacks
                # on read (tec_output_unpack)
                self.tensors[n.id] = self.tensors[n.inputs[0]]
            else:
                raise TecError(E_LOWERING, f"no sm100 lowering for node '{n.id}' ({n.op})")
        for o in self.outputs:
            if o not in self.tensors:
                raise TecError(E_LOWERING, f"output '{o}' was not produced")

    # ---------------------------------------------------------------- conv
    def _conv_members(self, n: GraphNode):
        root, head, sides, tail = split_conv_members(n)
        side_ids = {last for _, last, _ in sides}
        items, prev = [], root.id
        for m in head:
            others = [i for i in m.inputs if i != prev]
            if len(others) != len(m.inputs) - 1:
                raise TecError(E_LOWERING, "fused members are not a single chain")
            if m.op == "bias_add" and int(m.attrs.get("axis", 1)) != 1:
                raise TecError(E_LOWERING, "bias_add must broadcast over channels")
            items.append((m.op, others[0] if others else None, m))
            prev = m.id
        used = {it[1] for it in items if it[0] in ("add", "mul")}
        if side_ids - used:
            raise TecError(E_LOWERING, f"fused node '{n.id}': a side chain feeds no add / mul")
        for op in ("bias_add", "add", "mul"):
            # one operand slot each in tec_epilogue: a second member of the
            # same kind would silently read the first one's operand
            if sum(1 for it in items if it[0] == op) > 1:
                raise TecError(E_LOWERING, f"fused node '{n.id}' has more than one '{op}' member")
        return root, items, sides, tail

    def _conv_input(self, d: _abi.ConvDesc, src: DevTensor) -> int:
        """Device pointer of x in the packed layout conv `d` reads,
        inserting a layout step when the producer's layout differs."""
        lay = _abi.ConvLayout()
        _abi.check(self.lib.tec_conv_layout_of(C.byref(d), C.byref(lay)))
        direct = (src.layout == "nhwc" and src.dtype == lay.act_dtype and lay.cp == d.c
                  and not (self.cmode == _abi.COMPUTE_F32 and not d.depthwise))
        if direct:
            return src.ptr()
        if (self.cmode == _abi.COMPUTE_F32TC and not d.depthwise and src.layout == "nhwc"
                and src.dtype == _abi.DT_F32
                and not (d.stride_h == 2 and d.stride_w == 2 and 4 * d.c <= 16)):  # not s2d
            # f32 NHWC -> the conv's three bf16 planes in one pass
            packed = self._scratch(lay.act_bytes)
            self.steps.append(_abi.Step(kind=_abi.STEP_PACK_NHWC, conv=d, src=src.ptr(),
                                        dst=packed.data_ptr()))
            return packed.data_ptr()
        # src -> NCHW f32 (the reference layout) -> tec_activation_pack
        if src.layout == "nchw" and src.dtype == _DT[self.in_dtype]:
            nchw = src.buf  # the reference layout and dtype tec_activation_pack reads
        elif self.compute == "i8" and (src.layout != "nhwc" or src.dtype != _abi.DT_I8):
            raise TecError(E_LOWERING, "i8 conv input must be i8 (NCHW feed or NHWC activation)")
        else:
            n_, c_, h_, w_ = src.nchw4
            udt = _DT[self.in_dtype]
            nchw = self._scratch(n_ * c_ * h_ * w_ * _BYTES[udt])
            self.steps.append(_abi.Step(kind=_abi.STEP_UNPACK, src_dtype=src.dtype,
                                        dst_dtype=udt, src=src.ptr(),
                                        dst=nchw.data_ptr(), n=n_, c=c_, h=h_, w_=w_))
        if self.cmode == _abi.COMPUTE_F32 and not d.depthwise:
            return nchw.data_ptr()  # the exact path reads NCHW f32 as is
        packed = self._scratch(lay.act_bytes)
        self.steps.append(_abi.Step(kind=_abi.STEP_PACK, conv=d, src=nchw.data_ptr(),
                                    dst=packed.data_ptr()))
        return packed.data_ptr()

    def _elem_prog(self, members, src_dt: int, dst_dt: int, count: int) -> _abi.ElemProg:
        if len(members) > _abi.MAX_ELEM_OPS:
            raise TecError(E_LOWERING, f"more than {_abi.MAX_ELEM_OPS} elementwise members")
        p = _abi.ElemProg(n_ops=len(members), src_dtype=src_dt, dst_dtype=dst_dt, count=count)
        for k, m in enumerate(members):
            p.kind[k] = _ELEM[m.op]
            if m.op == "cast":
                p.cast_to[k] = _DT[m.attrs.get("dtype", "i32")]
            elif m.op == "scale":
                p.scale[k] = float(m.attrs.get("scale", 1.0))
            elif m.op == "requantize":
                p.mult[k] = int(m.attrs.get("multiplier", 1))
                p.shift[k] = int(m.attrs.get("shift", 0))
        return p

    def _elem_step(self, members, src: DevTensor, dst_ptr: int, dst_dt: int, count: int):
        if src.layout != "nhwc":
            src = self._to_nhwc(src, src.dtype)
        self.steps.append(_abi.Step(kind=_abi.STEP_ELEMWISE, src=src.ptr(), dst=dst_ptr,
                                    src_dtype=src.dtype, dst_dtype=dst_dt,
                                    elem=self._elem_prog(members, src.dtype, dst_dt, count)))

    def _compile_elemwise(self, n: GraphNode):
        ms = n.members if n.op == "fused" else [n]
        for a, b in zip(ms, ms[1:]):
            if b.op not in _ELEM or b.inputs != [a.id]:
                raise TecError(E_LOWERING, f"fused node '{n.id}' is not a unary elementwise chain")
        x = self.tensors[ms[0].inputs[0]]
        out_dt = self._node_dtype(n)
        y = self._out_buffer(n, out_dt, n.out_type.num_elements())
        self._elem_step(ms, x, y.data_ptr(), out_dt, n.out_type.num_elements())
        self.tensors[n.id] = DevTensor(y, list(n.out_type.shape), out_dt, "nhwc")

    def _compile_conv(self, n: GraphNode):
        root, items, sides, tail = self._conv_members(n)
        x = self.tensors[root.inputs[0]]
        wname = root.inputs[1]
        bn = None
        wnode = self.g.node(wname)
        if wnode.op == "bn_fold_weight":  # fold_batch_norm: W * gamma / sqrt(var + eps)
            bn = wnode
            wname = wnode.inputs[0]
        if wname not in self.param_names or (bn and not all(i in self.param_names for i in bn.inputs)):
            raise TecError(E_LOWERING, f"conv weight '{wname}' must be a graph input parameter")
        wt = self.g.node(wname).out_type
        if root.op == "matmul":
            m_, k_ = x.shape[0], int(np.prod(x.shape[1:]))
            d = _abi.ConvDesc(n=m_, c=k_, h=1, w=1, k=wt.shape[1], r=1, s=1, stride_h=1,
                              stride_w=1, pad_h=0, pad_w=0, depthwise=0, compute=self.cmode)
        else:
            from .ops import conv_desc
            d = conv_desc(root.op, self.g.node(root.inputs[0]).out_type.shape, wt.shape,
                          root.attrs, self.cmode)
        if self.g.node(root.inputs[0]).out_type.dtype != self.in_dtype:
            raise TecError(E_LOWERING, f"executor compute '{self.compute}' runs {self.in_dtype} "
                                       "convolutions")
        xptr = self._conv_input(d, x)
        lay = _abi.ConvLayout()
        _abi.check(self.lib.tec_conv_layout_of(C.byref(d), C.byref(lay)))
        wpk = self._scratch(lay.wt_bytes)
        self._bind_weight(wname, d, wpk, transpose=root.op == "matmul", bn=bn)
        node_dt = self._node_dtype(n)
        oh, ow = (lay.oh, lay.ow)
        count = d.n * d.k * oh * ow
        y = self._out_buffer(n, node_dt, count)
        # the epilogue's result: the node's own buffer, or (with a tail) the
        # accumulator-dtype scratch the tail's elementwise launch reads
        if (tail or sides) and self.compute != "i8":
            raise TecError(E_LOWERING, f"fused node '{n.id}': elementwise members around a conv "
                                       "need compute 'i8'")
        if len(sides) > 1:
            raise TecError(E_LOWERING, f"fused node '{n.id}': more than one side chain")
        epi = _abi.Epilogue()
        # int8 graphs: a [requantize] tail and a [cast(i32), scale(c)]
        # shortcut fold into the conv epilogue itself (conv_epilogue.cuh Q
        # programs: i8 residual in, i8 out) when the kernels' conditions
        # hold; otherwise they run as elementwise launches around the conv.
        fuse_tail = (len(tail) == 1 and tail[0].op == "requantize" and d.k % 16 == 0
                     and not d.depthwise)
        if fuse_tail:
            epi.rq_mult = int(tail[0].attrs.get("multiplier", 1))
            epi.rq_shift = int(tail[0].attrs.get("shift", 0))
            tail = []
        fused_side = {}
        for first, last, members in list(sides):
            c = _i8_shortcut_scale(members)
            src = self.tensors[first]
            adds = [it for it in items if it[0] == "add" and it[1] == last]
            if (c is not None and fuse_tail and d.k % 32 == 0 and src.layout == "nhwc"
                    and src.dtype == _abi.DT_I8 and adds):
                fused_side[last] = (src, c)
                sides.remove((first, last, members))
        out_dt = lay.acc_dtype if tail else node_dt
        conv_dst = self.tail_buf.data_ptr() if tail else y.data_ptr()
        side_dst = {}
        for first, last, members in sides:
            # the operand's dtype is the conv output's (epilogue operands)
            self._elem_step(members, self.tensors[first], self.side_buf.data_ptr(), lay.acc_dtype,
                            count)
            side_dst[last] = DevTensor(self.side_buf, list(n.out_type.shape), lay.acc_dtype, "nhwc")
        for i, (op, other, m) in enumerate(items):
            epi.ops[i] = _EPI[op]
            if op == "relu":
                continue
            if op == "scale":
                epi.scale[i] = float(m.attrs.get("scale", 1.0))
            elif op == "bias_add":
                if other not in self.param_names and self.g.node(other).op != "bn_fold_bias":
                    raise TecError(E_LOWERING, "bias must be a graph input parameter")
                epi.bias = self._bias_ptr(other)
            elif other in fused_side:
                r, c = fused_side[other]
                epi.residual = r.ptr()
                epi.residual_i8 = 1
                epi.residual_scale = c
            else:
                r = side_dst.get(other) or self.tensors[other]
                want_dt = lay.acc_dtype if self.compute == "i8" else out_dt
                if r.layout == "nchw" and r.dtype != _abi.DT_I8:
                    # a graph input (the reference's NCHW) as the shortcut:
                    # one relayout launch into the conv output's NHWC / dtype
                    r = self._to_nhwc(r, want_dt)
                if r.layout != "nhwc" or r.dtype != want_dt:
                    raise TecError(E_LOWERING, f"'{op}' operand must be an NHWC {out_dt} tensor")
                if op == "add":
                    epi.residual = r.ptr()
                else:
                    epi.mul_operand = r.ptr()
        epi.n_ops = len(items)
        if fuse_tail:
            epi.ops[epi.n_ops] = _abi.EPI_REQUANTIZE
            epi.n_ops += 1
        kn = _abi.Knobs(**self.knobs.get(n.id, self.knobs.get(n.id.split("#")[0], {})))
        self.steps.append(_abi.Step(kind=_abi.STEP_DEPTHWISE if d.depthwise else _abi.STEP_CONV,
                                    dst_dtype=out_dt, conv=d, epi=epi, knobs=kn, src=xptr,
                                    w=wpk.data_ptr(), dst=conv_dst))
        shape = list(n.out_type.shape)
        if tail:
            acc = DevTensor(self.tail_buf, shape, out_dt, "nhwc")
            self._elem_step(tail, acc, y.data_ptr(), node_dt, count)
        self.tensors[n.id] = DevTensor(y, shape, node_dt, "nhwc")

    def _bind_weight(self, name: str, d: _abi.ConvDesc, wpk: torch.Tensor, transpose: bool,
                     bn: Optional[GraphNode] = None):
        src_shape = self.g.node(name).out_type.shape

        npdt = np.int8 if self.compute == "i8" else np.float32

        def prep(params: Dict[str, np.ndarray], st: int, d=d, wpk=wpk):
            w = np.asarray(params[name], dtype=npdt)
            if list(w.shape) != list(src_shape):
                raise TecError(E_SHAPE, f"parameter '{name}' is {list(w.shape)}, expected {src_shape}")
            if transpose:  # matmul [K, N] -> OIHW [N, K, 1, 1]
                w = np.ascontiguousarray(w.T).reshape(w.shape[1], w.shape[0], 1, 1)
            wd = torch.from_numpy(np.ascontiguousarray(w)).to(self.dev)
            if bn is not None:
                # BN folded inside the pretransform: the per-channel factor
                # gamma / sqrt(var + eps) (K values, host), the products on device
                _, g_, v_ = bn.inputs
                sc = bn_scale(params[g_], params[v_], float(bn.attrs.get("eps", 1e-5)))
                sd = torch.from_numpy(sc).to(self.dev)
                _abi.check(self.lib.tec_weight_pretransform_bn(C.byref(d), wd.data_ptr(),
                                                               sd.data_ptr(), wpk.data_ptr(), st))
            else:
                _abi.check(self.lib.tec_weight_pretransform(C.byref(d), wd.data_ptr(),
                                                            wpk.data_ptr(), st))
            torch.cuda.current_stream(self.dev).synchronize()
        self.param_prep.append(prep)

    def _bias_ptr(self, name: str) -> int:
        if name not in self.params:
            node = self.g.node(name)
            k = node.out_type.shape[0]
            integer = self.compute == "i8"
            self.params[name] = torch.empty(k, dtype=torch.int32 if integer else torch.float32,
                                            device=self.dev)
            if node.op == "bn_fold_bias":  # (b - mean) * s + beta, K values on the host
                for i in node.inputs:
                    if i not in self.param_names and self.g.node(i).op != "const":
                        raise TecError(E_LOWERING, f"bn_fold_bias operand '{i}' is not a parameter")

            def prep(params, st, name=name, npdt=np.int32 if integer else np.float32):
                if node.op == "bn_fold_bias":
                    vals = [params[i] if i in params else self.g.node(i).data for i in node.inputs]
                    params = {name: bn_eval("bn_fold_bias", vals, float(node.attrs.get("eps", 1e-5)))}
                b = np.asarray(params[name], dtype=npdt)
                if b.shape != tuple(self.params[name].shape):
                    raise TecError(E_SHAPE, f"parameter '{name}' has shape {b.shape}")
                self.params[name].copy_(torch.from_numpy(b))
            self.param_prep.append(prep)
        return self.params[name].data_ptr()

    # ---------------------------------------------------------------- pools
    def _to_nhwc(self, src: DevTensor, dtype: Optional[int] = None) -> DevTensor:
        if src.layout == "nhwc":
            return src
        dt = self.act_dt if dtype is None else dtype
        n_, c_, h_, w_ = src.nchw4
        out = self._scratch(n_ * c_ * h_ * w_ * _BYTES[dt]).view(_TORCH[dt])

        self.steps.append(_abi.Step(kind=_abi.STEP_TO_NHWC, src_dtype=src.dtype,
                                    dst_dtype=dt, src=src.ptr(), dst=out.data_ptr(),
                                    n=n_, c=c_, h=h_, w_=w_))
        return DevTensor(out, src.shape, dt, "nhwc")

    def _compile_maxpool(self, n: GraphNode):
        x = self._to_nhwc(self.tensors[n.inputs[0]])
        k = [int(v) for v in n.attrs.get("kernel", [3, 3])]
        st_ = [int(v) for v in n.attrs.get("strides", [2, 2])]
        pd = [int(v) for v in n.attrs.get("padding", [1, 1])]
        nn, c, h, w = x.nchw4
        pdsc = _abi.PoolDesc(n=nn, c=c, h=h, w=w, r=k[0], s=k[1], stride_h=st_[0],
                             stride_w=st_[1], pad_h=pd[0], pad_w=pd[1], dtype=x.dtype,
                             out_dtype=x.dtype)
        y = self._out_buffer(n, x.dtype, n.out_type.num_elements())
        if n.id in self.outputs:
            raise TecError(E_LOWERING, "max_pool2d as a graph output")
        self.steps.append(_abi.Step(kind=_abi.STEP_MAX_POOL, pool=pdsc, src=x.ptr(),
                                    dst=y.data_ptr()))
        self.tensors[n.id] = DevTensor(y, list(n.out_type.shape), x.dtype, "nhwc")

    def _compile_avgpool(self, n: GraphNode, src: DevTensor):
        x = self._to_nhwc(src)
        nn, c, h, w = x.nchw4
        out_dt = _abi.DT_F32 if (n.id in self.outputs or self.act_dt == _abi.DT_F32) else self.act_dt
        pdsc = _abi.PoolDesc(n=nn, c=c, h=h, w=w, r=1, s=1, stride_h=1, stride_w=1,
                             pad_h=0, pad_w=0, dtype=x.dtype, out_dtype=out_dt)
        y = self._out_buffer(n, out_dt, nn * c)
        self.steps.append(_abi.Step(kind=_abi.STEP_AVG_POOL, pool=pdsc, src=x.ptr(),
                                    dst=y.data_ptr()))
        self.tensors[n.id] = DevTensor(y, list(n.out_type.shape), out_dt, "nhwc")

    # ------------------------------------------------------------ execution
    def bind_params(self, params: Dict[str, np.ndarray]) -> None:
        missing = [p for p in self.param_names if p not in params]
        if missing:
            raise TecError(E_IO, f"no value for graph parameter(s) {missing[:4]}")
        st = torch.cuda.current_stream(self.dev).cuda_stream
        with torch.cuda.device(self.dev):
            for prep in self.param_prep:
                prep(params, st)

    def set_feed(self, name: str, value, stream: Optional[torch.cuda.Stream] = None) -> None:
        """Copies a feed into its device buffer ON `stream` (default: the
        current stream), so a later launch(stream) is ordered after it."""
        t = self.feeds[name]
        v = value if isinstance(value, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(value))
        if list(v.shape) != t.shape:
            raise TecError(E_SHAPE, f"input {name} is {list(v.shape)}, expected {t.shape}")
        s = stream or torch.cuda.current_stream(self.dev)
        with torch.cuda.stream(s):
            t.buf.copy_(v.reshape(-1).to(t.buf.dtype), non_blocking=True)

    def launch(self, stream: Optional[torch.cuda.Stream] = None) -> None:
        """Enqueue every step on `stream` (device-resident feeds)."""
        s = stream or torch.cuda.current_stream(self.dev)
        with torch.cuda.device(self.dev):
            _abi.check(self.lib.tec_plan_run(self._native, C.c_void_p(s.cuda_stream)))

    def capture(self) -> None:
        """Capture the launch list into a CUDA graph that launch() replays
        (tec_plan_capture: one eager pass, then stream capture). Buffers and
        parameters are bound by address, so re-binding parameters or feeds
        keeps the captured graph valid."""
        s = torch.cuda.Stream(self.dev)
        s.wait_stream(torch.cuda.current_stream(self.dev))
        with torch.cuda.device(self.dev):
            _abi.check(self.lib.tec_plan_capture(self._native, C.c_void_p(s.cuda_stream)))
        torch.cuda.current_stream(self.dev).wait_stream(s)
        self._captured = True

    def launch_step(self, i: int, stream: Optional[torch.cuda.Stream] = None) -> None:
        """Enqueue step i alone, eagerly (per-launch profiling)."""
        s = stream or torch.cuda.current_stream(self.dev)
        with torch.cuda.device(self.dev):
            _abi.check(self.lib.tec_plan_run_steps(self._native, i, 1, C.c_void_p(s.cuda_stream)))

    @property
    def n_launches(self) -> int:
        return int(self.lib.tec_plan_size(self._native))

    def output(self, name: str) -> torch.Tensor:
        """The device output in the reference layout (NCHW / [N, K]): f32,
        or the node's own integer dtype (i8 / i32, exact)."""
        t = self.tensors[name]
        shape = t.shape
        dt = t.dtype if t.dtype in (_abi.DT_I8, _abi.DT_I32) else _abi.DT_F32
        if t.layout == "nhwc" and len(shape) == 4 and shape[2] * shape[3] > 1:
            n_, c_, h_, w_ = shape
            out = torch.empty(shape, dtype=_TORCH[dt], device=self.dev)
            _abi.check(self.lib.tec_output_unpack(t.ptr(), t.dtype, out.data_ptr(), dt,
                                                  n_, c_, h_, w_,
                                                  torch.cuda.current_stream(self.dev).cuda_stream))
            return out
        v = t.buf[:int(np.prod(shape))].reshape(shape)
        return v if dt != _abi.DT_F32 else v.float()

    def status(self, stream: Optional[torch.cuda.Stream] = None) -> None:
        """Raises FoldOverflow if an integer step overflowed i32 since the
        last check (synchronizes `stream`)."""
        s = stream or torch.cuda.current_stream(self.dev)
        with torch.cuda.device(self.dev):
            _abi.check(self.lib.tec_plan_status(self._native, C.c_void_p(s.cuda_stream)))

    def run(self, feeds: Dict[str, np.ndarray]) -> Dict[str, np.ndarray]:
        """evaluate_graph(g, feeds) on the device; host arrays in and out."""
        with torch.cuda.device(self.dev):
            for name in self.feed_names:
                if name not in feeds:
                    raise TecError(E_IO, f"no value for graph input '{name}'")
                self.set_feed(name, feeds[name])
            self.launch()
            outs = {o: self.output(o).cpu().numpy() for o in self.outputs}
            self.status()
        return outs
