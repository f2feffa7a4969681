"""The reference's headline workloads.

ResNet-18 conv C1-C12 and MobileNet depthwise D1-D9, with pad = k // 2
(the reference pads symmetrically, R/src/ops.cpp:125). Algorithmic work
per launch follows BASELINE.md: FLOPs = 2*N*OC*OH*OW*IC*KH*KW (depthwise:
IC := 1); compulsory bytes = every operand + the output once
(R/src/loop_ir.cpp:524-534).
"""
from __future__ import annotations

import numpy as np
from dataclasses import dataclass

# name: (H=W, IC, OC, K, stride)
RESNET18_CONVS = {
    "C1": (224, 3, 64, 7, 2), "C2": (56, 64, 64, 3, 1), "C3": (56, 64, 64, 1, 1),
    "C4": (56, 64, 128, 3, 2), "C5": (56, 64, 128, 1, 2), "C6": (28, 128, 128, 3, 1),
    "C7": (28, 128, 256, 3, 2), "C8": (28, 128, 256, 1, 2), "C9": (14, 256, 256, 3, 1),
    "C10": (14, 256, 512, 3, 2), "C11": (14, 256, 512, 1, 2), "C12": (7, 512, 512, 3, 1),
}
# name: (H=W, C, stride), 3x3 kernels
MOBILENET_DW = {
    "D1": (112, 32, 1), "D2": (112, 64, 2), "D3": (56, 128, 1), "D4": (56, 128, 2),
    "D5": (28, 256, 1), "D6": (28, 256, 2), "D7": (14, 512, 1), "D8": (14, 512, 2),
    "D9": (7, 1024, 1),
}


@dataclass(frozen=True)
class ConvWorkload:
    name: str
    n: int
    c: int
    h: int
    w: int
    k: int
    r: int
    s: int
    stride: int
    pad: int
    depthwise: bool = False

    @property
    def oh(self) -> int:
        return (self.h + 2 * self.pad - self.r) // self.stride + 1

    @property
    def ow(self) -> int:
        return (self.w + 2 * self.pad - self.s) // self.stride + 1

    @property
    def flops(self) -> int:
        ic = 1 if self.depthwise else self.c
        return 2 * self.n * self.k * self.oh * self.ow * ic * self.r * self.s

    def bytes(self, in_bytes: int, out_bytes: int, bias_bytes: int = 4) -> int:
        wt = (self.c if self.depthwise else self.k * self.c) * self.r * self.s
        return (self.n * self.c * self.h * self.w * in_bytes + wt * in_bytes +
                self.k * bias_bytes + self.n * self.k * self.oh * self.ow * out_bytes)


def resnet_layer(name: str, batch: int) -> ConvWorkload:
    hw, c, k, r, s = RESNET18_CONVS[name]
    return ConvWorkload(name, batch, c, hw, hw, k, r, r, s, r // 2)


def mobilenet_layer(name: str, batch: int) -> ConvWorkload:
    hw, c, s = MOBILENET_DW[name]
    return ConvWorkload(name, batch, c, hw, hw, c, 3, 3, s, 1, depthwise=True)


# ------------------------------------------------ ResNet-18 graph (config 4)
def resnet18_graph(batch: int, num_classes: int = 1000, image: int = 224,
                   maxpool: bool = True, width: int = 64, head: bool = True,
                   dtype: str = "f32"):
    """ResNet-18 inference as a reference-format ComputeGraph (SURVEY 8d
    config 4): BN folded into each conv's bias, so every conv is
    conv2d -> bias_add (-> add shortcut) -> relu, which fuse_pass groups
    into one fused node per conv. Weights and biases are graph inputs
    (w_<layer>, b_<layer>); the head is global_avg_pool -> flatten ->
    matmul -> bias_add. `maxpool=False` drops the stem pool (the reference
    registry has no pooling op; that variant is what the reference's own
    fuse_pass / plan_memory can be run on) and replaces global_avg_pool by
    the reference composition scale(sum(sum(x, 3), 2)); `head=False` ends
    the graph at the last block's relu.
    Downsample branches are emitted before their block's first conv, so
    the block's second conv fuses [conv2d, bias_add, add, relu].

    dtype "i8" (SURVEY 8f.4, int8 end to end; body only, head=False): i8
    image and weights, i32 biases; every conv ends in requantize (i32 ->
    i8, multiplier / 2^16 ~ 1 / (4 sqrt(K)) -- 5.5 sqrt(K) with a shortcut or
    without relu --, about the accumulator's spread
    for the synthetic operands of int8_resnet18_params), so every
    activation between layers is i8 -- the downsample branch too; a
    shortcut enters the block's i32 accumulator domain as
    scale(cast(y, i32), round(4.6 sqrt(K)))."""
    from .graph import ComputeGraph, GraphNode, TensorType

    if dtype not in ("f32", "i8"):
        raise ValueError(f"resnet18_graph dtype {dtype!r} (f32 | i8)")
    if dtype == "i8" and head:
        raise ValueError("the int8 ResNet-18 graph is the body only (head=False)")
    i8 = dtype == "i8"
    nodes = []

    def inp(nid, shape, dt=None):
        nodes.append(GraphNode(nid, "input", out_type=TensorType(list(shape), dt or dtype)))
        return nid

    def conv(name, x, cin, cout, k, stride, relu=True, shortcut=None):
        w = inp(f"w_{name}", (cout, cin, k, k))
        b = inp(f"b_{name}", (cout,), "i32" if i8 else "f32")
        nodes.append(GraphNode(f"{name}", "conv2d", [x, w],
                               {"strides": [stride, stride], "padding": [k // 2, k // 2]}))
        nodes.append(GraphNode(f"{name}_bias", "bias_add", [name, b]))
        y = f"{name}_bias"
        if shortcut is not None:
            if i8:  # i8 shortcut (identity, or the requantized downsample) -> accumulator domain
                nodes.append(GraphNode(f"{name}_sc", "cast", [shortcut[0]], {"dtype": "i32"}))
                nodes.append(GraphNode(f"{name}_scs", "scale", [f"{name}_sc"],
                                       {"scale": float(round(4.6 * np.sqrt(cin * k * k)))}))
                nodes.append(GraphNode(f"{name}_add", "add", [y, f"{name}_scs"]))
            else:
                nodes.append(GraphNode(f"{name}_add", "add", [y, shortcut[0]]))
            y = f"{name}_add"
        if relu:
            nodes.append(GraphNode(f"{name}_relu", "relu", [y]))
            y = f"{name}_relu"
        if i8:
            # wider accumulator spread with a shortcut added / without relu
            spread = 4.0 if relu and shortcut is None else 5.5
            mult = max(1, int(round(65536.0 / (spread * np.sqrt(cin * k * k)))))
            nodes.append(GraphNode(f"{name}_q", "requantize", [y],
                                   {"multiplier": mult, "shift": 16}))
            y = f"{name}_q"
        return y

    x = inp("x", (batch, 3, image, image))
    y = conv("conv1", x, 3, width, 7, 2)
    if maxpool:
        nodes.append(GraphNode("pool1", "max_pool2d", [y],
                               {"kernel": [3, 3], "strides": [2, 2], "padding": [1, 1]}))
        y = "pool1"
    cin = width
    for stage, (cout, stride) in enumerate([(width, 1), (2 * width, 2), (4 * width, 2),
                                            (8 * width, 2)], start=1):
        for blk in range(2):
            s = stride if blk == 0 else 1
            pre = f"l{stage}_{blk}"
            sc = (y, True)
            if s != 1 or cin != cout:
                sc = (conv(f"{pre}_ds", y, cin, cout, 1, s, relu=False), False)
            h = conv(f"{pre}_a", y, cin, cout, 3, s)
            y = conv(f"{pre}_b", h, cout, cout, 3, 1, shortcut=sc)
            cin = cout
    if not head:
        g = ComputeGraph(nodes, [y])
        g.validate()
        return g
    if maxpool:
        nodes.append(GraphNode("gap", "global_avg_pool", [y]))
        nodes.append(GraphNode("flat", "flatten", ["gap"]))
        feat = "flat"
    else:
        nodes.append(GraphNode("gap_w", "sum", [y], {"axis": 3}))
        nodes.append(GraphNode("gap_h", "sum", ["gap_w"], {"axis": 2}))
        hw = image // 32
        nodes.append(GraphNode("gap", "scale", ["gap_h"], {"scale": 1.0 / (hw * hw)}))
        feat = "gap"
    wfc = inp("w_fc", (cin, num_classes))
    bfc = inp("b_fc", (num_classes,))
    nodes.append(GraphNode("fc", "matmul", [feat, wfc]))
    nodes.append(GraphNode("logits", "bias_add", ["fc", bfc]))
    g = ComputeGraph(nodes, ["logits"])
    g.validate()
    return g


def int8_resnet18_params(g, seed: int = 0):
    """Synthetic operands of resnet18_graph(dtype="i8"): x in [-32, 32],
    weights in [-8, 8], biases in [-100, 100] (i32). Returns (feeds, params)."""
    rng = np.random.default_rng(seed)
    feeds, params = {}, {}
    for n in g.nodes:
        if n.op != "input":
            continue
        shp = n.out_type.shape
        if n.id == "x":
            feeds["x"] = rng.integers(-32, 33, shp, dtype=np.int8)
        elif n.id.startswith("w_"):
            params[n.id] = rng.integers(-8, 9, shp, dtype=np.int8)
        else:
            params[n.id] = rng.integers(-100, 101, shp, dtype=np.int32)
    return feeds, params


# Conv GFLOP per image of resnet18_graph (1.8136 GMAC
# conv + 0.512 MMAC FC = 3.628 GFLOP/img).
RESNET18_GFLOP_PER_IMAGE = 3.628
