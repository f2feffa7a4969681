"""The reference's headline workloads.

ResNet-18 conv C1-C12 and MobileNet depthwise D1-D9, with pad = k // 2
(the reference pads symmetrically, R/src/ops.cpp:125). Algorithmic work
per launch follows BASELINE.md: FLOPs = 2*N*OC*OH*OW*IC*KH*KW (depthwise:
IC := 1); compulsory bytes = every operand + the output once
(R/src/loop_ir.cpp:524-534).
"""
from __future__ import annotations

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
