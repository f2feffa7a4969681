"""Per-layer wall time of the bench's e2e leg (tec_eval_fused_conv, host
NCHW f32 buffers, pinned) against each layer's PCIe bound
max(up / 45, down / 53, both / duplex) GB/s: python tools/e2e_layers.py [batch]."""
import ctypes as C
import json
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_1802_04799_b200 import _abi  # noqa: E402
from paper_1802_04799_b200.workloads import resnet_layer  # noqa: E402

lib = _abi.load()
duplex = bench.pcie_duplex_gbs()
g = torch.Generator().manual_seed(7)
BATCH = int(sys.argv[1]) if len(sys.argv) > 1 else 64
for name in bench.LAYERS:
    wl = resnet_layer(name, BATCH)
    x = (torch.rand((wl.n, wl.c, wl.h, wl.w), generator=g) * 2 - 1).pin_memory()
    w = (torch.rand((wl.k, wl.c, wl.r, wl.s), generator=g) * 2 - 1).pin_memory()
    b = (torch.rand((wl.k,), generator=g) * 2 - 1).pin_memory()
    y = torch.empty((wl.n, wl.k, wl.oh, wl.ow)).pin_memory()
    d = _abi.ConvDesc(n=wl.n, c=wl.c, h=wl.h, w=wl.w, k=wl.k, r=wl.r, s=wl.s, stride_h=wl.stride,
                      stride_w=wl.stride, pad_h=wl.pad, pad_w=wl.pad, depthwise=0,
                      compute=_abi.COMPUTE_F32TC)
    e = _abi.Epilogue()
    e.n_ops, e.ops[0], e.ops[1], e.bias = 2, _abi.EPI_BIAS, _abi.EPI_RELU, b.data_ptr()
    kn = _abi.Knobs()

    def one():
        _abi.check(lib.tec_eval_fused_conv(C.byref(d), C.byref(e), C.byref(kn), x.data_ptr(),
                                           w.data_ptr(), y.data_ptr(), 0))
    one()
    ts = []
    for _ in range(5):
        t0 = time.perf_counter()
        one()
        ts.append(time.perf_counter() - t0)
    t = sorted(ts)[2]
    up = (x.numel() + w.numel() + b.numel()) * 4
    down = y.numel() * 4
    bound = max(up / 45e9, down / 53e9, (up + down) / (duplex * 1e9))
    print(json.dumps({"layer": name, "ms": round(t * 1e3, 3), "bound_ms": round(bound * 1e3, 3),
                      "frac": round(bound / t, 3), "up_mb": round(up / 1e6, 1),
                      "down_mb": round(down / 1e6, 1)}), flush=True)
