#!/usr/bin/env python3
"""Launch one fused layer a few times (for ncu captures).
usage: run_layer.py LAYER BATCH COMPUTE ['knobs-json'] [launches]"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1802_04799_b200.device import DeviceConv  # noqa: E402
from paper_1802_04799_b200.workloads import mobilenet_layer, resnet_layer  # noqa: E402

name, batch, compute = sys.argv[1], int(sys.argv[2]), sys.argv[3]
knobs = json.loads(sys.argv[4]) if len(sys.argv) > 4 else {}
n = int(sys.argv[5]) if len(sys.argv) > 5 else 3
wl = mobilenet_layer(name, batch) if name.startswith("D") else resnet_layer(name, batch)
l = DeviceConv(wl, compute=compute, knobs=knobs or None)
for _ in range(n):
    l.launch()
torch.cuda.synchronize()
print("ok", name, batch, compute)
