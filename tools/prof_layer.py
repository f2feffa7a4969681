"""Eager launches of one layer (for TEC_SM100_PROFILE=1 wait breakdowns, which
synchronise and cannot run under graph capture):
python tools/prof_layer.py LAYER BATCH COMPUTE 'knobs-json' [reps]."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1802_04799_b200.device import DeviceConv  # noqa: E402
from paper_1802_04799_b200.workloads import mobilenet_layer, resnet_layer  # noqa: E402

name, batch, compute = sys.argv[1], int(sys.argv[2]), sys.argv[3]
knobs = json.loads(sys.argv[4]) if len(sys.argv) > 4 else {}
reps = int(sys.argv[5]) if len(sys.argv) > 5 else 3
wl = mobilenet_layer(name, batch) if name.startswith("D") else resnet_layer(name, batch)
layer = DeviceConv(wl, compute=compute, knobs=knobs or None)
for _ in range(reps):
    layer.launch()
torch.cuda.synchronize()
