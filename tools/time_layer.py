"""Median device time of one fused layer (L2 flushed between launches):
python tools/time_layer.py LAYER BATCH COMPUTE ['knobs-json'] [reps]."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from bench_workloads import _flushed_launch_us  # noqa: E402
from paper_1802_04799_b200.device import DeviceConv  # noqa: E402
from paper_1802_04799_b200.workloads import mobilenet_layer, resnet_layer  # noqa: E402

name, batch, compute = sys.argv[1], int(sys.argv[2]), sys.argv[3]
knobs = json.loads(sys.argv[4]) if len(sys.argv) > 4 else {}
wl = mobilenet_layer(name, batch) if name.startswith("D") else resnet_layer(name, batch)
layer = DeviceConv(wl, compute=compute, knobs=knobs or None)
stream = torch.cuda.Stream()
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
us = _flushed_launch_us(lambda: layer.launch(stream), flush, stream)
print(json.dumps({"layer": name, "us": round(us, 2), "batch": batch, "compute": compute, "knobs": knobs,
                  "env": {k: v for k, v in os.environ.items() if k.startswith("TEC_SM100")}}))
