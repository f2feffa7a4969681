"""Median device time (L2 flushed) of several (layer, compute, knobs) cases in
one process: python tools/sweep_layers.py BATCH 'json list of [layer, compute, knobs]'.
A case the lowering rejects prints its error instead of a time."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from bench_workloads import _flushed_launch_us  # noqa: E402
from paper_1802_04799_b200.device import DeviceConv  # noqa: E402
from paper_1802_04799_b200.workloads import mobilenet_layer, resnet_layer  # noqa: E402

batch = int(sys.argv[1])
cases = json.loads(sys.argv[2])
stream = torch.cuda.Stream()
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for name, compute, knobs in cases:
    wl = mobilenet_layer(name, batch) if name.startswith("D") else resnet_layer(name, batch)
    try:
        layer = DeviceConv(wl, compute=compute, knobs=knobs or None)
        us = _flushed_launch_us(lambda: layer.launch(stream), flush, stream)
        print(json.dumps({"layer": name, "compute": compute, "knobs": knobs, "us": round(us, 2)}), flush=True)
        del layer
    except Exception as e:  # noqa: BLE001 -- report and continue the sweep
        print(json.dumps({"layer": name, "compute": compute, "knobs": knobs, "error": str(e)[:160]}), flush=True)
