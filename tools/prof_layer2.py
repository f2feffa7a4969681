"""Per-layer kernel time with sub-microsecond resolution: CUDA-graph replay of
[flush, layer] x R minus [flush] x R (event resolution here is ~2 us).
usage: prof_layer2.py LAYER[,LAYER..] BATCH 'knobs-json-or-list' [R]
(TEC_COMPUTE=bf16|f32tc|i8 selects the arithmetic, default bf16)"""
import json
import sys

import torch

sys.path.insert(0, __import__('os').getcwd())
from paper_1802_04799_b200.device import DeviceConv
from paper_1802_04799_b200.workloads import resnet_layer

names = sys.argv[1].split(',')
batch = int(sys.argv[2])
kspec = json.loads(sys.argv[3]) if len(sys.argv) > 3 else {}
R = int(sys.argv[4]) if len(sys.argv) > 4 else 10
variants = kspec if isinstance(kspec, list) else [kspec]
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
stream = torch.cuda.Stream()


def graph_of(fn):
    with torch.cuda.stream(stream):
        fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=stream):
        fn()
    return g


def timed(g, reps=5):
    ts = []
    for _ in range(reps):
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(stream):
            a.record(stream)
            g.replay()
            b.record(stream)
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) * 1e3)
    ts.sort()
    return ts[len(ts) // 2]


def fl():
    for _ in range(R):
        flush.zero_()


gf = graph_of(fl)
base = timed(gf)
for n in names:
    for kn in variants:
        l = DeviceConv(resnet_layer(n, batch), knobs=kn or None,
                       compute=__import__('os').environ.get("TEC_COMPUTE", "bf16"))
        for _ in range(3):
            l.launch(stream)

        def body(l=l):
            for _ in range(R):
                flush.zero_()
                l.launch(stream)
        g = graph_of(body)
        t = (timed(g) - base) / R
        print(f"{n} {json.dumps(kn)} us {t:.2f} tflops {l.wl.flops / (t * 1e-6) / 1e12:.0f}", flush=True)
        del g, l
