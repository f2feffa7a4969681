"""Per-launch times of the ResNet-18 executor plan (eager launches, CUDA
events): python tools/prof_resnet.py [batch] [bf16|f32tc|i8]."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench_workloads as bw  # noqa: E402
from paper_1802_04799_b200.executor import DeviceGraph  # noqa: E402
from paper_1802_04799_b200.workloads import int8_resnet18_params, resnet18_graph  # noqa: E402

B = int(sys.argv[1]) if len(sys.argv) > 1 else 256
COMPUTE = sys.argv[2] if len(sys.argv) > 2 else "bf16"
i8 = COMPUTE == "i8"
g = resnet18_graph(B, head=False, dtype="i8") if i8 else resnet18_graph(B)


class A:
    no_tune = False


knobs = bw._tune_graph_convs(g, 0, A(), COMPUTE)
dg = DeviceGraph(g, compute=COMPUTE, knobs=knobs)
rng = np.random.default_rng(0)
if i8:
    feeds, params = int8_resnet18_params(g, 0)
else:
    params = {n.id: (rng.standard_normal(n.out_type.shape) * 0.05).astype(np.float32)
              for n in g.nodes if n.op == "input" and n.id != "x"}
    feeds = {"x": rng.uniform(-1, 1, (B, 3, 224, 224)).astype(np.float32)}
dg.bind_params(params)
dg.set_feed("x", feeds["x"])
s = torch.cuda.Stream()
for _ in range(3):
    for i in range(len(dg.steps)):
        dg.launch_step(i, s)
torch.cuda.synchronize()
ev = []
with torch.cuda.stream(s):
    for i, st in enumerate(dg.steps):
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record(s)
        dg.launch_step(i, s)
        b.record(s)
        ev.append((a, b))
torch.cuda.synchronize()
ts = [a.elapsed_time(b) * 1e3 for a, b in ev]
print("steps", len(dg.steps), "total us", round(sum(ts), 1))
KIND = {1: "conv", 2: "maxpool", 3: "avgpool", 4: "pack", 5: "unpack", 6: "to_nhwc", 7: "dw",
        8: "pack_nhwc", 9: "elemwise"}
by = {}
for i, t in enumerate(ts):
    st = dg.steps[i]
    d = st.conv
    k = KIND.get(st.kind, st.kind)
    by[k] = by.get(k, 0.0) + t
    desc = (f"c{d.c} {d.h}x{d.w} -> k{d.k} r{d.r} s{d.stride_h} epi{st.epi.n_ops}"
            if st.kind in (1, 4, 7) else (f"n={st.elem.count} ops={st.elem.n_ops}" if st.kind == 9 else ""))
    print(i, k, round(t, 1), desc)
print("by kind (us):", {k: round(v, 1) for k, v in by.items()})
