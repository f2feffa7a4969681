import sys, time, torch, numpy as np
sys.path.insert(0, __import__('os').path.dirname(__import__('os').path.dirname(__import__('os').path.abspath(__file__))))
import bench_workloads as bw
from paper_1802_04799_b200.executor import DeviceGraph
from paper_1802_04799_b200.workloads import resnet18_graph
import argparse
B = int(sys.argv[1]) if len(sys.argv) > 1 else 256
g = resnet18_graph(B)
class A: no_tune=False
knobs = bw._tune_graph_convs(g, 0, A())
dg = DeviceGraph(g, compute="bf16", knobs=knobs)
rng = np.random.default_rng(0)
params = {n.id: (rng.standard_normal(n.out_type.shape) * 0.05).astype(np.float32) for n in g.nodes if n.op == "input" and n.id != "x"}
dg.bind_params(params)
dg.set_feed("x", rng.uniform(-1, 1, (B, 3, 224, 224)).astype(np.float32))
s = torch.cuda.Stream()
for _ in range(3):
    for i in range(len(dg.steps)): dg.launch_step(i, s)
torch.cuda.synchronize()
names = []
for n in dg.g.nodes:
    if n.op != "input": names.append(n.id)
ev = []
with torch.cuda.stream(s):
    for i, st in enumerate(dg.steps):
        a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
        a.record(s); dg.launch_step(i, s); b.record(s); ev.append((a, b))
torch.cuda.synchronize()
ts = [a.elapsed_time(b) * 1e3 for a, b in ev]
print("steps", len(dg.steps), "total us", sum(ts))
KIND = {1: "conv", 2: "maxpool", 3: "avgpool", 4: "pack", 5: "unpack", 6: "to_nhwc", 7: "dw"}
for i, t in enumerate(ts):
    st = dg.steps[i]
    d = st.conv
    desc = (f"c{d.c} {d.h}x{d.w} -> k{d.k} r{d.r} s{d.stride_h} epi{st.epi.n_ops}"
            if st.kind in (1, 4, 7) else "")
    print(i, KIND.get(st.kind, st.kind), round(t, 1), desc)
