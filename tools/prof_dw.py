"""Per-layer, per-variant depthwise kernel times (MobileNet D1-D9, batch 64).

For each layer and each kernel variant of dw_space (unroll 2 / 4: the 3x3
column-streaming kernel, 8: the TMA-tiled kernel) prints the L2-flushed
device time from bench_workloads._flushed_launch_us and the achieved GB/s on
the algorithmic bytes. Usage: python tools/prof_dw.py [--compute bf16|f32]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch

    from bench_workloads import _flushed_launch_us
    from paper_1802_04799_b200.device import DeviceConv
    from paper_1802_04799_b200.workloads import MOBILENET_DW, mobilenet_layer
    ap = argparse.ArgumentParser()
    ap.add_argument("--compute", default="bf16")
    ap.add_argument("--batch", type=int, default=64)
    ap.add_argument("--layers", default=",".join(MOBILENET_DW))
    ap.add_argument("--unrolls", default="2,4,8")
    a = ap.parse_args()
    unrolls = [int(u) for u in a.unrolls.split(",")]
    stream = torch.cuda.Stream()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    rows = []
    for i, n in enumerate(MOBILENET_DW):
        if n not in a.layers.split(","):
            continue
        row = {"layer": n}
        for u in unrolls:
            l = DeviceConv(mobilenet_layer(n, a.batch), compute=a.compute, device=0, seed=i,
                           out_dtype=0 if a.compute == "f32" else None, knobs={"unroll": u})
            for _ in range(3):
                l.launch(stream)
            torch.cuda.synchronize()
            us = _flushed_launch_us(lambda l=l: l.launch(stream), flush, stream)
            row[f"u{u}_us"] = round(us, 2)
            row[f"u{u}_gbs"] = round(l.algorithmic_bytes() / us / 1e3, 1)
            del l
        print(json.dumps(row), flush=True)
        rows.append(row)
    best = sum(min(r[f"u{u}_us"] for u in unrolls) for r in rows)
    print(json.dumps({"sum_best_us": round(best, 2)}))


if __name__ == "__main__":
    main()
