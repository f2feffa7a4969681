#!/usr/bin/env python3
"""Tunes the bench's per-layer knobs with the ML tuner (pairwise-rank GBT +
simulated annealing, tuner.tune) and writes them into a knob file in
bench.py's format {precision: {layer: knobs}} -- the file the batch-64
parity tests run (tests/test_bench_parity.py).

usage: tune_knobs.py PRECISION[,PRECISION..] OUT.json [budget] [batch]"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1802_04799_b200.device import make_desc  # noqa: E402
from paper_1802_04799_b200.tuner import conv_space, tune  # noqa: E402
from paper_1802_04799_b200.workloads import RESNET18_CONVS, resnet_layer  # noqa: E402

precs = sys.argv[1].split(",")
out = sys.argv[2]
budget = int(sys.argv[3]) if len(sys.argv) > 3 else 24
batch = int(sys.argv[4]) if len(sys.argv) > 4 else 64
knobs = json.load(open(out)) if os.path.exists(out) else {}
report = {}
for prec in precs:
    knobs.setdefault(prec, {})
    for n in RESNET18_CONVS:
        sp = conv_space(f"{n}_b{batch}_{prec}", make_desc(resnet_layer(n, batch), prec))
        t0 = time.time()
        res = tune(sp, budget=min(budget, sp.size()), batch_size=8, method="ml", repeats=5,
                   full=True)
        best = res.best
        knobs[prec][n] = best.config if best else {}
        report[f"{prec}/{n}"] = {"space": sp.size(), "trials": len(res.trials),
                                 "best_us": round(best.cost, 2) if best else None,
                                 "knobs": knobs[prec][n], "seconds": round(time.time() - t0, 1)}
        print(json.dumps({f"{prec}/{n}": report[f"{prec}/{n}"]}), flush=True)
with open(out, "w") as f:
    json.dump(knobs, f, indent=1)
