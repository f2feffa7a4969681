"""Summarise an ncu launch-list CSV of a bench.py run into profiles/.

    ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
        --clock-control none --csv --log-file launches.csv \
        python bench.py --steps 1 --warmup 3 --knobs-in profiles/<round>_tuned_knobs.json \
        --no-e2e --no-cpu-baseline
    python profiles/ncu_to_json.py launches.csv profiles/<round>_launches_bench_step.json \
        [--traffic profiles/traffic.json]

Takes the last 12 launches of the last run of >= 12 back-to-back fused-conv
launches -- the CUDA-graph step replays (C1..C12 in bench order; the
per-layer timing loop interleaves L2-flush kernels, so it never forms such
a run). ncu serialises and cold-starts every launch and records per-launch duration, share of the step and DRAM
bytes. --traffic also writes {"dram_bytes_per_step": ...}, which bench.py
reports as roofline.traffic.
"""
import csv
import json
import sys

LAYERS = [f"C{i}" for i in range(1, 13)]


def load(path):
    rows = []
    with open(path) as f:
        lines = [l for l in f if l.startswith('"')]
    for r in csv.DictReader(lines):
        rows.append(r)
    kernels = {}
    order = []
    for r in rows:
        key = (r["ID"], r["Kernel Name"])
        if key not in kernels:
            kernels[key] = {}
            order.append(key)
        v = r["Metric Value"].replace(",", "")
        unit = r.get("Metric Unit", "")
        val = float(v)
        if unit in ("usecond",):
            val *= 1e3
        elif unit in ("msecond",):
            val *= 1e6
        elif unit in ("Kbyte", "KB"):
            val *= 1e3
        elif unit in ("Mbyte", "MB"):
            val *= 1e6
        elif unit in ("Gbyte", "GB"):
            val *= 1e9
        kernels[key][r["Metric Name"]] = val
    return [(k[1], kernels[k]) for k in order]


def short(name):
    name = name.replace("tec_sm100::", "").replace("(anonymous namespace)::", "")
    name = name.replace("MmaKind::kF16", "0").replace("MmaKind::kI8", "2").replace("MmaKind::kTF32", "1")
    return name.split("(")[0]


def main():
    src, dst = sys.argv[1], sys.argv[2]
    traffic_path = sys.argv[sys.argv.index("--traffic") + 1] if "--traffic" in sys.argv else None
    all_k = load(src)
    runs, cur = [], []
    for n, m in all_k:
        if "conv_" in n:
            cur.append((n, m))
        else:
            if len(cur) >= 12:
                runs.append(cur)
            cur = []
    if len(cur) >= 12:
        runs.append(cur)
    if not runs:
        raise SystemExit(f"no run of 12 back-to-back conv launches in {src}")
    step = runs[-1][-12:]
    total = sum(m.get("gpu__time_duration.sum", 0.0) for _, m in step)
    out = {
        "source": "ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum "
                  "--clock-control none; one CUDA-graph step of bench.py (12 fused-conv launches, "
                  "one per layer), cold-cache and serialised by ncu",
        "launches": [],
        "total_ns": total,
    }
    dram = 0.0
    for layer, (n, m) in zip(LAYERS, step):
        ns = m.get("gpu__time_duration.sum", 0.0)
        rd, wr = m.get("dram__bytes_read.sum"), m.get("dram__bytes_write.sum")
        dram += (rd or 0) + (wr or 0)
        out["launches"].append({"layer": layer, "kernel": short(n), "ns": ns,
                                "share": round(ns / total, 4) if total else None,
                                "dram_read_bytes": rd, "dram_write_bytes": wr})
    out["dram_bytes_per_step"] = dram
    with open(dst, "w") as f:
        json.dump(out, f, indent=1)
    if traffic_path:
        with open(traffic_path, "w") as f:
            json.dump({"dram_bytes_per_step": dram, "from": dst}, f, indent=1)
    print(f"{len(step)} launches, {total / 1e3:.1f} us total, {dram / 1e6:.1f} MB DRAM")


if __name__ == "__main__":
    main()
