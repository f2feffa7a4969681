#!/usr/bin/env python3
"""bench.py -- the headline benchmark (BASELINE.json `metric`):

  "ResNet-18 conv C1-C12 TFLOP/s (% roofline); ResNet-18 img/s at 1/2/4/8 GPU"
  on configs[1]: all twelve ResNet-18 conv workloads at
  batch 64, each a fused [conv2d, bias_add, relu] node (the group fuse_pass
  builds, R/src/graph_passes.cpp:240-244) run as ONE sm_100a kernel through
  the C ABI.

The headline `value` is at the REFERENCE'S precision: f32 in, f32 out
(compute "f32tc", conv_f32tc.cu -- f32 on the tcgen05 tensor cores, held to
the reference comparator's 1e-4, tests/test_conv_gpu.py + test_bench_parity.py).
The same line carries, as named sub-results measured in the same run:
  precisions.bf16  bf16 in / f32 accumulate / bf16 out (stated tolerance)
  precisions.i8    int8 x int8 -> i32, bit-exact (configs[4], the VDLA path),
                   against an int8 peak measured in this run
  resnet18         ResNet-18 inference, global batch 256 sharded over the
                   ranks (configs[3], strong scaling), img/s + e2e img/s
  depthwise        MobileNet D1-D9 depthwise + bias + relu, batch 64, bf16 and
                   f32 (configs[2]), GB/s against the HBM roofline

One "step" = the 12 fused layers once over one batch of synthetic inputs
(reference value distributions, random-init weights), inputs resident in HBM.
`value` = total algorithmic FLOPs (2*N*OC*OH*OW*IC*KH*KW per layer) / time.
Knobs come from profiles/tuned_knobs.json -- the SAME file the batch-64
parity tests (tests/test_bench_parity.py) run, so every knob set the bench
times is covered by a parity test; other knob files are refused unless
--allow-untested-knobs.

Multi-GPU: `--gpus N` without torchrun re-launches itself under
torch.distributed.run (N ranks, 127.0.0.1). The single-operator configs are
replicas: value = FLOPs of all ranks / max-over-ranks time
("scaling": "weak"); ResNet-18 is batch-sharded (strong scaling).
`--cpu-dry-run` runs the same rank plumbing on gloo without a GPU.

`--impl reference` runs the reference's own CPU implementation (the tec
library compiled from /root/reference sources into oracle/_ref by
oracle/Makefile) on a bounded sample of the same workload.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

from paper_1802_04799_b200.workloads import RESNET18_CONVS, resnet_layer  # noqa: E402

METRIC = "ResNet-18 conv C1\u2013C12 TFLOP/s (% roofline); ResNet-18 img/s at 1/2/4/8 GPU"
LAYERS = list(RESNET18_CONVS)
REF_DRIVER = os.path.join(REPO, "oracle", "_ref", "ref_driver")


def load_peaks():
    p = os.path.join(REPO, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            j = json.load(f)
        return (float(j["bf16_tflops"]), float(j["hbm_gbs"]),
                float(j.get("bf16_tflops_sustained", j["bf16_tflops"])), "measured")
    except Exception:
        return 1590.0, 6650.0, 1400.0, "fallback"


# ------------------------------------------------------------ CPU reference
def _ref_chunks(rows=1, chunk_oc=None):
    """Bounded sample of the workload: for every layer, `rows` output rows of
    one image at full width and depth, split into output-channel chunks so
    the work spreads over all host cores."""
    jobs = []
    for name in LAYERS:
        hw, c, k, r, s = RESNET18_CONVS[name]
        per = chunk_oc or max(8, min(k, (1 << 20) // max(1, c * r * r * (hw // s))))
        for oc0 in range(0, k, per):
            jobs.append((name, c, hw, hw, min(per, k - oc0), r, s, r // 2, rows))
    return jobs


def _ref_one(job, seed):
    name, c, h, w, oc, r, s, p, rows = job
    out = subprocess.run([REF_DRIVER, "bench", "conv2d", str(c), str(h), str(w), str(oc),
                          str(r), str(s), str(p), str(rows), str(seed)],
                         capture_output=True, text=True, check=True)
    return json.loads(out.stdout)


def run_reference_sample(threads, seed=0):
    """Runs the sample on `threads` concurrent reference processes; returns
    (flops, wall_seconds, description)."""
    from concurrent.futures import ThreadPoolExecutor
    jobs = _ref_chunks()
    t0 = time.perf_counter()
    with ThreadPoolExecutor(max_workers=threads) as ex:
        res = list(ex.map(lambda j: _ref_one(j, seed), jobs))
    wall = time.perf_counter() - t0
    flops = sum(2 * r["macs"] for r in res)
    desc = (f"reference tec eval_graph_node(fused conv2d+bias_add+relu) on 1 output row of "
            f"each of C1-C12 (batch 1, full width/channels, {len(jobs)} OC chunks), "
            f"{threads} concurrent processes; f32")
    return flops, wall, desc


def run_port_sample(threads, seed=0):
    """Fallback when oracle/_ref is absent: the C restatement (oracle/)."""
    import numpy as np
    from oracle.oracle_api import fused_conv
    rng = np.random.default_rng(seed)
    flops = 0
    t0 = time.perf_counter()
    for name in LAYERS:
        hw, c, k, r, s = RESNET18_CONVS[name]
        hs = r  # one output row
        x = rng.uniform(-1, 1, (1, c, hs, hw)).astype(np.float32)
        w = rng.uniform(-1, 1, (k, c, r, r)).astype(np.float32)
        b = rng.uniform(-1, 1, (k,)).astype(np.float32)
        y = fused_conv("conv2d", x, w, (s, s), (r // 2, r // 2),
                       [("bias_add", b), ("relu",)], threads=threads)
        flops += 2 * y.size * c * r * r
    return flops, time.perf_counter() - t0, f"oracle C port, 1 row per layer, {threads} threads"


def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for ln in f:
                if ln.startswith("model name"):
                    return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


# oracle/Makefile builds the reference with its own CMake default (Release)
REF_FLAGS = "g++ -std=c++20 -O3 -DNDEBUG (the reference's CMake Release flags, oracle/Makefile)"


def cpu_baseline_block(threads):
    if os.path.exists(REF_DRIVER):
        flops, wall, desc = run_reference_sample(threads)
        kind = "reference"
    else:
        flops, wall, desc = run_port_sample(threads)
        kind = "port"
    return {"value": flops / wall / 1e12, "unit": "TFLOP/s", "cores": threads,
            "kind": kind, "sample": desc, "sample_flops": flops,
            "sample_seconds": round(wall, 3), "cpu_model": cpu_model(),
            "compiler_flags": REF_FLAGS if kind == "reference" else "gcc -O3 -ffp-contract=off"}


def impl_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    threads = os.cpu_count() or 1
    if not os.path.exists(REF_DRIVER):
        kind = "port"
    else:
        kind = "reference"
    vals = []
    sample = None
    # each step is a ~1 s bounded CPU sample: at most 20 timed steps keep the
    # reference arm within a few minutes whatever K the caller asks for
    steps = min(args.steps, 20)
    for i in range(args.warmup + steps):
        if kind == "reference":
            flops, wall, sample = run_reference_sample(threads, seed=i)
        else:
            flops, wall, sample = run_port_sample(threads, seed=i)
        if i >= args.warmup:
            vals.append((flops, wall))
    tot_f = sum(v[0] for v in vals)
    tot_t = sum(v[1] for v in vals)
    value = tot_f / tot_t / 1e12
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "TFLOP/s",
        "n_gpus": args.gpus, "steps": steps, "steps_requested": args.steps, "warmup": args.warmup,
        "ms_per_step": tot_t / max(1, len(vals)) * 1e3, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {"workload": "C1-C12 fused conv2d+bias_add+relu (bounded CPU sample)",
                   "global_batch": 1, "parallelism": "process-sharded host cores"},
        "cpu_baseline": {"value": value, "unit": "TFLOP/s", "cores": threads,
                         "kind": kind, "sample": sample, "cpu_model": cpu_model(),
                         "compiler_flags": REF_FLAGS if kind == "reference" else
                         "gcc -O3 -ffp-contract=off"},
        "e2e": {"value": value, "unit": "TFLOP/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------ clocks sampler
class ClockSampler:
    """Samples SM clock and throttle reasons through NVML every ~5 ms while
    the timed region runs (nvidia-smi's 100 ms loop is longer than a step)."""
    REASONS = {"hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20,
               "hw_thermal_slowdown": 0x40, "sw_power_cap": 0x4}

    def __init__(self, device):
        self.device = device
        self.sm, self.reasons, self.max_mhz = [], set(), None
        self._stop = threading.Event()
        self._ready = threading.Event()  # NVML initialised, first sample taken

    def _run(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            h = pynvml.nvmlDeviceGetHandleByIndex(self.device)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)
            self._ready.set()
            while not self._stop.is_set():
                self.sm.append(pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM))
                r = pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)
                for name, bit in self.REASONS.items():
                    if r & bit:
                        self.reasons.add(name)
                time.sleep(0.001)
        except Exception as e:  # pragma: no cover
            self.error = repr(e)
        finally:
            self._ready.set()

    def __enter__(self):
        self.t = threading.Thread(target=self._run, daemon=True)
        self.t.start()
        # NVML start-up can take longer than a short timed region: start the
        # region only once the sampler runs
        self._ready.wait(timeout=10.0)
        return self

    def __exit__(self, *a):
        self._stop.set()
        self.t.join(timeout=2)

    def summary(self):
        if not self.sm:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": [], "samples": 0,
                    "error": getattr(self, "error", None)}
        return {"sm_mhz": statistics.median(self.sm), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.sm)}


# ------------------------------------------------------------ our arm
KNOBS_FILE = os.path.join(REPO, "profiles", "tuned_knobs.json")
# element bytes of the algorithmic operands (x, w | y) per arithmetic
PRECISIONS = {"f32tc": (4, 4), "bf16": (2, 2), "i8": (1, 4)}


def load_knobs(path=KNOBS_FILE):
    if path and os.path.exists(path):
        with open(path) as f:
            return json.load(f)
    return {}


def measure_int8_peak():
    """Dense int8 tensor-core peak of THIS GPU: best of 10 cuBLASLt int8
    GEMMs (torch._int_mm, 8192^3, 2*N^3 ops). None when unavailable."""
    import torch
    try:
        n = 8192
        a = torch.randint(-8, 8, (n, n), dtype=torch.int8, device="cuda")
        b = torch.randint(-8, 8, (n, n), dtype=torch.int8, device="cuda").t()
        for _ in range(3):
            torch._int_mm(a, b)
        torch.cuda.synchronize()
        best = None
        for _ in range(10):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            torch._int_mm(a, b)
            e1.record()
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1)
            best = ms if best is None else min(best, ms)
        del a, b
        return 2 * n ** 3 / (best * 1e-3) / 1e12
    except Exception:
        return None


def measure_step(compute, knobs, batch, local, rank, world, steps, warmup, peak, hbm_gbs,
                 sampler=None):
    """Times the 12-layer step at one arithmetic: K CUDA-graph replays
    between barriers (max over ranks), then each layer's L2-flushed kernel
    time. Returns the step's numbers and its per-layer roofline table."""
    import torch
    import torch.distributed as dist

    from paper_1802_04799_b200.device import DeviceConv
    in_b, out_b = PRECISIONS[compute]
    layers = [DeviceConv(resnet_layer(n, batch), compute=compute, device=local,
                         seed=1000 * rank + i, knobs=knobs.get(n) or None)
              for i, n in enumerate(LAYERS)]
    flops = [l.wl.flops for l in layers]
    step_flops = sum(flops)
    stream = torch.cuda.Stream()
    torch.cuda.synchronize()

    def step():
        for l in layers:
            l.launch(stream)

    with torch.cuda.stream(stream):
        for _ in range(max(1, warmup)):
            step()
    torch.cuda.synchronize()
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph, stream=stream):
        step()
    torch.cuda.synchronize()
    for _ in range(2):
        graph.replay()
    torch.cuda.synchronize()

    # ---- timed region: K graph replays, events on the replay stream.
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    import contextlib
    with (sampler if sampler is not None else contextlib.nullcontext()):
        with torch.cuda.stream(stream):
            ev0.record(stream)
            for _ in range(steps):
                graph.replay()
            ev1.record(stream)
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    t = torch.tensor([ev0.elapsed_time(ev1)], device="cuda")
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    max_ms = float(t.item())
    value = world * step_flops * steps / (max_ms / 1e3) / 1e12

    # ---- per-layer kernel durations, L2 flushed before each launch. Event
    # timestamps here move in ~2 us steps, too coarse for one 6-45 us launch:
    # a CUDA graph of R x (flush, launch) is timed against R x flush alone
    # (median of 3 each) and the difference / R is the launch's device time.
    # The flush-only baseline is re-measured next to every layer
    # (bench_workloads._flushed_launch_us): one baseline taken before the
    # loop drifted with the clocks over the pass and ate the small layers.
    from bench_workloads import _flushed_launch_us
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    per_layer = []
    for l, fl in zip(layers, flops):
        us = _flushed_launch_us(lambda l=l: l.launch(stream), flush, stream)
        byts = l.wl.bytes(in_b, out_b)
        ai = fl / byts
        bound_tf = min(peak, ai * hbm_gbs / 1e3)
        achieved = fl / (us * 1e-6) / 1e12
        per_layer.append({
            "layer": l.wl.name, "knobs": knobs.get(l.wl.name) or {},
            "us": round(us, 2), "tflops": round(achieved, 1),
            "gflop": round(fl / 1e9, 3), "mbytes": round(byts / 1e6, 2),
            "ai_flop_per_byte": round(ai, 1),
            "bound": "tensor" if bound_tf >= peak else "hbm",
            "roof_tflops": round(bound_tf, 1), "frac_of_roof": round(achieved / bound_tf, 3),
        })
    kern_s = sum(p["us"] for p in per_layer) * 1e-6
    # attainable step time: every layer at its own min(peak, AI x HBM) roof
    roof_s = sum(p["gflop"] * 1e9 / (p["roof_tflops"] * 1e12) for p in per_layer)
    out = {"value": value, "ms_per_step": max_ms / steps, "step_flops": step_flops,
           "kernel_tflops": step_flops / kern_s / 1e12, "kernel_us": kern_s * 1e6,
           "frac_of_attainable": roof_s / kern_s, "layers": per_layer,
           "launches": len(layers) * steps}
    del graph, layers, flush
    torch.cuda.empty_cache()
    return out


def impl_ours(args):
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    peak_tf, hbm_gbs, peak_tf_sus, peak_src = load_peaks()
    batch = args.batch

    knobs_path = args.knobs_in or KNOBS_FILE
    knobs = load_knobs(knobs_path)
    knobs_src = os.path.relpath(knobs_path, REPO) if os.path.exists(knobs_path) else "library defaults"

    int8_peak = measure_int8_peak()
    peaks = {"f32tc": peak_tf / 6.0, "bf16": peak_tf,
             "i8": int8_peak if int8_peak else 2.0 * peak_tf}
    peak_notes = {
        "f32tc": f"MEASURED_PEAKS.json bf16_tflops ({peak_src}) / 6: every f32 multiply-add is "
                 "six bf16 tensor-core products (h*h, h*m, m*h, h*l, l*h, m*m)",
        "bf16": f"MEASURED_PEAKS.json bf16_tflops ({peak_src})",
        "i8": ("measured in this run: best of 10 cuBLASLt int8 GEMMs 8192^3 (torch._int_mm)"
               if int8_peak else "2 x bf16_tflops (no int8 GEMM available to measure)"),
    }
    headline = args.precision
    clk = ClockSampler(local)
    res = {}
    order = [headline] + [p for p in ("bf16", "i8", "f32tc") if p != headline and
                          p in args.also.split(",")]
    for prec in order:
        res[prec] = measure_step(prec, knobs.get(prec, {}), batch, local, rank, world,
                                 args.steps, args.warmup, peaks[prec], hbm_gbs,
                                 sampler=clk if prec == headline else None)
    h = res[headline]

    # ---- ResNet-18, global batch 256 sharded over the ranks (strong scaling)
    resnet = None
    if not args.no_resnet18:
        import bench_workloads
        rargs = argparse.Namespace(**vars(args))
        rargs.global_batch = args.global_batch or 256
        rargs.no_cpu_baseline = True
        rargs.steps = min(args.steps, 50)
        resnet = {}
        for rc in ("bf16", "f32tc", "i8"):
            rl = bench_workloads.resnet18_line(rargs, sys.modules[__name__], knobs_file=knobs_path,
                                               compute=rc)
            if rl is not None:
                resnet[rc] = {"img_s": rl["value"], "unit": "img/s",
                              "global_batch": rargs.global_batch, "n_gpus": rl["n_gpus"],
                              "ms_per_step": rl["ms_per_step"], "scaling": "strong",
                              "dtype": rl["dtype"], "e2e_img_s": rl["e2e"]["value"],
                              "roofline_frac": rl["roofline"]["frac"],
                              "config": rl["config"]["workload"]}
        resnet = resnet or None

    # ---- configs[2]: MobileNet D1-D9 depthwise + bias + relu, batch 64
    # (HBM-bound; GB/s against the HBM roofline), bf16 and f32
    depthwise = {}
    if not args.no_depthwise:
        import bench_workloads
        for dc in ("bf16", "f32"):
            dargs = argparse.Namespace(**vars(args))
            dargs.steps = min(args.steps, 100)
            dl = bench_workloads.depthwise_line(dargs, sys.modules[__name__], dc)
            if dl is not None:
                depthwise[dc] = {"value": dl["value"], "unit": "GB/s",
                                 "ms_per_step": dl["ms_per_step"], "roofline": dl["roofline"],
                                 "parity": "bit-identical to the oracle (tests/test_bench_parity.py)",
                                 "layers": dl["layers"]}

    # ---- e2e through the reference-facing host API (tec_eval_fused_conv):
    # pinned host NCHW f32 inputs -> H2D -> pack -> fused kernel -> unpack -> D2H.
    e2e = None
    if not args.no_e2e:
        e2e = run_e2e(args, batch, local, headline, world)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline_block(os.cpu_count() or 1)

    traffic, traffic_src = None, None
    tp = os.path.join(REPO, "profiles", "traffic.json")
    if os.path.exists(tp):
        try:
            tj = json.load(open(tp)).get(headline) or {}
            # the roofline covers the 12 launches of a step: their DRAM bytes
            # (ncu launch list of this same step, cold caches)
            traffic, traffic_src = tj.get("dram_bytes_per_step"), tj.get("source")
        except Exception:
            traffic = None

    def sub(prec):
        r = res[prec]
        unit = "TOPS" if prec == "i8" else "TFLOP/s"
        return {"value": round(r["value"], 2), "unit": unit, "dtype": prec,
                "ms_per_step": round(r["ms_per_step"], 4),
                "roofline": {"bound": "tensor", "achieved": round(r["kernel_tflops"], 1),
                             "peak": round(peaks[prec], 1), "unit": unit,
                             "frac": round(r["kernel_tflops"] / peaks[prec], 3),
                             "frac_of_attainable": round(r["frac_of_attainable"], 3),
                             "peak_source": peak_notes[prec]},
                "parity": {"f32tc": "1e-4 comparator vs the f32 oracle (tests/test_bench_parity.py)",
                           "bf16": "2e-3 comparator vs the oracle on bf16-rounded inputs",
                           "i8": "bit-exact vs the oracle"}[prec],
                "layers": r["layers"]}

    if rank == 0:
        dtype = {"f32tc": "f32", "bf16": "bf16", "i8": "i8"}[headline]
        line = {
            "metric": METRIC, "value": round(h["value"], 2),
            "unit": "TOPS" if headline == "i8" else "TFLOP/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(h["ms_per_step"], 4), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": dtype, "data": "synthetic",
            "config": {
                "workload": f"configs[1]: ResNet-18 C1-C12 fused conv2d+bias_add+relu, batch "
                            f"{batch} per GPU, " + {
                                "f32tc": "f32 in / f32 out (f32 on tcgen05: exact 3-way bf16 "
                                         "split, six products, RN-folded K chunks; 1e-4 parity)",
                                "bf16": "bf16 in / f32 accumulate / bf16 out",
                                "i8": "int8 in / i32 out (bit-exact)"}[headline],
                "global_batch": batch * world, "parallelism": f"replicas x{world} (no collective)",
                "l2": "step working set (all 12 layers) > 126 MB L2; per-layer timings "
                      "flush L2 (256 MB write) before each launch (graph of 10 x (flush, "
                      "launch) minus 10 x flush)",
                "timing": "CUDA graph of the 12 launches replayed K times; CUDA events on "
                          "the replay stream; max over ranks",
                "knobs": knobs_src,
            },
            "roofline": {
                "bound": "tensor", "achieved": round(h["kernel_tflops"], 1),
                "peak": round(peaks[headline], 1), "unit": "TFLOP/s",
                "frac": round(h["kernel_tflops"] / peaks[headline], 3),
                "frac_of_attainable": round(h["frac_of_attainable"], 3),
                "traffic": traffic, "traffic_source": traffic_src,
                "peak_source": peak_notes[headline],
                "kernel": "the 12 fused conv launches: sum of algorithmic flops / sum of "
                          "per-layer L2-flushed kernel times",
            },
            "layers": h["layers"],
            "precisions": {p: sub(p) for p in res if p != headline},
            "resnet18": resnet,
            "depthwise": depthwise or None,
            "gpu_launches": h["launches"],
            "clocks": clk.summary(),
            "e2e": e2e,
            "cpu_baseline": cpu,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def run_e2e(args, batch, device, compute, world):
    """The headline metric through the public C ABI a reference user calls
    (tec_eval_fused_conv: host NCHW f32 buffers), H2D + pack + kernel +
    unpack + D2H inside the timed region, max over ranks."""
    import ctypes as C

    import torch
    import torch.distributed as dist

    from paper_1802_04799_b200 import _abi
    lib = _abi.load()
    steps = max(1, min(3, args.steps))
    g = torch.Generator().manual_seed(7)
    prepared = []
    h2d = d2h = 0
    flops = 0
    cm = {"f32tc": _abi.COMPUTE_F32TC, "bf16": _abi.COMPUTE_BF16, "i8": _abi.COMPUTE_I8}[compute]
    for name in LAYERS:
        wl = resnet_layer(name, batch)
        if compute == "i8":
            x = torch.randint(-8, 8, (wl.n, wl.c, wl.h, wl.w), dtype=torch.int8, generator=g)
            w = torch.randint(-8, 8, (wl.k, wl.c, wl.r, wl.s), dtype=torch.int8, generator=g)
            b = torch.randint(-100, 101, (wl.k,), dtype=torch.int32, generator=g)
            y = torch.empty((wl.n, wl.k, wl.oh, wl.ow), dtype=torch.int32)
        else:
            x = torch.rand((wl.n, wl.c, wl.h, wl.w), generator=g) * 2 - 1
            w = torch.rand((wl.k, wl.c, wl.r, wl.s), generator=g) * 2 - 1
            b = torch.rand((wl.k,), generator=g) * 2 - 1
            y = torch.empty((wl.n, wl.k, wl.oh, wl.ow))
        x, w, b, y = x.pin_memory(), w.pin_memory(), b.pin_memory(), y.pin_memory()
        d = _abi.ConvDesc(n=wl.n, c=wl.c, h=wl.h, w=wl.w, k=wl.k, r=wl.r, s=wl.s,
                          stride_h=wl.stride, stride_w=wl.stride, pad_h=wl.pad,
                          pad_w=wl.pad, depthwise=0, compute=cm)
        e = _abi.Epilogue()
        e.n_ops = 2
        e.ops[0] = _abi.EPI_BIAS
        e.ops[1] = _abi.EPI_RELU
        e.bias = b.data_ptr()
        prepared.append((d, e, x, w, y, b))
        h2d += x.numel() * x.element_size() + w.numel() * w.element_size() + b.numel() * 4
        d2h += y.numel() * 4
        flops += wl.flops
    kn = _abi.Knobs()

    def one():
        for d, e, x, w, y, b in prepared:
            _abi.check(lib.tec_eval_fused_conv(C.byref(d), C.byref(e), C.byref(kn),
                                               x.data_ptr(), w.data_ptr(), y.data_ptr(),
                                               device))
    one()  # warm-up: workspace allocation
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    t0 = time.perf_counter()
    for _ in range(steps):
        one()
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t0) / steps
    if world > 1:
        t = torch.tensor([dt], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dt = float(t.item())
    pcie = pcie_duplex_gbs()
    moved = (h2d + d2h) / dt / 1e9
    return {"value": round(world * flops / dt / 1e12, 3),
            "unit": "TOPS" if compute == "i8" else "TFLOP/s",
            "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
            "ms_per_step": round(dt * 1e3, 2), "compute": compute,
            # the e2e roofline: this box's pinned PCIe rate with both
            # directions busy (the step moves h2d + d2h bytes)
            "pcie_gbs": round(moved, 1), "pcie_duplex_peak_gbs": round(pcie, 1),
            "frac_of_pcie": round(moved / pcie, 3) if pcie else None,
            "path": "tec_eval_fused_conv (C ABI, host NCHW buffers, pinned), wall clock incl. "
                    "H2D, layout packing, kernel, unpack, D2H; max over ranks"}


def pcie_duplex_gbs(nbytes=128 << 20, reps=4):
    """Pinned host<->device copy rate with an H2D and a D2H stream running
    together (GB/s of both directions summed): what a step that uploads its
    inputs and downloads its outputs can reach."""
    import torch
    h_in = torch.empty(nbytes, dtype=torch.uint8).pin_memory()
    h_out = torch.empty(nbytes, dtype=torch.uint8).pin_memory()
    d_in = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
    d_out = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()

    def both():
        with torch.cuda.stream(s1):
            d_in.copy_(h_in, non_blocking=True)
        with torch.cuda.stream(s2):
            h_out.copy_(d_out, non_blocking=True)
    both()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        both()
    torch.cuda.synchronize()
    return 2 * nbytes * reps / (time.perf_counter() - t0) / 1e9


# ------------------------------------------------------------ multi-rank plumbing
def relaunch_under_torchrun(args):
    """`bench.py --gpus N` outside torchrun: re-run this command as N ranks
    (torch.distributed.run, one node, 127.0.0.1) and pass rank 0's output
    through."""
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr=127.0.0.1",
           f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    env = dict(os.environ, OMP_NUM_THREADS=os.environ.get("OMP_NUM_THREADS", "1"))
    return subprocess.call(cmd, env=env)


def impl_cpu_dry_run(args):
    """The rank plumbing of the multi-GPU bench on gloo, no GPU: every rank
    shards the ResNet-18 global batch, times its (tiny, oracle-free numpy)
    stand-in step between barriers, the max over ranks is reduced, and the
    logits slices are gathered in rank order -- what the GPU run does, with
    the kernels replaced by a host matmul."""
    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_1802_04799_b200.parallel import gather_rows, shard_batch
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if world > 1:
        dist.init_process_group("gloo")
    gb = args.global_batch or 256
    start, cnt = shard_batch(gb, world, rank)
    rng = np.random.default_rng(rank)
    a = rng.standard_normal((cnt, 512)).astype(np.float32)
    w = rng.standard_normal((512, 10)).astype(np.float32)
    if world > 1:
        dist.barrier()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        logits = a @ w
    dt = time.perf_counter() - t0
    t = torch.tensor([dt], dtype=torch.float64)
    ranks = [torch.zeros(1, dtype=torch.int64) for _ in range(world)]
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dist.all_gather(ranks, torch.tensor([rank], dtype=torch.int64))
    full = gather_rows(torch.from_numpy(logits), gb)
    if rank == 0:
        print(json.dumps({
            "metric": METRIC, "dry_run": True, "backend": "gloo" if world > 1 else "none",
            "n_gpus": world, "ranks": [int(r.item()) for r in ranks] if world > 1 else [0],
            "global_batch": gb, "gathered_rows": int(full.shape[0]),
            "max_rank_seconds": float(t.item()), "steps": args.steps}), flush=True)
    if world > 1:
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--batch", type=int, default=64)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-tune", action="store_true", help="library default knobs (workloads)")
    ap.add_argument("--knobs-in", default="",
                    help="knob file {precision: {layer: knobs}} instead of profiles/tuned_knobs.json")
    ap.add_argument("--allow-untested-knobs", action="store_true",
                    help="accept a knob file the parity tests do not cover")
    ap.add_argument("--precision", default="f32tc", choices=["f32tc", "bf16", "i8"],
                    help="headline arithmetic (default: f32, the reference's precision)")
    ap.add_argument("--also", default="bf16,i8", help="sub-result precisions in the same line")
    ap.add_argument("--no-resnet18", action="store_true")
    ap.add_argument("--no-depthwise", action="store_true")
    ap.add_argument("--cpu-dry-run", action="store_true",
                    help="multi-rank plumbing on gloo without a GPU (tests)")
    ap.add_argument("--workload", default="conv",
                    choices=["conv", "resnet18", "depthwise", "c2b1", "int8"],
                    help="conv = the headline configs[1]; others: bench_workloads.py")
    ap.add_argument("--global-batch", type=int, default=0, help="resnet18: total images")
    ap.add_argument("--dw-compute", default="bf16", choices=["bf16", "f32"])
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3  # timing rule: >= 3 warm-up steps
    if args.knobs_in and os.path.abspath(args.knobs_in) != os.path.abspath(KNOBS_FILE) and \
            not args.allow_untested_knobs:
        raise SystemExit(f"bench.py: {args.knobs_in} is not the knob file the parity tests cover "
                         f"({os.path.relpath(KNOBS_FILE, REPO)}); pass --allow-untested-knobs")
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(relaunch_under_torchrun(args))
    if args.cpu_dry_run:
        impl_cpu_dry_run(args)
    elif args.impl == "reference":
        impl_reference(args)
    elif args.workload != "conv":
        import bench_workloads
        bench_workloads.WORKLOADS[args.workload](args, sys.modules[__name__])
    else:
        impl_ours(args)


if __name__ == "__main__":
    main()
