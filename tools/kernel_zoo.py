#!/usr/bin/env python3
"""Every kernel family of libtec_sm100.so once, on small shapes, through the
host C ABI (tec_eval_fused_conv: layout pack -> kernel -> unpack), checked
against the oracle. No torch: it runs under compute-sanitizer in seconds
(tests/test_sanitizer_gpu.py, the analogue of the reference's race_check,
R/src/interp.cpp:548-580). `--fault` runs only the watchdog mutation case.

Device path per case: 1 MiB canary guards around the output (out-of-bounds
writes) and bit-identical results over repeated launches and fewer
persistent CTAs (races).

usage: kernel_zoo.py [--fault] [--no-device]
"""
import os
import sys

import numpy as np

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)

from oracle.oracle_api import bf16_round, fused_conv as oracle, same_values  # noqa: E402
from paper_1802_04799_b200.ops import fused_conv  # noqa: E402

# (name, op, x shape, w shape, stride, pad, compute, knobs, residual)
CASES = [
    ("bf16-im2col", "conv2d", (2, 64, 9, 11), (64, 64, 3, 3), 1, 1, "bf16", {"tile_k": 1}, False),
    ("bf16-im2col-splitk", "conv2d", (1, 128, 7, 7), (256, 128, 3, 3), 1, 1, "bf16",
     {"tile_k": 1, "tile_n": 128, "split_k": 2}, False),
    ("bf16-halo-streamed", "conv2d", (2, 64, 12, 12), (64, 64, 3, 3), 1, 1, "bf16",
     {"tile_k": 2, "stages": 1}, False),
    ("bf16-halo-resident", "conv2d", (2, 64, 12, 12), (64, 64, 3, 3), 1, 1, "bf16",
     {"tile_k": 2, "stages": 2}, True),
    ("bf16-halo-paired", "conv2d", (2, 64, 12, 12), (64, 64, 3, 3), 1, 1, "bf16",
     {"tile_k": 4}, False),
    ("bf16-halo-multicast", "conv2d", (3, 64, 12, 12), (64, 64, 3, 3), 1, 1, "bf16",
     {"tile_k": 2, "stages": 1, "cluster_n": 2}, False),
    ("bf16-s2d-stem", "conv2d", (1, 3, 32, 32), (64, 3, 7, 7), 2, 3, "bf16", {}, False),
    # CTA pairs (cta_group::2): M = 49 leaves the pair's second tile a phantom
    ("bf16-im2col-pair", "conv2d", (1, 128, 7, 7), (256, 128, 3, 3), 1, 1, "bf16",
     {"tile_k": 1, "tile_n": 128, "cluster_n": 2}, False),
    ("i8-im2col-pair", "conv2d", (3, 64, 9, 9), (128, 64, 3, 3), 1, 1, "i8",
     {"tile_k": 1, "tile_n": 64, "cluster_n": 2}, False),
    ("f32tc-pair-streamk", "conv2d", (1, 128, 14, 14), (128, 128, 3, 3), 1, 1, "f32tc",
     {"tile_k": 1, "tile_n": 128, "split_k": -1, "cluster_n": 2}, False),
    ("f32tc-pair", "conv2d", (3, 64, 9, 9), (128, 64, 3, 3), 1, 1, "f32tc",
     {"tile_k": 1, "tile_n": 128, "cluster_n": 2}, True),
    ("i8-im2col", "conv2d", (2, 64, 9, 9), (64, 64, 3, 3), 2, 1, "i8", {"tile_k": 1}, False),
    ("i8-halo", "conv2d", (2, 64, 10, 10), (64, 64, 3, 3), 1, 1, "i8", {"tile_k": 2}, False),
    ("f32-exact", "conv2d", (1, 16, 8, 8), (16, 16, 3, 3), 1, 1, "f32", {}, True),
    ("f32tc-planes", "conv2d", (2, 64, 9, 9), (128, 64, 3, 3), 1, 1, "f32tc", {}, True),
    ("f32tc-splitk", "conv2d", (1, 128, 7, 7), (128, 128, 3, 3), 1, 1, "f32tc",
     {"split_k": 3}, False),
    ("f32tc-interleaved-stem", "conv2d", (1, 3, 32, 32), (64, 3, 7, 7), 2, 3, "f32tc", {}, False),
    ("f32tc-sw32", "conv2d", (1, 32, 8, 8), (32, 32, 3, 3), 1, 1, "f32tc", {}, False),
    ("dw-tma-bf16", "depthwise_conv2d", (2, 64, 14, 14), (64, 1, 3, 3), 1, 1, "bf16",
     {"unroll": 8}, False),
    ("dw-tma-f32", "depthwise_conv2d", (2, 64, 14, 14), (64, 1, 3, 3), 2, 1, "f32",
     {"unroll": 8}, False),
    ("dw-direct", "depthwise_conv2d", (2, 64, 14, 14), (64, 1, 3, 3), 1, 1, "bf16",
     {"unroll": 4}, False),
    ("dw-generic", "depthwise_conv2d", (1, 16, 9, 9), (16, 1, 3, 3), 1, 1, "f32",
     {"unroll": 1}, False),
    ("dw-i8", "depthwise_conv2d", (1, 32, 9, 9), (32, 1, 3, 3), 1, 1, "i8", {}, False),
]


def run_case(name, op, xs, ws, s, p, compute, knobs, residual, seed=0):
    rng = np.random.default_rng(seed)
    k = ws[0]
    if compute == "i8":
        x = rng.integers(-8, 8, xs, dtype=np.int8)
        w = rng.integers(-8, 8, ws, dtype=np.int8)
        b = rng.integers(-100, 101, (k,), dtype=np.int32)
    else:
        x = rng.uniform(-1, 1, xs).astype(np.float32)
        w = rng.uniform(-1, 1, ws).astype(np.float32)
        b = rng.uniform(-1, 1, (k,)).astype(np.float32)
    oh = (xs[2] + 2 * p - ws[2]) // s + 1
    ow = (xs[3] + 2 * p - ws[3]) // s + 1
    epi = [("bias_add", b)]
    if residual:
        epi.append(("add", rng.uniform(-1, 1, (xs[0], k, oh, ow)).astype(np.float32)))
    epi.append(("relu",))
    attrs = {"strides": (s, s), "padding": (p, p)}
    y = fused_conv(op, x, w, attrs, epi, compute=None if compute == "i8" else compute,
                   knobs=knobs)
    xr, wr = (bf16_round(x), bf16_round(w)) if compute == "bf16" else (x, w)
    want = oracle(op, xr, wr, (s, s), (p, p), epi)
    tol = {"bf16": 2e-3, "f32tc": 1e-4}.get(compute, 0.0)
    ok = np.array_equal(y, want) if tol == 0.0 else same_values(y, want, tol)
    if op == "depthwise_conv2d" and compute != "i8":
        ok = np.array_equal(y, want)
    return ok


def device_guard_and_determinism(name, op, xs, ws, s, p, compute, knobs, residual, seed=0):
    """The same case on the DEVICE path (tec_conv2d_fused / tec_depthwise_fused
    on caller buffers): the output sits between two 1 MiB guard regions
    filled with a canary pattern that must survive (no out-of-bounds
    writes), and repeated launches -- and launches with fewer persistent
    CTAs (knob grid) -- must give bit-identical results (no races: every
    kernel's reduction order is fixed by construction)."""
    import ctypes as C
    import torch
    from paper_1802_04799_b200 import _abi
    from paper_1802_04799_b200.ops import conv_desc
    rng = np.random.default_rng(seed)
    lib = _abi.load()
    cm = {"bf16": _abi.COMPUTE_BF16, "i8": _abi.COMPUTE_I8, "f32": _abi.COMPUTE_F32,
          "f32tc": _abi.COMPUTE_F32TC}[compute]
    shape = []
    attrs = {"strides": (s, s), "padding": (p, p)}
    d = conv_desc(op, xs, ws, attrs, cm, shape)
    lay = _abi.ConvLayout()
    _abi.check(lib.tec_conv_layout_of(C.byref(d), C.byref(lay)))
    dev = torch.device("cuda", 0)
    if compute == "i8":
        x = torch.randint(-8, 8, xs, dtype=torch.int8, device=dev)
        w = torch.randint(-8, 8, ws, dtype=torch.int8, device=dev)
        b = torch.randint(-100, 101, (ws[0],), dtype=torch.int32, device=dev)
    else:
        x = torch.rand(xs, device=dev) * 2 - 1
        w = torch.rand(ws, device=dev) * 2 - 1
        b = torch.rand((ws[0],), device=dev) * 2 - 1
    xp = torch.empty(lay.act_bytes, dtype=torch.uint8, device=dev)
    wp = torch.empty(lay.wt_bytes, dtype=torch.uint8, device=dev)
    st = torch.cuda.current_stream().cuda_stream
    _abi.check(lib.tec_weight_pretransform(C.byref(d), w.data_ptr(), wp.data_ptr(), st))
    _abi.check(lib.tec_activation_pack(C.byref(d), x.data_ptr(), xp.data_ptr(), st))
    out_dt = {"i8": _abi.DT_I32, "bf16": _abi.DT_BF16}.get(compute, _abi.DT_F32)
    es = 2 if out_dt == _abi.DT_BF16 else 4
    n_out = shape[0] * shape[1] * shape[2] * shape[3]
    guard = 1 << 20
    buf = torch.full((guard * 2 + n_out * es,), 0xA5, dtype=torch.uint8, device=dev)
    res = None
    if residual and compute not in ("i8",):
        res = (torch.rand((n_out,), device=dev) * 2 - 1).to(
            torch.bfloat16 if out_dt == _abi.DT_BF16 else torch.float32)
    epi = _abi.Epilogue()
    ops = [_abi.EPI_BIAS] + ([_abi.EPI_ADD] if res is not None else []) + [_abi.EPI_RELU]
    for i, o in enumerate(ops):
        epi.ops[i] = o
    epi.n_ops = len(ops)
    epi.bias = b.data_ptr()
    if res is not None:
        epi.residual = res.data_ptr()
    fn = lib.tec_depthwise_fused if op == "depthwise_conv2d" else lib.tec_conv2d_fused
    outs = []
    for grid in (0, 0, 4, 2):
        kn = _abi.Knobs(**dict(knobs, grid=grid) if grid else knobs)
        if op == "depthwise_conv2d" and grid:
            continue  # the depthwise kernels size their own grid
        _abi.check(fn(C.byref(d), C.byref(epi), C.byref(kn), xp.data_ptr(), wp.data_ptr(),
                      buf.data_ptr() + guard, out_dt, None, st))
        torch.cuda.synchronize()
        outs.append(buf[guard:guard + n_out * es].clone())
    canary_ok = bool((buf[:guard] == 0xA5).all() and (buf[guard + n_out * es:] == 0xA5).all())
    if knobs.get("split_k") == -1:
        # stream-K: the segment boundaries follow the grid (each grid sums in
        # a fixed order); repeats at one grid must match bit for bit
        same = torch.equal(outs[0], outs[1])
    else:
        same = all(torch.equal(o, outs[0]) for o in outs[1:])
    return canary_ok, same


def main():
    if "--fault" in sys.argv:
        # the f32tc epilogue drops one accumulator-free arrive
        # (TEC_SM100_FAULT=1): the MMA warp's mbarrier watchdog must trap
        os.environ["TEC_SM100_FAULT"] = "1"
        run_case("fault", "conv2d", (4, 64, 16, 16), (64, 64, 3, 3), 1, 1, "f32tc",
                 {"grid": 1}, False)
        print("fault case returned without a trap")
        return 1
    bad = []
    device_checks = "--no-device" not in sys.argv
    for c in CASES:
        ok = run_case(*c)
        msg = "ok" if ok else "MISMATCH"
        if device_checks:
            canary, same = device_guard_and_determinism(*c)
            ok = ok and canary and same
            msg += ("" if canary else " OUT-OF-BOUNDS-WRITE") + ("" if same else " NONDETERMINISTIC")
        print(f"{c[0]}: {msg}", flush=True)
        if not ok:
            bad.append(c[0])
    print("zoo:", "all ok" if not bad else f"mismatch in {bad}")
    return 1 if bad else 0


if __name__ == "__main__":
    sys.exit(main())
