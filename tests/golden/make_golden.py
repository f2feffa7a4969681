#!/usr/bin/env python3
"""Generates the golden fixtures in tests/golden/ by running the REFERENCE.

Run in the build container (where /root/reference exists and
`make -C oracle ref` has built oracle/_ref/ref_driver):

    python tests/golden/make_golden.py

For every case it writes, under tests/golden/<case>/:
  graph.json            the reference-format graph (R/src/graph.cpp:146-207)
  <input>.bin/.json     inputs in the reference's tensor format
                        (R/src/io.cpp:111-127); random ones come from the
                        reference's own random_tensor (R/src/tensor.cpp:74-88)
                        via `ref_driver gen`
  out/<output>.bin/.json  outputs of the reference's evaluate_graph
                        (R/src/graph.cpp:227-256) via `ref_driver eval`
  fused.json            fuse_pass + plan_memory of the graph
  status                "ok" or the reference error code when it throws
The reference itself is never needed again: tests read only these files.
"""
from __future__ import annotations

import json
import os
import shutil
import subprocess
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
DRIVER = os.path.join(REPO, "oracle", "_ref", "ref_driver")


def save_tensor(d, name, arr, dtype):
    os.makedirs(d, exist_ok=True)
    with open(os.path.join(d, name + ".json"), "w") as f:
        json.dump({"name": name, "shape": list(arr.shape), "dtype": dtype}, f)
    raw = arr.astype({"f32": "<f4", "i32": "<i4", "i8": "i1"}[dtype]).tobytes()
    with open(os.path.join(d, name + ".bin"), "wb") as f:
        f.write(raw)


def conv_graph(op, x_shape, w_shape, strides, padding, epi, dtype="f32",
               residual_shape=None):
    acc = "i32" if dtype == "i8" else "f32"
    nodes = [
        {"id": "x", "op": "input", "shape": list(x_shape), "dtype": dtype},
        {"id": "w", "op": "input", "shape": list(w_shape), "dtype": dtype},
    ]
    prev = "conv"
    body = [{"id": "conv", "op": op, "inputs": ["x", "w"],
             "attrs": {"strides": list(strides), "padding": list(padding)}}]
    for i, e in enumerate(epi):
        nid = f"e{i}_{e[0]}"
        if e[0] == "scale":
            body.append({"id": nid, "op": "scale", "inputs": [prev],
                         "attrs": {"scale": e[1]}})
        elif e[0] == "bias_add":
            nodes.append({"id": "b", "op": "input", "shape": [w_shape[0]],
                          "dtype": acc})
            body.append({"id": nid, "op": "bias_add", "inputs": [prev, "b"]})
        elif e[0] in ("add", "mul"):
            rid = "r" if e[0] == "add" else "m"
            nodes.append({"id": rid, "op": "input",
                          "shape": list(residual_shape), "dtype": acc})
            body.append({"id": nid, "op": e[0], "inputs": [prev, rid]})
        elif e[0] == "relu":
            body.append({"id": nid, "op": "relu", "inputs": [prev]})
        prev = nid
    return {"nodes": nodes + body, "outputs": [prev]}


def out_hw(h, w, k, strides, padding):
    return ((h + 2 * padding[0] - k[0]) // strides[0] + 1,
            (w + 2 * padding[1] - k[1]) // strides[1] + 1)


CASES = []


def case(name, op, x_shape, w_shape, strides=(1, 1), padding=(0, 0), epi=(),
         dtype="f32", explicit=None, seed=1):
    CASES.append(dict(name=name, op=op, x_shape=x_shape, w_shape=w_shape,
                      strides=strides, padding=padding, epi=list(epi),
                      dtype=dtype, explicit=explicit, seed=seed))


# Known-answer tests: 3x3 ones kernel, pad 1 -> corner 4, edge 6,
# centre 9 (times the value).
case("kat_ones_pad1", "conv2d", (1, 1, 3, 3), (1, 1, 3, 3), padding=(1, 1),
     explicit={"x": np.full((1, 1, 3, 3), 2.0, np.float32),
               "w": np.ones((1, 1, 3, 3), np.float32)})
case("kat_depthwise", "depthwise_conv2d", (1, 2, 3, 3), (2, 1, 3, 3),
     padding=(1, 1),
     explicit={"x": np.stack([np.full((3, 3), 1.0), np.full((3, 3), -3.0)])
               [None].astype(np.float32),
               "w": np.stack([np.ones((3, 3)), np.full((3, 3), 0.5)])
               [:, None].astype(np.float32)})
case("kat_stride2", "conv2d", (1, 1, 5, 5), (1, 1, 3, 3), strides=(2, 2),
     padding=(1, 1),
     explicit={"x": np.arange(25, dtype=np.float32).reshape(1, 1, 5, 5),
               "w": np.ones((1, 1, 3, 3), np.float32)})
# The reference's own conv test shape (R/tests/test_lower.cpp:197-209).
case("conv_unpadded_ref_test", "conv2d", (1, 2, 6, 6), (3, 2, 3, 3), seed=71)
# Random f32 cases with the fused epilogues fuse_pass produces.
case("conv_bias_relu", "conv2d", (2, 8, 9, 9), (16, 8, 3, 3), padding=(1, 1),
     epi=[("bias_add",), ("relu",)], seed=3)
case("conv_s2_bias_relu", "conv2d", (1, 8, 11, 11), (16, 8, 3, 3),
     strides=(2, 2), padding=(1, 1), epi=[("bias_add",), ("relu",)], seed=5)
case("conv_1x1_s2", "conv2d", (1, 16, 8, 8), (32, 16, 1, 1), strides=(2, 2),
     epi=[("bias_add",)], seed=7)
case("conv_residual", "conv2d", (1, 16, 8, 8), (16, 16, 3, 3),
     padding=(1, 1),
     epi=[("scale", 0.5), ("bias_add",), ("add",), ("relu",)], seed=9)
case("conv_mul", "conv2d", (1, 4, 6, 6), (8, 4, 3, 3), padding=(1, 1),
     epi=[("mul",), ("relu",)], seed=10)
case("conv_asym", "conv2d", (1, 4, 7, 9), (8, 4, 3, 5), strides=(2, 1),
     padding=(1, 2), epi=[("bias_add",), ("relu",)], seed=11)
case("conv_stem_k7s2", "conv2d", (1, 3, 16, 16), (16, 3, 7, 7),
     strides=(2, 2), padding=(3, 3), epi=[("bias_add",), ("relu",)], seed=13)
case("conv_odd_oc", "conv2d", (1, 5, 6, 7), (3, 5, 3, 3), padding=(1, 1),
     epi=[("bias_add",)], seed=15)
# C2 slice at full channel depth: 8 of the 56 rows (16.5 M MACs).
case("c2_slice", "conv2d", (1, 64, 8, 56), (64, 64, 3, 3), padding=(1, 1),
     epi=[("bias_add",), ("relu",)], seed=17)
# Depthwise (MobileNet D-layer structure).
case("dw_bias_relu", "depthwise_conv2d", (1, 16, 10, 10), (16, 1, 3, 3),
     padding=(1, 1), epi=[("bias_add",), ("relu",)], seed=19)
case("dw_s2", "depthwise_conv2d", (2, 32, 9, 9), (32, 1, 3, 3),
     strides=(2, 2), padding=(1, 1), epi=[("bias_add",), ("relu",)], seed=21)
# int8 path (i8 x i8 -> i32, bit-exact).
case("i8_conv_bias_relu", "conv2d", (1, 32, 8, 8), (32, 32, 3, 3),
     padding=(1, 1), epi=[("bias_add",), ("relu",)], dtype="i8", seed=23)
case("i8_conv_scale_s2", "conv2d", (1, 16, 9, 9), (32, 16, 3, 3),
     strides=(2, 2), padding=(1, 1), epi=[("scale", 3.0), ("bias_add",)],
     dtype="i8", seed=25)
case("i8_dw", "depthwise_conv2d", (1, 32, 8, 8), (32, 1, 3, 3),
     padding=(1, 1), epi=[("bias_add",), ("relu",)], dtype="i8", seed=27)
# Saturation range: all -128 with K = 4608 -> 75,497,472.
case("i8_saturation", "conv2d", (1, 512, 3, 3), (16, 512, 3, 3),
     padding=(1, 1), dtype="i8",
     explicit={"x": np.full((1, 512, 3, 3), -128, np.int8),
               "w": np.full((16, 512, 3, 3), -128, np.int8)})
# FoldOverflow: a scale that pushes i32 out of range must raise.
case("i8_overflow", "conv2d", (1, 512, 3, 3), (16, 512, 3, 3),
     padding=(1, 1), dtype="i8", epi=[("scale", 64.0)],
     explicit={"x": np.full((1, 512, 3, 3), -128, np.int8),
               "w": np.full((16, 512, 3, 3), -128, np.int8)})


def run(cmd):
    subprocess.run(cmd, check=True)


def build_case(c):
    d = os.path.join(HERE, c["name"])
    if os.path.exists(d):
        shutil.rmtree(d)
    os.makedirs(os.path.join(d, "out"))
    acc = "i32" if c["dtype"] == "i8" else "f32"
    k = c["w_shape"][2:]
    oh, ow = out_hw(c["x_shape"][2], c["x_shape"][3], k, c["strides"],
                    c["padding"])
    rshape = (c["x_shape"][0], c["w_shape"][0], oh, ow)
    g = conv_graph(c["op"], c["x_shape"], c["w_shape"], c["strides"],
                   c["padding"], c["epi"], c["dtype"], rshape)
    with open(os.path.join(d, "graph.json"), "w") as f:
        json.dump(g, f, indent=1)
    seed = c["seed"]
    for n in g["nodes"]:
        if n["op"] != "input":
            continue
        if c["explicit"] and n["id"] in c["explicit"]:
            save_tensor(d, n["id"], c["explicit"][n["id"]], n["dtype"])
        else:
            seed += 1
            run([DRIVER, "gen", d, n["id"], n["dtype"], str(seed)] +
                [str(s) for s in n["shape"]])
    p = subprocess.run([DRIVER, "eval", os.path.join(d, "graph.json"), d,
                        os.path.join(d, "out")], capture_output=True, text=True)
    status = "ok" if p.returncode == 0 else p.stderr.strip()
    with open(os.path.join(d, "status"), "w") as f:
        f.write(status + "\n")
    run([DRIVER, "fuse", os.path.join(d, "graph.json"),
         os.path.join(d, "fused.json")])
    print(f"{c['name']}: {status}")


# --------------------------------------------------------- whole graphs
# tests/golden/graphs/<name>/: multi-node reference graphs for the graph
# passes (fuse_pass + plan_memory -> fused.json) and, when `evaluate`, for
# the device executor (inputs + out/ from the reference's evaluate_graph).
def graph_cases():
    sys.path.insert(0, REPO)
    from paper_1802_04799_b200.graph import graph_to_json
    from paper_1802_04799_b200.workloads import resnet18_graph
    gap = {"nodes": [{"id": "x", "op": "input", "shape": [2, 16, 7, 7], "dtype": "f32"},
                     {"id": "sw", "op": "sum", "inputs": ["x"], "attrs": {"axis": 3}},
                     {"id": "sh", "op": "sum", "inputs": ["sw"], "attrs": {"axis": 2}},
                     {"id": "avg", "op": "scale", "inputs": ["sh"],
                      "attrs": {"scale": 1.0 / 49}}],
           "outputs": ["avg"]}
    fc = {"nodes": [{"id": "x", "op": "input", "shape": [4, 64], "dtype": "f32"},
                    {"id": "w", "op": "input", "shape": [64, 24], "dtype": "f32"},
                    {"id": "b", "op": "input", "shape": [24], "dtype": "f32"},
                    {"id": "mm", "op": "matmul", "inputs": ["x", "w"]},
                    {"id": "logits", "op": "bias_add", "inputs": ["mm", "b"]}],
          "outputs": ["logits"]}
    return [
        ("gap_chain", gap, True),
        ("fc_head", fc, True),
        # ResNet-18 body at width 8 on a 32x32 image (17 convs, residual
        # adds, downsample branches): evaluated by the reference (~3 s).
        ("tiny_resnet_body", graph_to_json(resnet18_graph(1, image=32, width=8,
                                                          maxpool=False, head=False)), True),
        # Full-size ResNet-18 (reference-compatible variant, batch 8):
        # graph passes only.
        ("resnet18_b8", graph_to_json(resnet18_graph(8, maxpool=False)), False),
    ]


def build_graph_case(name, g, evaluate, seed=100):
    d = os.path.join(HERE, "graphs", name)
    if os.path.exists(d):
        shutil.rmtree(d)
    os.makedirs(os.path.join(d, "out"))
    with open(os.path.join(d, "graph.json"), "w") as f:
        json.dump(g, f, indent=1)
    run([DRIVER, "fuse", os.path.join(d, "graph.json"), os.path.join(d, "fused.json")])
    if evaluate:
        for n in g["nodes"]:
            if n["op"] == "input":
                seed += 1
                run([DRIVER, "gen", d, n["id"], n.get("dtype", "f32"), str(seed)] +
                    [str(v) for v in n["shape"]])
        run([DRIVER, "eval", os.path.join(d, "graph.json"), d, os.path.join(d, "out")])
    print(f"graphs/{name}: {'evaluated' if evaluate else 'passes only'}")


# ----------------------------------------------------- graph passes
# tests/golden/passes/<name>/: graph.json (+ prefs.json) and the reference's
# fold_constants / apply_layouts result (fold.json / layouts.json, or
# fold.status with the error when the reference throws).
def _const(nid, arr, dtype):
    import base64
    raw = np.ascontiguousarray(arr).astype({"f32": "<f4", "i32": "<i4", "i8": "i1"}[dtype]).tobytes()
    return {"id": nid, "op": "const", "shape": list(arr.shape), "dtype": dtype,
            "data": base64.b64encode(raw).decode()}


def pass_cases():
    rng = np.random.default_rng(123)
    f = lambda *s: rng.uniform(-2, 2, s).astype(np.float32)  # noqa: E731
    i = lambda *s: rng.integers(-1000, 1000, s).astype(np.int32)  # noqa: E731
    elem = {"nodes": [_const("c1", f(2, 3), "f32"), _const("c2", f(2, 3), "f32"),
                      {"id": "x", "op": "input", "shape": [2, 3], "dtype": "f32"},
                      {"id": "a", "op": "add", "inputs": ["c1", "c2"]},
                      {"id": "m", "op": "mul", "inputs": ["a", "c2"]},
                      {"id": "r", "op": "relu", "inputs": ["m"]},
                      {"id": "s", "op": "scale", "inputs": ["r"], "attrs": {"scale": 0.3}},
                      {"id": "e", "op": "exp", "inputs": ["s"]},
                      {"id": "q", "op": "sqrt", "inputs": ["e"]},
                      {"id": "y", "op": "add", "inputs": ["x", "q"]}], "outputs": ["y"]}
    ints = {"nodes": [_const("k1", i(3, 4), "i32"), _const("k2", i(3, 4), "i32"),
                      _const("kb", i(4), "i32"),
                      {"id": "x", "op": "input", "shape": [3], "dtype": "i32"},
                      {"id": "p", "op": "mul", "inputs": ["k1", "k2"]},
                      {"id": "s", "op": "scale", "inputs": ["p"], "attrs": {"scale": 3.0}},
                      {"id": "b", "op": "bias_add", "inputs": ["s", "kb"]},
                      {"id": "t", "op": "sum", "inputs": ["b"], "attrs": {"axis": 1}},
                      {"id": "y", "op": "add", "inputs": ["x", "t"]}], "outputs": ["y"]}
    seq = {"nodes": [_const("v", f(4, 33) * 1000, "f32"),
                     {"id": "x", "op": "input", "shape": [4], "dtype": "f32"},
                     {"id": "t", "op": "sum", "inputs": ["v"], "attrs": {"axis": 1}},
                     {"id": "y", "op": "mul", "inputs": ["x", "t"]}], "outputs": ["y"]}
    ovf = {"nodes": [_const("k", np.full((2,), 2_000_000_000, np.int32), "i32"),
                     {"id": "x", "op": "input", "shape": [2], "dtype": "i32"},
                     {"id": "d", "op": "add", "inputs": ["k", "k"]},
                     {"id": "y", "op": "add", "inputs": ["x", "d"]}], "outputs": ["y"]}
    conv = {"nodes": [_const("w", f(4, 2, 3, 3), "f32"), _const("cx", f(1, 2, 5, 5), "f32"),
                      _const("b", f(4), "f32"),
                      {"id": "x", "op": "input", "shape": [1, 4, 5, 5], "dtype": "f32"},
                      {"id": "c", "op": "conv2d", "inputs": ["cx", "w"],
                       "attrs": {"strides": [1, 1], "padding": [1, 1]}},
                      {"id": "cb", "op": "bias_add", "inputs": ["c", "b"]},
                      {"id": "y", "op": "add", "inputs": ["x", "cb"]}], "outputs": ["y"]}
    lay = {"nodes": [{"id": "x", "op": "input", "shape": [5, 6], "dtype": "f32"},
                     {"id": "z", "op": "input", "shape": [5, 6], "dtype": "f32"},
                     {"id": "r", "op": "relu", "inputs": ["x"]},
                     {"id": "a", "op": "add", "inputs": ["r", "z"]},
                     {"id": "s", "op": "scale", "inputs": ["a"], "attrs": {"scale": 2.0}}],
           "outputs": ["s"]}
    return [("fold_elemwise", elem, None), ("fold_int", ints, None), ("fold_seq_sum", seq, None),
            ("fold_overflow", ovf, None), ("fold_conv", conv, None),
            ("layouts_tiled", lay, {"r": "tiled4x4", "a": "tiled4x4"})]


def build_pass_case(name, g, prefs, seed=500):
    """fold cases: the reference's evaluate_graph of the ORIGINAL graph
    (inputs + out/, or out.status when it throws). The reference's own
    fold_constants is not used as a golden: it keeps pointers into the node
    vector it is still appending to (R/src/graph_passes.cpp:46-70), so it
    reads freed memory once the vector grows (reports NotEnoughData here).
    layout cases: the reference's apply_layouts result (layouts.json)."""
    d = os.path.join(HERE, "passes", name)
    if os.path.exists(d):
        shutil.rmtree(d)
    os.makedirs(os.path.join(d, "out"))
    gp = os.path.join(d, "graph.json")
    with open(gp, "w") as fh:
        json.dump(g, fh, indent=1)
    if prefs is None:
        for n in g["nodes"]:
            if n["op"] == "input":
                seed += 1
                run([DRIVER, "gen", d, n["id"], n.get("dtype", "f32"), str(seed)] +
                    [str(v) for v in n["shape"]])
        pr = subprocess.run([DRIVER, "eval", gp, d, os.path.join(d, "out")],
                            capture_output=True, text=True)
        with open(os.path.join(d, "out.status"), "w") as fh:
            fh.write(("ok" if pr.returncode == 0 else pr.stderr.strip()) + "\n")
    else:
        pp = os.path.join(d, "prefs.json")
        with open(pp, "w") as fh:
            json.dump(prefs, fh)
        run([DRIVER, "layouts", gp, pp, os.path.join(d, "layouts.json")])
    print(f"passes/{name}")


def main():
    if not os.path.exists(DRIVER):
        sys.exit(f"{DRIVER} missing: run `make -C oracle ref` first")
    only = set(sys.argv[1:])
    for c in CASES:
        if not only or c["name"] in only:
            build_case(c)
    for name, g, ev in graph_cases():
        if not only or name in only:
            build_graph_case(name, g, ev)
    for name, g, prefs in pass_cases():
        if not only or name in only:
            build_pass_case(name, g, prefs)


if __name__ == "__main__":
    main()
