"""Loader for tests/golden/<case>/ fixtures written by make_golden.py from
the reference binary. Maps each reference graph to (op, x, w, strides,
padding, epilogue items) the way fuse_pass would group it."""
from __future__ import annotations

import json
import os
from dataclasses import dataclass
from typing import List, Optional

import numpy as np

from oracle.oracle_api import load_tensor

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


@dataclass
class GoldenCase:
    name: str
    op: str
    x: np.ndarray
    w: np.ndarray
    strides: tuple
    padding: tuple
    epilogue: list
    expected: Optional[np.ndarray]
    status: str
    graph: dict
    fused: dict


def names() -> List[str]:
    return sorted(d for d in os.listdir(GOLDEN)
                  if os.path.isfile(os.path.join(GOLDEN, d, "graph.json")))


def load(name: str) -> GoldenCase:
    d = os.path.join(GOLDEN, name)
    with open(os.path.join(d, "graph.json")) as f:
        g = json.load(f)
    with open(os.path.join(d, "fused.json")) as f:
        fused = json.load(f)
    with open(os.path.join(d, "status")) as f:
        status = f.read().strip()
    nodes = {n["id"]: n for n in g["nodes"]}
    conv = nodes["conv"]
    attrs = conv.get("attrs", {})
    epi = []
    for n in g["nodes"]:
        if n["op"] in ("input", conv["op"]):
            continue
        if n["op"] == "relu":
            epi.append(("relu",))
        elif n["op"] == "scale":
            epi.append(("scale", n["attrs"]["scale"]))
        else:
            other = [i for i in n["inputs"] if nodes[i]["op"] == "input"][0]
            epi.append((n["op"], load_tensor(d, other)))
    out_id = g["outputs"][0]
    expected = None
    if status == "ok":
        expected = load_tensor(os.path.join(d, "out"), out_id)
    return GoldenCase(name, conv["op"], load_tensor(d, "x"), load_tensor(d, "w"),
                      tuple(attrs.get("strides", (1, 1))),
                      tuple(attrs.get("padding", (0, 0))), epi, expected,
                      status, g, fused)
