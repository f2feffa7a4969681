"""fold_constants / apply_layouts (graph.py) against the reference.

fold: our folded graph, evaluated by the REFERENCE binary
(oracle/_ref/ref_driver eval), must give bit-identical outputs to the
reference's evaluation of the original graph (tests/golden/passes/*/out).
(The reference's own fold_constants reads freed memory once its node vector
grows -- see tests/golden/make_golden.py -- so its output is not a golden.)
layouts: structurally identical to the reference's apply_layouts output."""
import json
import os
import subprocess

import numpy as np
import pytest

from oracle.oracle_api import load_tensor
from paper_1802_04799_b200 import TecError
from paper_1802_04799_b200.graph import (apply_layouts, fold_constants, graph_from_json,
                                         graph_to_json)

HERE = os.path.dirname(os.path.abspath(__file__))
PASSES = os.path.join(HERE, "golden", "passes")
DRIVER = os.path.join(os.path.dirname(HERE), "oracle", "_ref", "ref_driver")
HOST_FOLD = ["fold_elemwise", "fold_int", "fold_seq_sum"]


def _case(name):
    d = os.path.join(PASSES, name)
    with open(os.path.join(d, "graph.json")) as f:
        return d, json.load(f)


def _ref_eval(gjson, feeds_dir, tmp_path):
    gp = tmp_path / "folded.json"
    gp.write_text(json.dumps(gjson))
    out = tmp_path / "out"
    out.mkdir()
    subprocess.run([DRIVER, "eval", str(gp), feeds_dir, str(out)], check=True,
                   capture_output=True)
    return str(out)


def _check_fold(name, tmp_path):
    d, gj = _case(name)
    g = graph_from_json(gj)
    folded = fold_constants(g)
    # every foldable node is gone: only inputs, consts and their consumers
    assert all(n.op in ("input", "const") or
               any(folded.node(i).op == "input" for i in n.inputs) or
               any(folded.node(i).op not in ("const",) for i in n.inputs)
               for n in folded.nodes)
    if not os.path.exists(DRIVER):
        pytest.skip("oracle/_ref not built")
    out = _ref_eval(graph_to_json(folded), d, tmp_path)
    for o in g.outputs:
        got, want = load_tensor(out, o), load_tensor(os.path.join(d, "out"), o)
        assert np.array_equal(got.view(np.uint32) if got.dtype == np.float32 else got,
                              want.view(np.uint32) if want.dtype == np.float32 else want), o


@pytest.mark.parametrize("name", HOST_FOLD)
def test_fold_constants_matches_reference_eval(name, tmp_path):
    _check_fold(name, tmp_path)


def test_fold_overflow_is_fold_overflow():
    _, gj = _case("fold_overflow")
    with pytest.raises(TecError) as e:
        fold_constants(graph_from_json(gj))
    assert e.value.code == "FoldOverflow"


def test_fold_through_const_without_payload_is_not_enough_data():
    g = graph_from_json({"nodes": [{"id": "c", "op": "const", "shape": [2], "dtype": "f32"},
                                   {"id": "r", "op": "relu", "inputs": ["c"]}],
                         "outputs": ["r"]})
    with pytest.raises(TecError) as e:
        fold_constants(g)
    assert e.value.code == "NotEnoughData"


@pytest.mark.gpu
def test_fold_conv_on_device_matches_reference_eval(tmp_path):
    _check_fold("fold_conv", tmp_path)


def test_apply_layouts_matches_reference():
    d, gj = _case("layouts_tiled")
    with open(os.path.join(d, "prefs.json")) as f:
        prefs = json.load(f)
    with open(os.path.join(d, "layouts.json")) as f:
        want = json.load(f)
    got = graph_to_json(apply_layouts(graph_from_json(gj), prefs))
    key = lambda n: (n["id"], n["op"], n.get("inputs", []), n.get("attrs", {}),  # noqa: E731
                     n.get("shape"), n.get("dtype"))
    assert [key(n) for n in got["nodes"]] == [key(n) for n in want["nodes"]]
    assert got["outputs"] == want["outputs"]
    with pytest.raises(TecError):
        apply_layouts(graph_from_json(gj), {"s": "tiled9x9"})
