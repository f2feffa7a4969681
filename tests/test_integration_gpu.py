"""The drop-in, proven from the reference's side: integration/tec_sm100_shim.*
(the C++ binding a tec maintainer adds) compiled against the
reference's own headers and library (oracle/Makefile `shim`) runs whole
reference graphs -- reference graph_from_json -> reference fuse_pass ->
conv-rooted fused nodes as ONE tec_eval_fused_conv call each, every other
node through the reference's own eval_graph_node -- and the outputs are
compared with the reference's evaluate_graph results (tests/golden/graphs,
written by the reference binary):
  * f32 (TEC_COMPUTE_F32): bit-identical, end to end;
  * f32tc (tensor cores): node by node -- every fused conv node, fed the
    reference's own intermediate tensors, within the 1e-4 comparator
    (R/src/tensor.cpp:56-72); end to end the differences compound through
    20 layers whose activations grow to ~1e12 (random weights), so the
    whole-graph output is held to TOL_F32TC_GRAPH = 1e-3.
"""
import json
import os
import subprocess

import numpy as np
import pytest

from oracle.oracle_api import fused_conv as oracle_conv, load_tensor, same_values, save_tensor

pytestmark = pytest.mark.gpu

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SHIM = os.path.join(REPO, "oracle", "_ref", "shim_driver")
GRAPHS = os.path.join(REPO, "tests", "golden", "graphs")
needs_shim = pytest.mark.skipif(not os.path.exists(SHIM),
                                reason="shim_driver not built (make -C oracle shim)")


def _outputs(name):
    with open(os.path.join(GRAPHS, name, "graph.json")) as f:
        return json.load(f)["outputs"]


@needs_shim
@pytest.mark.parametrize("mode", ["f32", "f32tc"])
@pytest.mark.parametrize("name", ["tiny_resnet_body", "fc_head", "gap_chain"])
def test_reference_graph_through_the_shim(name, mode, tmp_path):
    d = os.path.join(GRAPHS, name)
    res = subprocess.run([SHIM, "eval", os.path.join(d, "graph.json"), d, str(tmp_path), mode],
                         capture_output=True, text=True, timeout=600)
    assert res.returncode == 0, res.stderr
    info = json.loads(res.stdout)
    with open(os.path.join(d, "fused.json")) as f:  # the reference's own fuse_pass output
        fused = json.load(f)["graph"]["nodes"]
    convs = sum(1 for n in fused if n["op"] == "fused" and
                n["members"][0]["op"] in ("conv2d", "depthwise_conv2d"))
    assert info["sm100_nodes"] == convs  # every conv-rooted fused node ran on the GPU
    for o in _outputs(name):
        got = load_tensor(str(tmp_path), o)
        want = load_tensor(os.path.join(d, "out"), o)
        if mode == "f32":
            assert np.array_equal(got.view(np.uint32), want.view(np.uint32)), o
        else:
            assert same_values(got, want, 1e-3), o


@needs_shim
@pytest.mark.parametrize("mode", ["f32", "f32tc"])
def test_every_fused_node_on_reference_intermediates(mode):
    d = os.path.join(GRAPHS, "tiny_resnet_body")
    res = subprocess.run([SHIM, "check", os.path.join(d, "graph.json"), d, mode],
                         capture_output=True, text=True, timeout=900)
    assert res.returncode == 0, res.stderr
    info = json.loads(res.stdout)
    assert info["checked"] == 20 and info["failed"] == 0, info


@needs_shim
def test_native_eval_hook_matches_oracle(tmp_path):
    """native_conv: the OperatorDef::native_eval signature (ops.hpp:63-67)."""
    rng = np.random.default_rng(4)
    x = rng.uniform(-1, 1, (2, 16, 9, 9)).astype(np.float32)
    w = rng.uniform(-1, 1, (8, 16, 3, 3)).astype(np.float32)
    for sub, t, nm in (("x", x, "x"), ("w", w, "w")):
        os.makedirs(tmp_path / sub, exist_ok=True)
        save_tensor(str(tmp_path / sub), nm, t)
    res = subprocess.run([SHIM, "op", str(tmp_path / "x"), str(tmp_path / "w"), str(tmp_path),
                          "2", "1"], capture_output=True, text=True, timeout=300)
    assert res.returncode == 0, res.stderr
    got = load_tensor(str(tmp_path), "y")
    want = oracle_conv("conv2d", x, w, (2, 2), (1, 1), [])
    assert np.array_equal(got.view(np.uint32), want.view(np.uint32))
