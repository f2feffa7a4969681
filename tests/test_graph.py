"""Graph API (paper_1802_04799_b200/graph.py) against the reference's graph
passes, pinned by tests/golden/graphs/*/fused.json (written by the reference's
fuse_pass + plan_memory, R/src/graph_passes.cpp:196-329, via
oracle/_ref/ref_driver). CPU only."""
import json
import os

import numpy as np
import pytest

import graph_oracle
from oracle.oracle_api import load_tensor
from paper_1802_04799_b200 import TecError
from paper_1802_04799_b200.graph import (ComputeGraph, GraphNode, TensorType, check_memory_plan,
                                         fuse_pass, graph_from_json, graph_to_json, plan_memory)
from paper_1802_04799_b200.workloads import resnet18_graph

GRAPHS = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "graphs")
NAMES = sorted(os.listdir(GRAPHS))


def _load(name):
    d = os.path.join(GRAPHS, name)
    with open(os.path.join(d, "graph.json")) as f:
        g = json.load(f)
    with open(os.path.join(d, "fused.json")) as f:
        fused = json.load(f)
    return d, g, fused


def _shape_of(node):
    return (node["id"], node["op"], list(node.get("inputs", [])),
            [(m["id"], m["op"], m.get("inputs", [])) for m in node.get("members", [])])


@pytest.mark.parametrize("name", NAMES)
def test_fuse_pass_matches_reference(name):
    _, gj, fused = _load(name)
    ours = graph_to_json(fuse_pass(graph_from_json(gj)))
    ref = fused["graph"]
    assert [_shape_of(n) for n in ours["nodes"]] == [_shape_of(n) for n in ref["nodes"]]
    assert ours["outputs"] == ref["outputs"]


@pytest.mark.parametrize("name", NAMES)
def test_plan_memory_matches_reference(name):
    _, gj, fused = _load(name)
    f = fuse_pass(graph_from_json(gj))
    p = plan_memory(f)
    check_memory_plan(f, p)
    ref = fused["plan"]
    assert p.slot_of == ref["slot_of"]
    assert p.slot_bytes == ref["slot_bytes"]
    assert p.total_bytes == ref["total_bytes"]
    assert p.naive_bytes == ref["naive_bytes"]


@pytest.mark.parametrize("name", NAMES)
def test_json_round_trip(name):
    _, gj, _ = _load(name)
    g = graph_from_json(gj)
    again = graph_from_json(json.dumps(graph_to_json(g)))
    assert graph_to_json(again) == graph_to_json(g)


def test_const_payload_round_trip():
    g = ComputeGraph([GraphNode("c", "const", out_type=TensorType([2, 3], "f32"),
                                data=np.arange(6, dtype=np.float32).reshape(2, 3)),
                      GraphNode("r", "relu", ["c"])], ["r"])
    g.validate()
    again = graph_from_json(graph_to_json(g))
    assert np.array_equal(again.node("c").data, g.node("c").data)


def test_resnet18_fusion_shape():
    f = fuse_pass(resnet18_graph(2))
    fused = [n for n in f.nodes if n.op == "fused"]
    convs = [n for n in fused if n.members[0].op == "conv2d"]
    assert len(convs) == 20  # every conv of ResNet-18 is one fused node
    assert sum(1 for n in convs if [m.op for m in n.members] ==
               ["conv2d", "bias_add", "add", "relu"]) == 8  # block tails
    assert [m.op for m in fused[-1].members] == ["matmul", "bias_add"]
    p = plan_memory(f)
    check_memory_plan(f, p)
    assert p.total_bytes < p.naive_bytes / 2


def test_validate_errors():
    base = [GraphNode("x", "input", out_type=TensorType([1, 4, 5, 5])),
            GraphNode("w", "input", out_type=TensorType([8, 3, 3, 3]))]
    g = ComputeGraph(base + [GraphNode("c", "conv2d", ["x", "w"])], ["c"])
    with pytest.raises(TecError) as e:
        g.validate()
    assert e.value.code == "ShapeMismatch"
    g = ComputeGraph([GraphNode("r", "relu", ["x"])] + base, ["r"])
    with pytest.raises(TecError):
        g.validate()
    g = ComputeGraph(base + [GraphNode("x", "relu", ["x"])], ["x"])
    with pytest.raises(TecError):
        g.validate()
    with pytest.raises(TecError):
        ComputeGraph(base, []).validate()


def test_memory_plan_checker_catches_clobber():
    f = fuse_pass(resnet18_graph(1, image=64, width=8))
    p = plan_memory(f)
    check_memory_plan(f, p)
    # force two simultaneously-live tensors into one slot
    ids = [n.id for n in f.nodes if n.id in p.slot_of]
    p.slot_of[ids[1]] = p.slot_of[ids[0]]
    with pytest.raises(TecError):
        check_memory_plan(f, p)


@pytest.mark.parametrize("name", ["gap_chain", "fc_head", "tiny_resnet_body"])
def test_graph_oracle_matches_reference_eval(name):
    """The test-side graph evaluator (oracle restatement) is bit-identical
    to the reference's evaluate_graph on these graphs."""
    d, gj, _ = _load(name)
    g = graph_from_json(gj)
    f = fuse_pass(g)
    inputs = {n.id: load_tensor(d, n.id) for n in g.nodes if n.op == "input"}
    got = graph_oracle.evaluate(f, inputs, {}, "f32")
    for o in g.outputs:
        want = load_tensor(os.path.join(d, "out"), o)
        assert np.array_equal(got[o].reshape(want.shape).view(np.uint32), want.view(np.uint32)), o


def test_tensor_io_reads_reference_files_and_round_trips(tmp_path):
    from paper_1802_04799_b200.graph import load_tensor as gl, save_tensor as gs
    d = os.path.join(GRAPHS, "tiny_resnet_body")
    x = gl(d, "x")
    assert x.dtype == np.float32 and np.array_equal(x, load_tensor(d, "x"))
    for arr in (x, np.arange(-5, 5, dtype=np.int8).reshape(2, 5), np.arange(6, dtype=np.int32)):
        gs(str(tmp_path), "t", arr)
        back = gl(str(tmp_path), "t")
        assert back.dtype == arr.dtype and np.array_equal(back, arr)
    with pytest.raises(TecError) as e:
        gl(str(tmp_path), "missing")
    assert e.value.code == "IOError"
