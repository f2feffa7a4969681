"""Device graph executor (paper_1802_04799_b200/executor.py) and the pooling
kernels, on the GPU.

  * f32 mode (bit-exact SIMT conv path): whole graphs BIT-IDENTICAL to the
    reference's own evaluate_graph (tests/golden/graphs, written by the
    reference binary).
  * bf16 mode: against tests/graph_oracle.py's bf16 emulation (operands and
    intermediates rounded to bf16 exactly as the executor does; only the
    tensor-core accumulation order differs). Stated tolerances below.
"""
import json
import os

import numpy as np
import pytest
import torch

import graph_oracle
from oracle.oracle_api import bf16_round, global_avg_pool, load_tensor, max_pool2d
from paper_1802_04799_b200 import TecError
from paper_1802_04799_b200.executor import DeviceGraph
from paper_1802_04799_b200.graph import fuse_pass, graph_from_json
from paper_1802_04799_b200.workloads import resnet18_graph

pytestmark = pytest.mark.gpu

GRAPHS = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "graphs")
# bf16 whole-network tolerance: relative L2 error of the outputs. Per layer
# the tensor core's accumulation order moves ~1e-3 of the values by one
# bf16 ulp; measured end-to-end on ResNet-18: see DESIGN.md.
TOL_NET_BF16 = 3e-2


def _golden(name):
    d = os.path.join(GRAPHS, name)
    with open(os.path.join(d, "graph.json")) as f:
        g = graph_from_json(json.load(f))
    inputs = {n.id: load_tensor(d, n.id) for n in g.nodes if n.op == "input"}
    return d, g, inputs


def _split(dg, inputs):
    feeds = {k: v for k, v in inputs.items() if k in dg.feed_names}
    params = {k: v for k, v in inputs.items() if k in dg.param_names}
    return feeds, params


@pytest.mark.parametrize("name", ["gap_chain", "fc_head", "tiny_resnet_body"])
def test_executor_f32_bit_identical_to_reference(name):
    d, g, inputs = _golden(name)
    dg = DeviceGraph(g, compute="f32")
    feeds, params = _split(dg, inputs)
    dg.bind_params(params)
    out = dg.run(feeds)
    for o in g.outputs:
        want = load_tensor(os.path.join(d, "out"), o)
        got = out[o].reshape(want.shape)
        assert np.array_equal(got.view(np.uint32), want.view(np.uint32)), \
            f"{o}: max abs diff {np.abs(got - want).max()}"


@pytest.mark.parametrize("name", ["fc_head", "tiny_resnet_body"])
def test_executor_bf16_vs_emulation(name):
    d, g, inputs = _golden(name)
    dg = DeviceGraph(g, compute="bf16")
    feeds, params = _split(dg, inputs)
    dg.bind_params(params)
    out = dg.run(feeds)
    want = graph_oracle.evaluate(fuse_pass(g), feeds, params, "bf16")
    for o in g.outputs:
        got, w = out[o].reshape(want[o].shape), want[o]
        rel = np.linalg.norm(got - w) / max(np.linalg.norm(w), 1e-30)
        assert rel < TOL_NET_BF16, f"{o}: rel L2 {rel}"


def _resnet_inputs(g, seed=0):
    rng = np.random.default_rng(seed)
    vals = {}
    for n in g.nodes:
        if n.op != "input":
            continue
        shp = n.out_type.shape
        if n.id == "x":
            vals[n.id] = rng.uniform(-1, 1, shp).astype(np.float32)
        elif n.id.startswith("w_"):
            fan_in = int(np.prod(shp[1:])) if len(shp) == 4 else shp[0]
            vals[n.id] = (rng.standard_normal(shp) * np.sqrt(2.0 / fan_in)).astype(np.float32)
        else:
            vals[n.id] = rng.uniform(-0.1, 0.1, shp).astype(np.float32)
    return vals


def test_resnet18_bf16_end_to_end():
    """Full ResNet-18 (max_pool2d stem, global_avg_pool head), batch 2."""
    g = resnet18_graph(2)
    dg = DeviceGraph(g, compute="bf16")
    vals = _resnet_inputs(g)
    feeds, params = _split(dg, vals)
    dg.bind_params(params)
    out = dg.run(feeds)["logits"]
    want = graph_oracle.evaluate(fuse_pass(g), feeds, params, "bf16")["logits"]
    rel = np.linalg.norm(out - want) / np.linalg.norm(want)
    assert rel < TOL_NET_BF16, rel
    # CUDA-graph replay gives the same bytes as the direct launch list
    dg.capture()
    out2 = dg.run(feeds)["logits"]
    assert np.array_equal(out, out2)


def test_resnet18_batch_linearity():
    """Image i of a batch-4 run equals a batch-1 run of image i (the
    batch-sharding property the multi-GPU path relies on)."""
    g4, g1 = resnet18_graph(4), resnet18_graph(1)
    d4, d1 = DeviceGraph(g4, "bf16"), DeviceGraph(g1, "bf16")
    vals = _resnet_inputs(g4, seed=3)
    f4, p4 = _split(d4, vals)
    d4.bind_params(p4)
    d1.bind_params(p4)
    y4 = d4.run(f4)["logits"]
    for i in (0, 3):
        y1 = d1.run({"x": f4["x"][i:i + 1]})["logits"]
        assert np.array_equal(y4[i:i + 1], y1)


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
def test_max_pool2d_kernel(dtype):
    rng = np.random.default_rng(1)
    x = rng.uniform(-1, 1, (2, 64, 17, 23)).astype(np.float32)
    if dtype == "bf16":
        x = bf16_round(x)
    want = max_pool2d(x)
    from paper_1802_04799_b200.graph import ComputeGraph, GraphNode, TensorType
    # pool inside a tiny graph: conv(1x1 identity) -> max_pool2d -> conv(identity)
    nodes = [GraphNode("x", "input", out_type=TensorType([2, 64, 17, 23])),
             GraphNode("w0", "input", out_type=TensorType([64, 64, 1, 1])),
             GraphNode("w1", "input", out_type=TensorType([64, 64, 1, 1])),
             GraphNode("c0", "conv2d", ["x", "w0"]),
             GraphNode("p", "max_pool2d", ["c0"], {"kernel": [3, 3], "strides": [2, 2],
                                                  "padding": [1, 1]}),
             GraphNode("c1", "conv2d", ["p", "w1"])]
    from paper_1802_04799_b200.graph import ComputeGraph as CG
    g = CG(nodes, ["c1"])
    g.validate()
    eye = np.eye(64, dtype=np.float32)[:, :, None, None]
    dg = DeviceGraph(g, compute=dtype)
    dg.bind_params({"w0": eye, "w1": eye})
    got = dg.run({"x": x})["c1"]
    assert np.array_equal(got, want)


def test_global_avg_pool_kernel_bf16():
    rng = np.random.default_rng(2)
    x = bf16_round(rng.uniform(-1, 1, (3, 128, 7, 7)).astype(np.float32))
    from paper_1802_04799_b200.graph import ComputeGraph, GraphNode, TensorType
    nodes = [GraphNode("x", "input", out_type=TensorType([3, 128, 7, 7])),
             GraphNode("w0", "input", out_type=TensorType([128, 128, 1, 1])),
             GraphNode("c0", "conv2d", ["x", "w0"]),
             GraphNode("gap", "global_avg_pool", ["c0"])]
    g = ComputeGraph(nodes, ["gap"])
    g.validate()
    dg = DeviceGraph(g, compute="bf16")
    dg.bind_params({"w0": np.eye(128, dtype=np.float32)[:, :, None, None]})
    got = dg.run({"x": x})["gap"].reshape(3, 128)
    assert np.array_equal(got, global_avg_pool(x))


def test_unsupported_node_raises_lowering_error():
    from paper_1802_04799_b200.graph import ComputeGraph, GraphNode, TensorType
    g = ComputeGraph([GraphNode("x", "input", out_type=TensorType([4, 4])),
                      GraphNode("s", "sort", ["x"])], ["s"])
    g.validate()
    with pytest.raises(TecError) as e:
        DeviceGraph(g)
    assert e.value.code == "LoweringError"


def test_native_plan_runtime_steps_and_errors():
    """The executor's launch list is a native tec_plan: its size is the
    compiled step count, running steps one by one (tec_plan_run_steps) gives
    the same bytes as tec_plan_run, and a conv step without a kernel is
    rejected at tec_plan_create (LoweringError), not at run time."""
    import ctypes as C

    from paper_1802_04799_b200 import _abi
    g = resnet18_graph(1, width=8, head=False, maxpool=False)
    dg = DeviceGraph(g, compute="bf16")
    vals = _resnet_inputs(g, seed=5)
    feeds, params = _split(dg, vals)
    dg.bind_params(params)
    assert dg.n_launches == len(dg.steps) > 0
    out = dg.run(feeds)
    for name in dg.feed_names:
        dg.set_feed(name, feeds[name])
    for i in range(dg.n_launches):
        dg.launch_step(i)
    torch.cuda.synchronize()
    for o in dg.outputs:
        assert np.array_equal(dg.output(o).cpu().numpy(), out[o])
    lib = _abi.load()
    bad = _abi.Step(kind=_abi.STEP_CONV, dst_dtype=_abi.DT_BF16, conv=dg.steps[0].conv)
    bad.conv.compute = 99  # no such compute mode
    h = C.c_void_p()
    st = lib.tec_plan_create((_abi.Step * 1)(bad), 1, C.byref(h))
    assert st != 0 and not h.value
    assert lib.tec_plan_run_steps(dg._native, dg.n_launches, 1, None) != 0  # out of range


# f32tc whole-network bar: per conv the 1e-4 comparator holds (node by node,
# tests/test_integration_gpu.py); through a network the differences compound
TOL_NET_F32TC = 1e-3


@pytest.mark.parametrize("name", ["fc_head", "tiny_resnet_body"])
def test_executor_f32tc_vs_reference(name):
    """Reference precision on the tensor cores: every conv of the graph in
    f32tc, against the reference's own evaluate_graph output."""
    from oracle.oracle_api import same_values
    d, g, inputs = _golden(name)
    dg = DeviceGraph(g, compute="f32tc")
    feeds, params = _split(dg, inputs)
    dg.bind_params(params)
    out = dg.run(feeds)
    for o in g.outputs:
        want = load_tensor(os.path.join(d, "out"), o)
        assert same_values(out[o].reshape(want.shape), want, TOL_NET_F32TC), o


def test_resnet18_f32tc_end_to_end():
    """Full ResNet-18 at batch 2, f32 on the tensor cores, vs the f32 graph
    oracle (the reference's arithmetic), captured replay bit-stable."""
    from oracle.oracle_api import same_values
    g = resnet18_graph(2)
    dg = DeviceGraph(g, compute="f32tc")
    vals = _resnet_inputs(g)
    feeds, params = _split(dg, vals)
    dg.bind_params(params)
    out = dg.run(feeds)["logits"]
    want = graph_oracle.evaluate(fuse_pass(g), feeds, params, "f32")["logits"]
    assert same_values(out, want, TOL_NET_F32TC)
    dg.capture()
    assert np.array_equal(out, dg.run(feeds)["logits"])
