"""f4: the NHWC layout pass and batch-norm folding.

nhwc_layout_pass is apply_layouts (R/src/graph_passes.cpp:84-178) with an
"nhwc" preference on every rank-4 device op: transforms appear only where
an activation crosses between the reference NCHW layout and the kernels'
NHWC one. fold_batch_norm rewrites conv -> [bias_add] -> batch_norm into
conv(bn_fold_weight(W)) -> bias_add(bn_fold_bias(B)); the fold nodes are
parameter computations, constant-folded at compile time (fold_constants) or
folded inside tec_weight_pretransform_bn at bind time on the device.

CPU: pass structure, fusion, constant folding, folded-vs-unfolded numerics.
GPU: the executor on BN graphs -- f32 bit-exact against the oracle
evaluation of the folded graph, f32tc / bf16 within their bars."""
import numpy as np
import pytest

import graph_oracle
from oracle.oracle_api import fused_conv, same_values
from paper_1802_04799_b200._abi import TecError
from paper_1802_04799_b200.graph import (ComputeGraph, GraphNode, TensorType, apply_layouts,
                                         bn_eval, fold_batch_norm, fold_constants, fuse_pass,
                                         nhwc_layout_pass)
from paper_1802_04799_b200.workloads import resnet18_graph


def _bn_graph(const_params=False, with_bias=True, k=32, c=16, hw=10):
    """x -> conv(3x3) [-> bias_add] -> batch_norm -> relu -> conv(1x1) -> batch_norm (output)."""
    rng = np.random.default_rng(3)
    vals = {"w1": rng.standard_normal((k, c, 3, 3)).astype(np.float32) * 0.2,
            "b1": rng.uniform(-0.1, 0.1, k).astype(np.float32),
            "w2": rng.standard_normal((k, k, 1, 1)).astype(np.float32) * 0.2}
    for j in (1, 2):
        vals[f"g{j}"] = rng.uniform(0.5, 1.5, k).astype(np.float32)
        vals[f"be{j}"] = rng.uniform(-0.2, 0.2, k).astype(np.float32)
        vals[f"mu{j}"] = rng.uniform(-0.3, 0.3, k).astype(np.float32)
        vals[f"var{j}"] = rng.uniform(0.2, 2.0, k).astype(np.float32)
    kind = "const" if const_params else "input"
    nodes = [GraphNode("x", "input", out_type=TensorType([2, c, hw, hw], "f32"))]
    for name, v in vals.items():
        nd = GraphNode(name, kind, out_type=TensorType(list(v.shape), "f32"))
        if const_params:
            nd.data = v
        nodes.append(nd)
    nodes.append(GraphNode("c1", "conv2d", ["x", "w1"], {"padding": [1, 1]}))
    y = "c1"
    if with_bias:
        nodes.append(GraphNode("c1b", "bias_add", ["c1", "b1"]))
        y = "c1b"
    nodes += [GraphNode("bn1", "batch_norm", [y, "g1", "be1", "mu1", "var1"], {"eps": 1e-5}),
              GraphNode("r1", "relu", ["bn1"]),
              GraphNode("c2", "conv2d", ["r1", "w2"]),
              GraphNode("bn2", "batch_norm", ["c2", "g2", "be2", "mu2", "var2"], {"eps": 1e-3})]
    g = ComputeGraph(nodes, ["bn2"])
    g.validate()
    feeds = {"x": rng.uniform(-1, 1, (2, c, hw, hw)).astype(np.float32)}
    return g, feeds, vals


# ------------------------------------------------------------------ CPU
def test_fold_batch_norm_structure_and_fusion():
    for with_bias in (True, False):
        g, _, _ = _bn_graph(with_bias=with_bias)
        f = fold_batch_norm(g)
        ops = [n.op for n in f.nodes if n.op not in ("input", "const")]
        assert "batch_norm" not in ops
        assert ops.count("bn_fold_weight") == 2 and ops.count("bn_fold_bias") == 2
        assert f.node("bn1").op == "bias_add" and f.node("bn2").op == "bias_add"
        fused = fuse_pass(f)
        groups = [[m.op for m in n.members] for n in fused.nodes if n.op == "fused"]
        # the parameter folds stay out of the conv groups
        assert ["conv2d", "bias_add", "relu"] in groups and ["conv2d", "bias_add"] in groups


def test_fold_constants_evaluates_the_folds():
    g, _, vals = _bn_graph(const_params=True)
    f = fold_constants(fold_batch_norm(g))
    w1 = f.node("c1").inputs[1]
    assert f.node(w1).op == "const"
    want = bn_eval("bn_fold_weight", [vals["w1"], vals["g1"], vals["var1"]], 1e-5)
    assert np.array_equal(f.node(w1).data, want)
    b1 = f.node("bn1").inputs[1]
    want_b = bn_eval("bn_fold_bias", [vals["b1"], vals["g1"], vals["be1"], vals["mu1"],
                                      vals["var1"]], 1e-5)
    assert np.array_equal(f.node(b1).data, want_b)


def test_folded_graph_matches_the_unfolded_batch_norm():
    """The fold changes only rounding: folded vs the literal batch_norm
    evaluation (oracle conv + bn_eval) agree to f32 accumulation noise."""
    g, feeds, vals = _bn_graph()
    x = feeds["x"]
    y1 = fused_conv("conv2d", x, vals["w1"], (1, 1), (1, 1), [("bias_add", vals["b1"])])
    y1 = bn_eval("batch_norm", [y1, vals["g1"], vals["be1"], vals["mu1"], vals["var1"]], 1e-5)
    y1 = np.maximum(y1, 0)
    y2 = fused_conv("conv2d", y1, vals["w2"], (1, 1), (0, 0), [])
    unfolded = bn_eval("batch_norm", [y2, vals["g2"], vals["be2"], vals["mu2"], vals["var2"]], 1e-3)
    folded = graph_oracle.evaluate(fuse_pass(fold_batch_norm(g)), feeds, vals, "f32")["bn2"]
    assert same_values(folded, unfolded, 1e-5)


def test_nhwc_layout_pass_places_transforms_at_the_boundary():
    for g in (resnet18_graph(1, image=64, width=8),
              resnet18_graph(1, image=64, width=32, head=False, dtype="i8")):
        f = fuse_pass(g)
        laid = nhwc_layout_pass(f)
        tr = [n for n in laid.nodes if n.op == "layout_transform"]
        srcs = {n.inputs[0] for n in tr}
        # the image enters NHWC once; weights and biases are never transformed
        assert "x" in srcs and not any(s.startswith(("w_", "b_")) for s in srcs)
        assert len(tr) == 2
        for n in laid.nodes:
            if n.op == "fused" and n.members[0].op == "conv2d":
                assert n.id.endswith("#h")
        # outputs keep their ids and are row-major
        assert set(laid.outputs) == set(g.outputs)
        out = laid.node(g.outputs[0])
        if g.outputs[0] != "logits":
            assert out.op == "layout_transform" and out.attrs["dst_layout"] == "row_major"


def test_nhwc_preference_rules():
    g, _, _ = _bn_graph()
    with pytest.raises(TecError):
        apply_layouts(g, {"w1": "nhwc"})  # an input
    nodes = [GraphNode("a", "input", out_type=TensorType([4, 4])),
             GraphNode("r", "relu", ["a"])]
    g2 = ComputeGraph(nodes, ["r"])
    g2.validate()
    with pytest.raises(TecError):
        apply_layouts(g2, {"r": "nhwc"})  # rank 2
    with pytest.raises(TecError):
        apply_layouts(g2, {"r": "nchw9"})


# ------------------------------------------------------------------ GPU
@pytest.mark.gpu
@pytest.mark.parametrize("compute", ["f32", "f32tc", "bf16"])
def test_executor_runs_batch_norm_graphs(compute):
    from paper_1802_04799_b200.executor import DeviceGraph
    g, feeds, vals = _bn_graph()
    dg = DeviceGraph(g, compute=compute)
    dg.bind_params(vals)
    got = dg.run(feeds)["bn2"]
    folded = fuse_pass(fold_batch_norm(g))
    if compute == "f32":
        # the device folds W * s with one f32 product, as the oracle does
        want = graph_oracle.evaluate(folded, feeds, vals, "f32")["bn2"]
        assert np.array_equal(got.view(np.uint32), want.view(np.uint32))
    elif compute == "f32tc":
        want = graph_oracle.evaluate(folded, feeds, vals, "f32")["bn2"]
        assert same_values(got, want, 1e-4)
    else:
        want = graph_oracle.evaluate(folded, feeds, vals, "bf16")["bn2"]
        rel = np.linalg.norm(got - want) / np.linalg.norm(want)
        assert rel < 3e-2, rel


@pytest.mark.gpu
def test_executor_bn_resnet_block_f32():
    """conv -> batch_norm -> relu -> conv -> batch_norm -> add(shortcut) -> relu,
    the residual block the way frameworks export it: folded on the device,
    bit-identical in f32 to the oracle evaluation of the folded graph."""
    from paper_1802_04799_b200.executor import DeviceGraph
    rng = np.random.default_rng(8)
    c = 32
    vals = {"w1": (rng.standard_normal((c, c, 3, 3)) * 0.1).astype(np.float32),
            "w2": (rng.standard_normal((c, c, 3, 3)) * 0.1).astype(np.float32)}
    nodes = [GraphNode("x", "input", out_type=TensorType([2, c, 12, 12], "f32"))]
    for name in ("w1", "w2"):
        nodes.append(GraphNode(name, "input", out_type=TensorType([c, c, 3, 3], "f32")))
    for j in (1, 2):
        for nm, lo, hi in (("g", 0.5, 1.5), ("be", -0.2, 0.2), ("mu", -0.3, 0.3), ("var", 0.2, 2.0)):
            vals[f"{nm}{j}"] = rng.uniform(lo, hi, c).astype(np.float32)
            nodes.append(GraphNode(f"{nm}{j}", "input", out_type=TensorType([c], "f32")))
    nodes += [GraphNode("c1", "conv2d", ["x", "w1"], {"padding": [1, 1]}),
              GraphNode("bn1", "batch_norm", ["c1", "g1", "be1", "mu1", "var1"]),
              GraphNode("r1", "relu", ["bn1"]),
              GraphNode("c2", "conv2d", ["r1", "w2"], {"padding": [1, 1]}),
              GraphNode("bn2", "batch_norm", ["c2", "g2", "be2", "mu2", "var2"]),
              GraphNode("a", "add", ["bn2", "x"]),
              GraphNode("r2", "relu", ["a"])]
    g = ComputeGraph(nodes, ["r2"])
    g.validate()
    feeds = {"x": rng.uniform(-1, 1, (2, c, 12, 12)).astype(np.float32)}
    dg = DeviceGraph(g, compute="f32")
    dg.bind_params(vals)
    got = dg.run(feeds)["r2"]
    want = graph_oracle.evaluate(fuse_pass(fold_batch_norm(g)), feeds, vals, "f32")["r2"]
    assert np.array_equal(got.view(np.uint32), want.view(np.uint32))
