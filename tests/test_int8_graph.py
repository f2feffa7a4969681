"""int8 graphs end to end: the int8 ResNet-18 body -- i8
activations between layers, i32 accumulation, requantize after every relu'd
conv, identity shortcuts as scale(cast(y, i32)) -- through the device
executor (compute "i8"), bit-exact against tests/graph_oracle.py (the conv
through the oracle restatement, every fused member evaluated one by one in
member order as R/src/graph.cpp:209-222 does).

CPU: graph construction and fusion, the op type rules, constant folding of
the new ops, the C ABI's program validation. GPU: tec_elementwise against
numpy, whole networks bit-exact, captured replay, overflow reporting."""
import ctypes as C

import numpy as np
import pytest

import graph_oracle
from paper_1802_04799_b200 import _abi
from paper_1802_04799_b200._abi import TecError
from paper_1802_04799_b200.executor import split_conv_members
from paper_1802_04799_b200.graph import ComputeGraph, GraphNode, TensorType, fold_constants, fuse_pass
from paper_1802_04799_b200.workloads import int8_resnet18_params, resnet18_graph


def _small(batch=2, image=64, width=16):
    g = resnet18_graph(batch, image=image, width=width, head=False, dtype="i8")
    feeds, params = int8_resnet18_params(g, seed=batch + width)
    return g, feeds, params


# ------------------------------------------------------------------ CPU
def test_int8_graph_fuses_one_node_per_conv():
    f = fuse_pass(resnet18_graph(1, image=64, width=16, head=False, dtype="i8"))
    convs = [n for n in f.nodes if n.op == "fused"]
    assert len(convs) == 20
    kinds = {tuple(m.op for m in n.members) for n in convs}
    assert kinds == {
        ("conv2d", "bias_add", "relu", "requantize"),
        ("conv2d", "bias_add", "cast", "scale", "add", "relu", "requantize"),  # block with shortcut
        ("conv2d", "bias_add", "requantize"),                                 # the downsample
    }
    for n in convs:
        root, head, sides, tail = split_conv_members(n)
        assert root.op == "conv2d"
        assert [m.op for m in tail] == ["requantize"]
        assert all(m.op in ("bias_add", "add", "relu") for m in head)
        for first, last, members in sides:
            assert [m.op for m in members] == ["cast", "scale"] and first not in {m.id for m in n.members}
        assert n.out_type.dtype == "i8"


def test_int8_graph_rejects_head_and_bad_ops():
    with pytest.raises(ValueError):
        resnet18_graph(1, dtype="i8")
    x = GraphNode("x", "input", out_type=TensorType([4], "f32"))
    for op, attrs in (("requantize", {"multiplier": 3, "shift": 2}),   # f32 data
                      ("cast", {"dtype": "i8"})):                      # f32 -> i8
        g = ComputeGraph([x, GraphNode("y", op, ["x"], attrs)], ["y"])
        with pytest.raises(TecError):
            g.validate()
    xi = GraphNode("x", "input", out_type=TensorType([4], "i32"))
    for attrs in ({"multiplier": 0, "shift": 2}, {"multiplier": 2 ** 31, "shift": 2},
                  {"multiplier": 3, "shift": 63}, {"multiplier": 1.5, "shift": 2}):
        g = ComputeGraph([xi, GraphNode("y", "requantize", ["x"], attrs)], ["y"])
        with pytest.raises(TecError):
            g.validate()


def test_fold_constants_matches_the_oracle_restatement():
    """Constant folding of cast / requantize (graph.py _fold_eval) equals the
    oracle's member evaluation, including ties and clamping."""
    vals = np.array([-2 ** 31, -70000, -384, -129, -128, -3, -2, -1, 0, 1, 2, 3, 127, 128,
                     383, 384, 70000, 2 ** 31 - 1], np.int32)
    for mult, shift in ((1, 0), (1, 1), (3, 2), (12345, 16), (2 ** 31 - 1, 40)):
        nodes = [GraphNode("c", "const", out_type=TensorType([vals.size], "i32")),
                 GraphNode("q", "requantize", ["c"], {"multiplier": mult, "shift": shift}),
                 GraphNode("w", "cast", ["q"], {"dtype": "i32"}),
                 GraphNode("x", "input", out_type=TensorType([vals.size], "i32")),
                 GraphNode("y", "add", ["x", "w"])]
        nodes[0].data = vals.copy()
        g = ComputeGraph(nodes, ["y"])
        g.validate()
        folded = fold_constants(g)
        cst = [n for n in folded.nodes if n.op == "const"]
        assert len(cst) == 1
        env = {"c": vals}
        want = graph_oracle._int_member(nodes[1], env)
        env["q"] = want
        want = graph_oracle._int_member(nodes[2], env)
        assert np.array_equal(np.asarray(cst[0].data).reshape(-1), want), (mult, shift)


def _prog(kinds, src, dst, **kw):
    p = _abi.ElemProg(n_ops=len(kinds), src_dtype=src, dst_dtype=dst, count=kw.get("count", 16))
    for i, k in enumerate(kinds):
        p.kind[i] = k
        p.cast_to[i] = kw.get("cast_to", _abi.DT_I32)
        p.mult[i] = kw.get("mult", 1)
        p.shift[i] = kw.get("shift", 0)
        p.scale[i] = kw.get("scale", 1.0)
    return p


@pytest.mark.parametrize("kinds,src,dst,kw", [
    ([_abi.ELEM_REQUANTIZE], _abi.DT_I8, _abi.DT_I8, {}),               # requantize of i8 data
    ([_abi.ELEM_REQUANTIZE], _abi.DT_I32, _abi.DT_I32, {}),             # chain ends in i8
    ([_abi.ELEM_REQUANTIZE], _abi.DT_I32, _abi.DT_I8, {"mult": 0}),     # multiplier range
    ([_abi.ELEM_REQUANTIZE], _abi.DT_I32, _abi.DT_I8, {"shift": 63}),   # shift range
    ([_abi.ELEM_SCALE], _abi.DT_I32, _abi.DT_I32, {"scale": 2.5}),      # non-integral factor
    ([_abi.ELEM_SCALE], _abi.DT_I8, _abi.DT_I8, {"scale": 2.0}),        # scale of i8 data
    ([_abi.ELEM_CAST], _abi.DT_I32, _abi.DT_I8, {"cast_to": _abi.DT_I8}),  # narrowing cast
    ([9], _abi.DT_I32, _abi.DT_I32, {}),                                # unknown member
    ([_abi.ELEM_RELU] * 5, _abi.DT_I32, _abi.DT_I32, {}),               # too many members
])
def test_elementwise_abi_rejects_bad_programs(kinds, src, dst, kw):
    lib = _abi.load()
    p = _prog(kinds[:4], src, dst, **kw)
    if len(kinds) > 4:
        p.n_ops = len(kinds)
    st = lib.tec_elementwise(C.byref(p), None, None, None, None)
    assert st in (2, 15), st  # ShapeMismatch / LoweringError, before any launch


# ------------------------------------------------------------------ GPU
def _dev():
    import torch
    return torch.device("cuda", 0)


@pytest.mark.gpu
def test_elementwise_kernel_matches_numpy():
    import torch
    lib = _abi.load()
    rng = np.random.default_rng(5)
    st = torch.cuda.current_stream().cuda_stream
    for count in (1, 15, 16, 17, 4096 + 7, 1 << 20):
        x32 = rng.integers(-2 ** 31, 2 ** 31, count, dtype=np.int64).astype(np.int32)
        x32[: min(count, 8)] = [-384, -383, -129, -128, 127, 128, 383, 384][: min(count, 8)]
        xi8 = rng.integers(-128, 128, count, dtype=np.int8)
        err = torch.zeros(1, dtype=torch.int32, device=_dev())
        cases = [
            ([_abi.ELEM_REQUANTIZE], x32, np.int8, {"mult": 3, "shift": 2}),
            ([_abi.ELEM_RELU, _abi.ELEM_REQUANTIZE], x32, np.int8, {"mult": 12345, "shift": 30}),
            ([_abi.ELEM_CAST, _abi.ELEM_SCALE], xi8, np.int32, {"scale": 1000.0}),
            ([_abi.ELEM_CAST], xi8, np.float32, {"cast_to": _abi.DT_F32}),
        ]
        dt = {np.dtype(np.int8): _abi.DT_I8, np.dtype(np.int32): _abi.DT_I32,
              np.dtype(np.float32): _abi.DT_F32}
        for kinds, x, out_np, kw in cases:
            p = _prog(kinds, dt[x.dtype], dt[np.dtype(out_np)], count=count, **kw)
            xd = torch.from_numpy(x).to(_dev())
            yd = torch.empty(count, dtype={np.int8: torch.int8, np.int32: torch.int32,
                                           np.float32: torch.float32}[out_np], device=_dev())
            _abi.check(lib.tec_elementwise(C.byref(p), xd.data_ptr(), yd.data_ptr(),
                                           err.data_ptr(), st))
            env = {"x": x}
            for i, k in enumerate(kinds):
                op = {_abi.ELEM_CAST: "cast", _abi.ELEM_SCALE: "scale", _abi.ELEM_RELU: "relu",
                      _abi.ELEM_REQUANTIZE: "requantize"}[k]
                attrs = {"multiplier": kw.get("mult", 1), "shift": kw.get("shift", 0),
                         "scale": kw.get("scale", 1.0),
                         "dtype": "f32" if kw.get("cast_to") == _abi.DT_F32 else "i32"}
                m = GraphNode(f"m{i}", op, ["x" if i == 0 else f"m{i - 1}"], attrs)
                env[m.id] = graph_oracle._int_member(m, env)
            want = env[f"m{len(kinds) - 1}"]
            assert np.array_equal(yd.cpu().numpy(), want), (kinds, count)
        assert int(err.item()) == 0
    # i32 range overflow raises the flag
    p = _prog([_abi.ELEM_CAST, _abi.ELEM_SCALE], _abi.DT_I8, _abi.DT_I32, count=64,
              scale=float(2 ** 25))
    xd = torch.full((64,), 127, dtype=torch.int8, device=_dev())
    yd = torch.empty(64, dtype=torch.int32, device=_dev())
    _abi.check(lib.tec_elementwise(C.byref(p), xd.data_ptr(), yd.data_ptr(), err.data_ptr(), st))
    assert int(err.item()) == 1


@pytest.mark.gpu
@pytest.mark.parametrize("width,image,batch", [(16, 64, 2), (64, 64, 2), (64, 224, 2)])
def test_int8_resnet18_bit_exact(width, image, batch):
    """The whole int8 body vs the oracle, bit for bit; width 16 exercises the
    i8 NHWC -> padded-channel repack (16 channels, int8 blocks are >= 32)."""
    from paper_1802_04799_b200.executor import DeviceGraph
    g, feeds, params = _small(batch, image, width)
    dg = DeviceGraph(g, compute="i8")
    dg.bind_params(params)
    out = dg.run(feeds)
    want = graph_oracle.evaluate(fuse_pass(g), feeds, params, "i8")
    for o in g.outputs:
        assert out[o].dtype == np.int8
        assert np.array_equal(out[o], want[o]), o
    dg.capture()
    again = dg.run(feeds)
    for o in g.outputs:
        assert np.array_equal(again[o], out[o])


@pytest.mark.gpu
@pytest.mark.parametrize("k,shortcut", [(24, False), (48, True), (64, True)])
def test_int8_block_fused_and_unfused_lowerings(k, shortcut):
    """One conv block in both lowerings: K = 24 keeps requantize (and the
    shortcut) as elementwise launches; K = 48 folds requantize into the
    epilogue with the shortcut as an i32 operand (the generic epilogue);
    K = 64 folds both (the Q programs). All bit-exact vs the oracle."""
    from paper_1802_04799_b200.executor import DeviceGraph
    rng = np.random.default_rng(k)
    # a 1x1 conv first, so the block input (and its shortcut) is an NHWC
    # activation rather than the NCHW graph input
    nodes = [GraphNode("x0", "input", out_type=TensorType([2, k, 12, 12], "i8")),
             GraphNode("w0", "input", out_type=TensorType([k, k, 1, 1], "i8")),
             GraphNode("c0", "conv2d", ["x0", "w0"]),
             GraphNode("x", "requantize", ["c0"], {"multiplier": 3, "shift": 4}),
             GraphNode("w", "input", out_type=TensorType([k, k, 3, 3], "i8")),
             GraphNode("b", "input", out_type=TensorType([k], "i32")),
             GraphNode("c", "conv2d", ["x", "w"], {"padding": [1, 1]}),
             GraphNode("cb", "bias_add", ["c", "b"])]
    y = "cb"
    if shortcut:
        nodes += [GraphNode("sc", "cast", ["x"], {"dtype": "i32"}),
                  GraphNode("ss", "scale", ["sc"], {"scale": 37.0}),
                  GraphNode("a", "add", [y, "ss"])]
        y = "a"
    nodes += [GraphNode("r", "relu", [y]),
              GraphNode("q", "requantize", ["r"], {"multiplier": 911, "shift": 16})]
    g = ComputeGraph(nodes, ["q"])
    g.validate()
    feeds = {"x0": rng.integers(-60, 61, (2, k, 12, 12), dtype=np.int8)}
    params = {"w0": rng.integers(-8, 9, (k, k, 1, 1), dtype=np.int8),
              "w": rng.integers(-8, 9, (k, k, 3, 3), dtype=np.int8),
              "b": rng.integers(-500, 501, (k,), dtype=np.int32)}
    dg = DeviceGraph(g, compute="i8")
    dg.bind_params(params)
    got = dg.run(feeds)["q"]
    want = graph_oracle.evaluate(fuse_pass(g), feeds, params, "i8")["q"]
    assert np.array_equal(got, want)
    assert 0 < (got == 0).mean() < 1 and (got > 0).any()
    n_elem = sum(1 for s in dg.steps if s.kind == _abi.STEP_ELEMWISE)
    # K = 24: both requantizes and the shortcut unfused; 48: the shortcut
    # (K % 32 != 0); 64: none
    assert n_elem == {24: 2 + shortcut, 48: 1, 64: 0}[k]


@pytest.mark.gpu
@pytest.mark.parametrize("mult,shift", [(911, 16), (2 ** 31 - 1, 40), (5, 1), (1, 0), (3, 32)])
def test_int8_requantize_epilogue_parameters(mult, shift):
    """The fused requantize (Q epilogue) for multiplier / shift pairs on both
    sides of its fast form (m < 2^shift <= 2^32: one 32x32 high product)."""
    from paper_1802_04799_b200.executor import DeviceGraph
    rng = np.random.default_rng(mult % 97 + shift)
    k = 64
    nodes = [GraphNode("x", "input", out_type=TensorType([2, k, 10, 10], "i8")),
             GraphNode("w", "input", out_type=TensorType([k, k, 3, 3], "i8")),
             GraphNode("b", "input", out_type=TensorType([k], "i32")),
             GraphNode("c", "conv2d", ["x", "w"], {"padding": [1, 1]}),
             GraphNode("cb", "bias_add", ["c", "b"]),
             GraphNode("r", "relu", ["cb"]),
             GraphNode("q", "requantize", ["r"], {"multiplier": mult, "shift": shift})]
    g = ComputeGraph(nodes, ["q"])
    g.validate()
    feeds = {"x": rng.integers(-60, 61, (2, k, 10, 10), dtype=np.int8)}
    params = {"w": rng.integers(-8, 9, (k, k, 3, 3), dtype=np.int8),
              "b": rng.integers(-2000, 2001, (k,), dtype=np.int32)}
    dg = DeviceGraph(g, compute="i8")
    dg.bind_params(params)
    assert sum(1 for st in dg.steps if st.kind == _abi.STEP_ELEMWISE) == 0  # fused
    got = dg.run(feeds)["q"]
    want = graph_oracle.evaluate(fuse_pass(g), feeds, params, "i8")["q"]
    assert np.array_equal(got, want)


@pytest.mark.gpu
def test_int8_depthwise_block():
    """A MobileNet-style int8 block: depthwise 3x3 + bias + relu + requantize
    (the depthwise kernels take no requantize epilogue: the tail runs as an
    elementwise launch) -> pointwise 1x1 + bias + relu + requantize (fused)."""
    from paper_1802_04799_b200.executor import DeviceGraph
    rng = np.random.default_rng(11)
    c, k = 64, 96
    nodes = [GraphNode("x", "input", out_type=TensorType([2, c, 14, 14], "i8")),
             GraphNode("wd", "input", out_type=TensorType([c, 1, 3, 3], "i8")),
             GraphNode("bd", "input", out_type=TensorType([c], "i32")),
             GraphNode("wp", "input", out_type=TensorType([k, c, 1, 1], "i8")),
             GraphNode("bp", "input", out_type=TensorType([k], "i32")),
             GraphNode("d", "depthwise_conv2d", ["x", "wd"], {"padding": [1, 1]}),
             GraphNode("db", "bias_add", ["d", "bd"]),
             GraphNode("dr", "relu", ["db"]),
             GraphNode("dq", "requantize", ["dr"], {"multiplier": 1500, "shift": 12}),
             GraphNode("p", "conv2d", ["dq", "wp"]),
             GraphNode("pb", "bias_add", ["p", "bp"]),
             GraphNode("pr", "relu", ["pb"]),
             GraphNode("pq", "requantize", ["pr"], {"multiplier": 700, "shift": 14})]
    g = ComputeGraph(nodes, ["pq"])
    g.validate()
    feeds = {"x": rng.integers(-50, 51, (2, c, 14, 14), dtype=np.int8)}
    params = {"wd": rng.integers(-8, 9, (c, 1, 3, 3), dtype=np.int8),
              "bd": rng.integers(-200, 201, (c,), dtype=np.int32),
              "wp": rng.integers(-8, 9, (k, c, 1, 1), dtype=np.int8),
              "bp": rng.integers(-200, 201, (k,), dtype=np.int32)}
    dg = DeviceGraph(g, compute="i8")
    dg.bind_params(params)
    got = dg.run(feeds)["pq"]
    want = graph_oracle.evaluate(fuse_pass(g), feeds, params, "i8")["pq"]
    assert np.array_equal(got, want)
    assert 0 < (got == 0).mean() < 1


@pytest.mark.gpu
def test_max_pool2d_i8_kernel():
    """tec_max_pool2d on i8 NHWC (the int8 stem pool, SIMD byte max):
    all-negative values, so a padded tap winning would show as 0."""
    import torch
    from oracle.oracle_api import max_pool2d
    lib = _abi.load()
    rng = np.random.default_rng(9)
    n, c, h, w = 3, 48, 17, 23
    x = rng.integers(-128, 0, (n, c, h, w), dtype=np.int8)
    x[0, :, 0, 0] = -128
    want = max_pool2d(x).astype(np.int8)
    xd = torch.from_numpy(np.ascontiguousarray(x.transpose(0, 2, 3, 1))).to(_dev())
    oh, ow = want.shape[2], want.shape[3]
    yd = torch.empty((n, oh, ow, c), dtype=torch.int8, device=_dev())
    pd = _abi.PoolDesc(n=n, c=c, h=h, w=w, r=3, s=3, stride_h=2, stride_w=2, pad_h=1, pad_w=1,
                       dtype=_abi.DT_I8, out_dtype=_abi.DT_I8)
    _abi.check(lib.tec_max_pool2d(C.byref(pd), xd.data_ptr(), yd.data_ptr(),
                                  torch.cuda.current_stream().cuda_stream))
    got = yd.cpu().numpy().transpose(0, 3, 1, 2)
    assert np.array_equal(got, want)


@pytest.mark.gpu
def test_int8_graph_overflow_is_reported():
    """An i32 overflow in a fused member raises FoldOverflow from run()
    (the reference throws at the member), and the flag is cleared after."""
    from paper_1802_04799_b200.executor import DeviceGraph
    nodes = [GraphNode("x", "input", out_type=TensorType([1, 32, 8, 8], "i8")),
             GraphNode("w", "input", out_type=TensorType([32, 32, 3, 3], "i8")),
             GraphNode("c", "conv2d", ["x", "w"], {"padding": [1, 1]}),
             GraphNode("s", "scale", ["c"], {"scale": float(2 ** 20)}),
             GraphNode("q", "requantize", ["s"], {"multiplier": 1, "shift": 24})]
    g = ComputeGraph(nodes, ["q"])
    g.validate()
    dg = DeviceGraph(g, compute="i8")
    dg.bind_params({"w": np.full((32, 32, 3, 3), 8, np.int8)})
    with pytest.raises(TecError) as ei:
        dg.run({"x": np.full((1, 32, 8, 8), 100, np.int8)})
    assert ei.value.code == "FoldOverflow"
    small = dg.run({"x": np.zeros((1, 32, 8, 8), np.int8)})["q"]
    assert not small.any()


def test_graph_tuning_keys_carry_the_epilogue_program():
    """bench_workloads tunes each (conv shape, epilogue program) of a graph:
    the int8 residual blocks are measured with their bias + i8-shortcut add +
    relu + requantize program, the plain ones with bias (+ relu) + requantize,
    bf16 blocks with or without the residual add."""
    import bench_workloads as bw
    from paper_1802_04799_b200 import _abi
    progs = {}
    for compute, g in (("i8", resnet18_graph(2, image=64, width=16, head=False, dtype="i8")),
                       ("bf16", resnet18_graph(2, image=64, width=16))):
        f = fuse_pass(g)
        progs[compute] = {bw._graph_conv_epilogue(n, compute)[0]: bw._graph_conv_epilogue(n, compute)[1]
                          for n in f.nodes if n.op == "fused" and n.members[0].op == "conv2d"}
    res_q = (_abi.EPI_BIAS, _abi.EPI_ADD, _abi.EPI_RELU, _abi.EPI_REQUANTIZE)
    assert res_q in progs["i8"] and progs["i8"][res_q]["residual_i8"] == 1
    assert (_abi.EPI_BIAS, _abi.EPI_RELU, _abi.EPI_REQUANTIZE) in progs["i8"]
    assert all(p["rq_shift"] == 16 for p in progs["i8"].values())
    assert (_abi.EPI_BIAS, _abi.EPI_ADD, _abi.EPI_RELU) in progs["bf16"]
    assert all(p is None for p in progs["bf16"].values())
