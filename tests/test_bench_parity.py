"""Parity at EXACTLY the configurations bench.py times (configs[1] C1-C12 and
configs[3] D1-D9 at batch 64), through the same device entry points the bench
launches (tec_activation_pack / tec_weight_pretransform / tec_conv2d_fused /
tec_depthwise_fused on device buffers, N = 64 in one launch) and with the
knob sets bench.py reads from profiles/tuned_knobs.json -- every entry of that
file is a test case here, so the bench never times an unchecked schedule.

Checks per layer (comparator = DenseTensor::same_values, R/src/tensor.cpp:56-72):
  * every image of the batch against an exact (float64) convolution of the
    same inputs -- a size-independent bound that covers all 64 images;
  * sampled images (first, middle, last) against the oracle restatement
    (oracle/tec_oracle.c, bit-identical to the reference).
Bars: i8 exact; f32tc 1e-4 (the reference's own rounding at K = 4608 is
accounted for as in test_conv_gpu.f32tc_within_bar); bf16 in / bf16 out
TOL_BF16_OUT = 2e-3 accumulation + 2^-9 output rounding; depthwise exact.
"""
import ctypes as C
import json
import os

import numpy as np
import pytest

from oracle.oracle_api import bf16_round, fused_conv as oracle_conv, same_values
from paper_1802_04799_b200 import _abi
from paper_1802_04799_b200.ops import conv_desc
from paper_1802_04799_b200.workloads import MOBILENET_DW, RESNET18_CONVS

from test_conv_gpu import f32tc_within_bar

pytestmark = pytest.mark.gpu

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KNOBS = json.load(open(os.path.join(REPO, "profiles", "tuned_knobs.json")))
BATCH = 64
SAMPLES = (0, 31, 63)
TOL_F32TC = 1e-4
TOL_BF16_OUT = 2e-3 + 2.0 ** -9
_CM = {"f32tc": _abi.COMPUTE_F32TC, "bf16": _abi.COMPUTE_BF16, "i8": _abi.COMPUTE_I8,
       "f32": _abi.COMPUTE_F32}


def _inputs(shape_x, shape_w, k, integer, seed):
    rng = np.random.default_rng(seed)
    if integer:
        return (rng.integers(-8, 8, shape_x, dtype=np.int8), rng.integers(-8, 8, shape_w, dtype=np.int8),
                rng.integers(-100, 101, (k,), dtype=np.int32))
    return (rng.uniform(-1, 1, shape_x).astype(np.float32),
            rng.uniform(-1, 1, shape_w).astype(np.float32),
            rng.uniform(-1, 1, (k,)).astype(np.float32))


def device_fused(op, x, w, b, attrs, compute, knobs, relu=True):
    """One launch on device buffers, exactly as bench.py's DeviceConv runs
    it (same descriptor, packing, knobs, output dtype); returns NCHW numpy."""
    import torch
    lib = _abi.load()
    shape = []
    d = conv_desc(op, x.shape, w.shape, attrs, _CM[compute], shape)
    lay = _abi.ConvLayout()
    _abi.check(lib.tec_conv_layout_of(C.byref(d), C.byref(lay)))
    dev = torch.device("cuda", 0)
    xd, wd = torch.from_numpy(x).to(dev), torch.from_numpy(w).to(dev)
    bd = torch.from_numpy(b).to(dev)
    xp = torch.empty(lay.act_bytes, dtype=torch.uint8, device=dev)
    wp = torch.empty(lay.wt_bytes, dtype=torch.uint8, device=dev)
    st = torch.cuda.current_stream().cuda_stream
    _abi.check(lib.tec_weight_pretransform(C.byref(d), wd.data_ptr(), wp.data_ptr(), st))
    _abi.check(lib.tec_activation_pack(C.byref(d), xd.data_ptr(), xp.data_ptr(), st))
    torch.cuda.synchronize()
    out_dt = {"i8": (_abi.DT_I32, torch.int32), "bf16": (_abi.DT_BF16, torch.bfloat16)}.get(
        compute, (_abi.DT_F32, torch.float32))
    n, k, oh, ow = shape
    y = torch.empty((n * oh * ow, k), dtype=out_dt[1], device=dev)
    err = torch.zeros(1, dtype=torch.int32, device=dev)
    epi = _abi.Epilogue()
    epi.ops[0] = _abi.EPI_BIAS
    if relu:
        epi.ops[1] = _abi.EPI_RELU
    epi.n_ops = 2 if relu else 1
    epi.bias = bd.data_ptr()
    kn = _abi.Knobs(**(knobs or {}))
    fn = lib.tec_depthwise_fused if op == "depthwise_conv2d" else lib.tec_conv2d_fused
    _abi.check(fn(C.byref(d), C.byref(epi), C.byref(kn), xp.data_ptr(), wp.data_ptr(),
                  y.data_ptr(), out_dt[0], err.data_ptr(), st))
    torch.cuda.synchronize()
    assert int(err.item()) == 0
    out = y.view(n, oh, ow, k).permute(0, 3, 1, 2).contiguous()
    return (out.float() if compute == "bf16" else out).cpu().numpy()


def exact_conv(x, w, b, stride, pad, depthwise=False, relu=True):
    """float64 conv + bias (+ relu) on the GPU -- the checker's exact sum."""
    import torch
    dev = torch.device("cuda", 0)
    xd = torch.from_numpy(x.astype(np.float64)).to(dev)
    wd = torch.from_numpy(w.astype(np.float64)).to(dev)
    y = torch.nn.functional.conv2d(xd, wd, stride=stride, padding=pad,
                                   groups=x.shape[1] if depthwise else 1)
    y = y + torch.from_numpy(b.astype(np.float64)).to(dev).view(1, -1, 1, 1)
    if relu:
        y = torch.relu(y)
    return y.cpu().numpy()


def _layer_case(layer, compute):
    hw, c, k, r, s = RESNET18_CONVS[layer]
    x, w, b = _inputs((BATCH, c, hw, hw), (k, c, r, r), k, compute == "i8",
                      seed=100 + sum(map(ord, layer)))
    return x, w, b, {"strides": (s, s), "padding": (r // 2, r // 2)}


@pytest.mark.parametrize("layer", list(RESNET18_CONVS))
@pytest.mark.parametrize("compute", ["f32tc", "bf16", "i8"])
def test_bench_config_batch64(layer, compute):
    knobs = KNOBS[compute][layer]
    x, w, b, attrs = _layer_case(layer, compute)
    y = device_fused("conv2d", x, w, b, attrs, compute, knobs)
    st, pd = attrs["strides"], attrs["padding"]
    epi = [("bias_add", b), ("relu",)]
    if compute == "bf16":
        xr, wr = bf16_round(x), bf16_round(w)
    else:
        xr, wr = x, w
    exact = exact_conv(xr, wr, b, st, pd)
    if compute == "i8":
        # |sum| < 2^53: the float64 conv is exact -- all 64 images bit-exact
        assert np.array_equal(y, exact.astype(np.int64).astype(np.int32))
    elif compute == "f32tc":
        assert same_values(y, exact.astype(np.float32), TOL_F32TC)
    else:
        assert same_values(y, exact.astype(np.float32), TOL_BF16_OUT)
    for i in SAMPLES:
        want = oracle_conv("conv2d", xr[i:i + 1], wr, st, pd, epi)
        got = y[i:i + 1]
        if compute == "i8":
            assert np.array_equal(got, want)
        elif compute == "f32tc":
            ok, n = f32tc_within_bar(got, want, exact[i:i + 1])
            assert ok, f"image {i}: {n} outputs beyond 1e-4 not explained by the reference's rounding"
        else:
            assert same_values(got, want, TOL_BF16_OUT)


@pytest.mark.parametrize("layer", list(MOBILENET_DW))
@pytest.mark.parametrize("compute", ["bf16", "f32"])
def test_depthwise_batch64(layer, compute):
    """configs[3] at batch 64 through the default (TMA) depthwise kernel:
    accumulation in the oracle's order, so the WHOLE batch is bit-identical
    to the oracle restatement."""
    hw, c, s = MOBILENET_DW[layer]
    x, w, b = _inputs((BATCH, c, hw, hw), (c, 1, 3, 3), c, False, seed=200 + sum(map(ord, layer)))
    attrs = {"strides": (s, s), "padding": (1, 1)}
    out_f32 = compute == "f32"
    y = device_fused("depthwise_conv2d", x, w, b, attrs, compute if out_f32 else "bf16", {})
    xr, wr = (x, w) if out_f32 else (bf16_round(x), bf16_round(w))
    want = oracle_conv("depthwise_conv2d", xr, wr, (s, s), (1, 1), [("bias_add", b), ("relu",)])
    if out_f32:
        assert np.array_equal(y.view(np.uint32), want.view(np.uint32))
    else:  # bf16 output: the oracle's f32 result rounded once to bf16
        assert np.array_equal(y, bf16_round(want))


def test_knob_file_covers_every_bench_layer():
    for prec in ("f32tc", "bf16", "i8"):
        assert set(KNOBS[prec]) == set(RESNET18_CONVS), prec
