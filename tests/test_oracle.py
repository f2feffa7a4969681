"""CPU tests: pin the C restatement (oracle/tec_oracle.c) against the
REFERENCE's own outputs (tests/golden, produced by the reference binary),
plus the hand-computed known-answer tests of SURVEY 8(c)."""
import numpy as np
import pytest

import golden_cases
from oracle.oracle_api import OracleError, fused_conv, same_values


@pytest.mark.parametrize("name", golden_cases.names())
def test_port_bit_identical_to_reference(name):
    c = golden_cases.load(name)
    if c.status != "ok":
        # The reference threw; the restatement must fail the same way.
        assert "FoldOverflow" in c.status
        with pytest.raises(OracleError) as ei:
            fused_conv(c.op, c.x, c.w, c.strides, c.padding, c.epilogue)
        assert ei.value.status == 3  # 1 + ErrorCode::kFoldOverflow
        return
    y = fused_conv(c.op, c.x, c.w, c.strides, c.padding, c.epilogue)
    assert y.dtype == c.expected.dtype and y.shape == c.expected.shape
    # Bit-identical: same accumulation order and rounding as the reference.
    assert same_values(y, c.expected, 0.0)
    assert np.array_equal(y.view(np.uint32) if y.dtype == np.float32 else y,
                          c.expected.view(np.uint32)
                          if y.dtype == np.float32 else c.expected)


def test_kat_ones_pad1_values():
    c = golden_cases.load("kat_ones_pad1")
    # 3x3 of 2.0, 3x3 ones kernel, pad 1: corner 4, edge 6, centre 9 (x2).
    want = np.array([[8, 12, 8], [12, 18, 12], [8, 12, 8]], np.float32)
    assert np.array_equal(c.expected[0, 0], want)


def test_kat_depthwise_values():
    c = golden_cases.load("kat_depthwise")
    assert np.array_equal(c.expected[0, 0],
                          np.array([[4, 6, 4], [6, 9, 6], [4, 6, 4]], np.float32))
    assert np.array_equal(c.expected[0, 1],
                          -1.5 * np.array([[4, 6, 4], [6, 9, 6], [4, 6, 4]],
                                          np.float32))


def test_kat_saturation_value():
    c = golden_cases.load("i8_saturation")
    # centre output: 512 channels x 9 taps x (-128)^2
    assert c.expected[0, 0, 1, 1] == 512 * 9 * 16384 == 75497472


def test_fuse_pass_groups_conv_epilogue():
    # fuse_pass puts [conv, scale, bias_add, add, relu] in ONE fused node
    # (R/src/graph_passes.cpp:240-244); the backend relies on that grouping.
    c = golden_cases.load("conv_residual")
    nodes = [n for n in c.fused["graph"]["nodes"] if n["op"] != "input"]
    assert len(nodes) == 1 and nodes[0]["op"] == "fused"
    assert [m["op"] for m in nodes[0]["members"]] == [
        "conv2d", "scale", "bias_add", "add", "relu"]
    assert nodes[0]["inputs"] == ["x", "w", "b", "r"]


def test_port_error_codes():
    x = np.zeros((1, 3, 4, 4), np.float32)
    w = np.zeros((2, 3, 5, 5), np.float32)
    with pytest.raises(OracleError) as ei:
        fused_conv("conv2d", x, w)  # window larger than input
    assert ei.value.status == 2  # ShapeMismatch
