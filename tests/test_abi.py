"""CPU tests of the C ABI boundary: the product library loads, exports every
symbol include/tec_sm100.h declares, and its host-only entry points apply
the reference's shape rules and error codes (no GPU needed)."""
import ctypes as C
import os
import re

import pytest

from paper_1802_04799_b200 import _abi
from paper_1802_04799_b200.ops import conv_desc

HEADER = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                      "include", "tec_sm100.h")


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(tec_[a-z0-9_]+)\s*\(", src)))


def test_header_symbols_exported():
    lib = _abi.load()
    names = declared_functions()
    assert len(names) >= 12
    for n in names:
        assert hasattr(lib, n), f"{n} declared in tec_sm100.h but not exported"
    assert set(names) == set(_abi.SIGNATURES), "ctypes table out of sync with header"


def test_api_version():
    assert _abi.load().tec_api_version() == 1


def _desc(**kw):
    base = dict(n=1, c=64, h=56, w=56, k=64, r=3, s=3, stride_h=1, stride_w=1,
                pad_h=1, pad_w=1, depthwise=0, compute=_abi.COMPUTE_BF16)
    base.update(kw)
    return _abi.ConvDesc(**base)


def test_infer_c2():
    out = (C.c_int64 * 4)()
    assert _abi.load().tec_conv_infer(C.byref(_desc()), out) == 0
    assert list(out) == [1, 64, 56, 56]


@pytest.mark.parametrize("h,w,r,s,stride,pad,shape", [
    (224, 224, 7, 7, 2, 3, [1, 64, 112, 112]),   # C1
    (56, 56, 1, 1, 2, 0, [1, 64, 28, 28]),       # C5-like
    (7, 7, 3, 3, 1, 1, [1, 64, 7, 7]),           # C12-like
])
def test_infer_resnet_shapes(h, w, r, s, stride, pad, shape):
    out = (C.c_int64 * 4)()
    d = _desc(h=h, w=w, r=r, s=s, stride_h=stride, stride_w=stride,
              pad_h=pad, pad_w=pad)
    assert _abi.load().tec_conv_infer(C.byref(d), out) == 0
    assert list(out) == shape


def test_window_larger_than_input_is_shape_mismatch():
    out = (C.c_int64 * 4)()
    st = _abi.load().tec_conv_infer(C.byref(_desc(h=2, w=2, pad_h=0, pad_w=0)), out)
    assert st == 2  # 1 + ErrorCode::kShapeMismatch
    assert b"window larger than input" in _abi.load().tec_last_error()


def test_depthwise_weight_shape_checked():
    with pytest.raises(_abi.TecError) as ei:
        conv_desc("depthwise_conv2d", (1, 8, 4, 4), (4, 1, 3, 3), {}, 1)
    assert ei.value.code == "ShapeMismatch"
    with pytest.raises(_abi.TecError) as ei:
        conv_desc("conv2d", (1, 8, 4, 4), (4, 3, 3, 3), {}, 1)
    assert ei.value.code == "ShapeMismatch"
    with pytest.raises(_abi.TecError) as ei:
        conv_desc("matmul", (1, 8, 4, 4), (4, 8, 3, 3), {}, 1)
    assert ei.value.code == "UnknownOperator"


def test_layout_planning():
    lay = _abi.ConvLayout()
    lib = _abi.load()
    assert lib.tec_conv_layout_of(C.byref(_desc()), C.byref(lay)) == 0
    assert lay.cp == 64 and lay.act_dtype == _abi.DT_BF16
    assert lay.act_bytes == 56 * 56 * 64 * 2
    # stem: 3 channels padded to one 32-byte block
    assert lib.tec_conv_layout_of(C.byref(_desc(c=3)), C.byref(lay)) == 0
    assert lay.cp == 16
    # f32 on tensor cores stores three exact bf16 planes [h | m | l]
    d = _desc(compute=_abi.COMPUTE_F32TC)
    assert lib.tec_conv_layout_of(C.byref(d), C.byref(lay)) == 0
    assert lay.cp == 192 and lay.act_dtype == _abi.DT_BF16
    assert lay.act_bytes == 56 * 56 * 192 * 2
    d = _desc(compute=_abi.COMPUTE_I8)
    assert lib.tec_conv_layout_of(C.byref(d), C.byref(lay)) == 0
    assert lay.cp == 64 and lay.acc_dtype == _abi.DT_I32


def test_struct_layouts_match_header(tmp_path):
    """The ctypes mirrors have the C structs' sizes and field offsets
    (compiled against include/tec_sm100.h with the host compiler)."""
    import shutil
    import subprocess
    if not shutil.which("gcc"):
        pytest.skip("no host C compiler")
    checks = {
        "tec_conv_desc": (_abi.ConvDesc, []),
        "tec_epilogue": (_abi.Epilogue, ["bias", "mul_operand", "rq_mult", "rq_shift",
                                         "residual_i8", "residual_scale"]),
        "tec_knobs": (_abi.Knobs, ["grid"]),
        "tec_pool_desc": (_abi.PoolDesc, ["out_dtype"]),
        "tec_kernel_plan": (_abi.KernelPlan, ["tma_store", "workspace_bytes"]),
        "tec_elem_prog": (_abi.ElemProg, ["kind", "shift", "cast_to", "mult", "scale", "src_dtype",
                                          "count"]),
        "tec_step": (_abi.Step, ["conv", "epi", "knobs", "pool", "src", "w", "dst", "w_", "elem"]),
    }
    lines = ['#include <stdio.h>', '#include <stddef.h>', '#include "tec_sm100.h"',
             'int main(void) {']
    for cname, (_, fields) in checks.items():
        lines.append(f'  printf("%zu\\n", sizeof({cname}));')
        for f in fields:
            lines.append(f'  printf("%zu\\n", offsetof({cname}, {f}));')
    lines.append("  return 0; }")
    src = tmp_path / "layout.c"
    src.write_text("\n".join(lines))
    exe = tmp_path / "layout"
    subprocess.run(["gcc", "-I", os.path.dirname(HEADER), str(src), "-o", str(exe)], check=True)
    got = [int(v) for v in subprocess.run([str(exe)], capture_output=True, text=True,
                                          check=True).stdout.split()]
    want = []
    for _, (py, fields) in checks.items():
        want.append(C.sizeof(py))
        want += [getattr(py, f).offset for f in fields]
    assert got == want


def test_plan_create_rejects_bad_arguments():
    lib = _abi.load()
    h = C.c_void_p()
    assert lib.tec_plan_create(None, -1, C.byref(h)) != 0
    assert lib.tec_plan_size(None) == 0
    lib.tec_plan_destroy(None)


def test_window_larger_than_padded_input_is_rejected():
    """-stride < h + 2p - r < 0: C++ truncation would give OH = 1 (the
    reference's infer_conv accepts it and then reads out of bounds); the ABI
    rejects it and Python sizes outputs from the ABI's shape."""
    from paper_1802_04799_b200.ops import conv_desc
    with pytest.raises(_abi.TecError) as ei:
        conv_desc("conv2d", (1, 4, 2, 2), (4, 4, 3, 3), {"strides": (2, 2)}, 1)
    assert ei.value.code == "ShapeMismatch"
    shape = []
    conv_desc("conv2d", (1, 4, 3, 3), (4, 4, 3, 3), {"strides": (2, 2)}, 1, shape)
    assert shape == [1, 4, 1, 1]
