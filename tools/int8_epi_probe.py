"""Times one int8 ResNet layer (b256) with the int8-graph epilogues and
prints the kernel plan: python tools/int8_epi_probe.py [LAYER] [BATCH]."""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1802_04799_b200 import _abi  # noqa: E402
from paper_1802_04799_b200.device import make_desc  # noqa: E402
from paper_1802_04799_b200.workloads import resnet_layer  # noqa: E402

layer = sys.argv[1] if len(sys.argv) > 1 else "C2"
batch = int(sys.argv[2]) if len(sys.argv) > 2 else 256
lib = _abi.load()
d = make_desc(resnet_layer(layer, batch), "i8")
FAM = {0: "?", 1: "im2col", 2: "halo", 3: "f32exact", 4: "dw", 5: "dw_tma", 6: "f32tc", 7: "f32tc_halo"}


def epi(kind):
    e = _abi.Epilogue()
    ops = {"bias": [_abi.EPI_BIAS], "bias_relu": [_abi.EPI_BIAS, _abi.EPI_RELU],
           "bias_relu_q": [_abi.EPI_BIAS, _abi.EPI_RELU, _abi.EPI_REQUANTIZE],
           "bias_q": [_abi.EPI_BIAS, _abi.EPI_REQUANTIZE],
           "bias_add_relu_q": [_abi.EPI_BIAS, _abi.EPI_ADD, _abi.EPI_RELU, _abi.EPI_REQUANTIZE],
           "bias_add32_relu_q": [_abi.EPI_BIAS, _abi.EPI_ADD, _abi.EPI_RELU, _abi.EPI_REQUANTIZE]}[kind]
    for i, o in enumerate(ops):
        e.ops[i] = o
    e.n_ops = len(ops)
    e.bias = 256
    e.rq_mult, e.rq_shift = 900, 16
    if _abi.EPI_ADD in ops:
        e.residual = 256
        if kind == "bias_add_relu_q":
            e.residual_i8, e.residual_scale = 1, 37
    return e


for knobs in ({}, {"tile_k": 1}, {"tile_k": 2}):
    for kind in ("bias_relu", "bias_relu_q", "bias_add_relu_q", "bias_add32_relu_q"):
        e = epi(kind)
        kn = _abi.Knobs(**knobs)
        plan = _abi.KernelPlan()
        st = lib.tec_conv_plan(C.byref(d), C.byref(e), C.byref(kn), C.byref(plan))
        if st:
            print(layer, knobs, kind, "plan error", lib.tec_last_error().decode())
            continue
        us = C.c_double()
        _abi.check(lib.tec_measure(C.byref(d), C.byref(e), C.byref(kn), 0, 3, 20, 1, C.byref(us)))
        print(f"{layer} b{batch} {str(knobs):16s} {kind:18s} {us.value:8.1f} us  "
              f"{FAM.get(plan.family, plan.family)} bn={plan.tile_n} m={plan.tile_m} "
              f"tma_store={plan.tma_store} grid={plan.grid}")
