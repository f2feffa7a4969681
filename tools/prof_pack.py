"""Time tec_activation_pack (NCHW input -> the conv's packed layout) for a
ResNet-18 layer at a batch: python tools/prof_pack.py [LAYER] [BATCH] [bf16|i8|f32tc]."""
import ctypes as C
import os
import sys

import torch

sys.path.insert(0, os.getcwd())
from paper_1802_04799_b200 import _abi
from paper_1802_04799_b200.device import make_desc
from paper_1802_04799_b200.workloads import resnet_layer

name = sys.argv[1] if len(sys.argv) > 1 else "C1"
batch = int(sys.argv[2]) if len(sys.argv) > 2 else 256
lib = _abi.load()
compute = sys.argv[3] if len(sys.argv) > 3 else "bf16"
d = make_desc(resnet_layer(name, batch), compute)
lay = _abi.ConvLayout()
_abi.check(lib.tec_conv_layout_of(C.byref(d), C.byref(lay)))
x = (torch.randint(-8, 8, (d.n * d.c * d.h * d.w,), dtype=torch.int8, device="cuda")
     if compute == "i8" else torch.rand(d.n * d.c * d.h * d.w, device="cuda"))
y = torch.empty(lay.act_bytes, dtype=torch.uint8, device="cuda")
s = torch.cuda.current_stream().cuda_stream
for _ in range(3):
    _abi.check(lib.tec_activation_pack(C.byref(d), x.data_ptr(), y.data_ptr(), s))
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
reps = 20
a.record()
for _ in range(reps):
    _abi.check(lib.tec_activation_pack(C.byref(d), x.data_ptr(), y.data_ptr(), s))
b.record()
torch.cuda.synchronize()
us = a.elapsed_time(b) * 1e3 / reps
nbytes = x.numel() * x.element_size() + lay.act_bytes
print(f"{name} b{batch} {compute} pack: {us:.1f} us, {nbytes / 1e6:.0f} MB, {nbytes / us / 1e6:.2f} TB/s")
