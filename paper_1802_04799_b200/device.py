"""Device-resident fused-conv layers: packed buffers in HBM + one C-ABI
launch per call (tec_conv2d_fused / tec_depthwise_fused on the caller's
stream). torch is used only to allocate device memory and to name streams;
all compute runs in libtec_sm100.so.
"""
from __future__ import annotations

import ctypes as C
from typing import Optional

import torch

from . import _abi
from .workloads import ConvWorkload

_COMPUTE = {"bf16": _abi.COMPUTE_BF16, "f32tc": _abi.COMPUTE_F32TC,
            "i8": _abi.COMPUTE_I8, "f32": _abi.COMPUTE_F32}
_TORCH_DT = {_abi.DT_F32: torch.float32, _abi.DT_BF16: torch.bfloat16,
             _abi.DT_I32: torch.int32, _abi.DT_I8: torch.int8}


def _stream_ptr(stream: Optional[torch.cuda.Stream]) -> int:
    s = stream or torch.cuda.current_stream()
    return s.cuda_stream


def make_desc(wl: ConvWorkload, compute: str = "bf16") -> _abi.ConvDesc:
    return _abi.ConvDesc(n=wl.n, c=wl.c, h=wl.h, w=wl.w, k=wl.k, r=wl.r, s=wl.s,
                         stride_h=wl.stride, stride_w=wl.stride, pad_h=wl.pad, pad_w=wl.pad,
                         depthwise=1 if wl.depthwise else 0, compute=_COMPUTE[compute])


class DeviceConv:
    """One fused [conv, bias_add, (add), relu] node, resident on a device."""

    def __init__(self, wl: ConvWorkload, compute: str = "bf16",
                 out_dtype: Optional[int] = None, residual: bool = False,
                 device: int = 0, seed: int = 0, knobs: Optional[dict] = None):
        self.wl = wl
        self.lib = _abi.load()
        self.compute = _COMPUTE[compute]
        self.dev = torch.device("cuda", device)
        self.desc = _abi.ConvDesc(n=wl.n, c=wl.c, h=wl.h, w=wl.w, k=wl.k,
                                  r=wl.r, s=wl.s, stride_h=wl.stride,
                                  stride_w=wl.stride, pad_h=wl.pad, pad_w=wl.pad,
                                  depthwise=1 if wl.depthwise else 0,
                                  compute=self.compute)
        lay = _abi.ConvLayout()
        _abi.check(self.lib.tec_conv_layout_of(C.byref(self.desc), C.byref(lay)))
        self.layout = lay
        integer = self.compute == _abi.COMPUTE_I8
        if out_dtype is None:
            out_dtype = (_abi.DT_I32 if integer else
                         _abi.DT_F32 if self.compute in (_abi.COMPUTE_F32, _abi.COMPUTE_F32TC)
                         else _abi.DT_BF16)
        self.out_dtype = out_dtype
        g = torch.Generator(device=self.dev)
        g.manual_seed(seed)
        st = _stream_ptr(None)
        # Synthetic inputs in the reference distributions (R/src/tensor.cpp:74-88).
        if integer:
            x_src = torch.randint(-8, 8, (wl.n, wl.c, wl.h, wl.w), dtype=torch.int8,
                                  device=self.dev, generator=g)
            w_shape = (wl.c, 1, wl.r, wl.s) if wl.depthwise else (wl.k, wl.c, wl.r, wl.s)
            w_src = torch.randint(-8, 8, w_shape, dtype=torch.int8, device=self.dev,
                                  generator=g)
            self.bias = torch.randint(-100, 101, (wl.k,), dtype=torch.int32,
                                      device=self.dev, generator=g)
        else:
            x_src = torch.rand((wl.n, wl.c, wl.h, wl.w), device=self.dev,
                               generator=g) * 2 - 1
            w_shape = (wl.c, 1, wl.r, wl.s) if wl.depthwise else (wl.k, wl.c, wl.r, wl.s)
            w_src = torch.rand(w_shape, device=self.dev, generator=g) * 2 - 1
            self.bias = torch.rand((wl.k,), device=self.dev, generator=g) * 2 - 1
        self.x = torch.empty(lay.act_bytes, dtype=torch.uint8, device=self.dev)
        self.w = torch.empty(lay.wt_bytes, dtype=torch.uint8, device=self.dev)
        _abi.check(self.lib.tec_activation_pack(C.byref(self.desc), x_src.data_ptr(),
                                                self.x.data_ptr(), st))
        _abi.check(self.lib.tec_weight_pretransform(C.byref(self.desc), w_src.data_ptr(),
                                                    self.w.data_ptr(), st))
        m = wl.n * wl.oh * wl.ow
        self.y = torch.empty((m, wl.k), dtype=_TORCH_DT[out_dtype], device=self.dev)
        self.residual = None
        self.epi = _abi.Epilogue()
        ops = [_abi.EPI_BIAS]
        if residual:
            self.residual = torch.rand((m, wl.k), device=self.dev, generator=g).to(
                self.y.dtype)
            ops.append(_abi.EPI_ADD)
            self.epi.residual = self.residual.data_ptr()
        ops.append(_abi.EPI_RELU)
        for i, o in enumerate(ops):
            self.epi.ops[i] = o
        self.epi.n_ops = len(ops)
        self.epi.bias = self.bias.data_ptr()
        self.knobs = _abi.Knobs(**(knobs or {}))
        # caller-owned split-K scratch (tec_workspace_bytes), zeroed once
        nbytes = C.c_size_t(0)
        if not wl.depthwise:
            _abi.check(self.lib.tec_workspace_bytes(C.byref(self.desc), C.byref(self.epi),
                                                    C.byref(self.knobs), C.byref(nbytes)))
        self.ws = torch.zeros(max(1, nbytes.value), dtype=torch.uint8, device=self.dev)
        self.ws_bytes = nbytes.value
        # the packed operands are ready before any launch, on any stream (the
        # conv kernels read weights before their PDL wait)
        torch.cuda.synchronize(self.dev)
        del x_src, w_src

    def launch(self, stream: Optional[torch.cuda.Stream] = None) -> None:
        if self.wl.depthwise:
            _abi.check(self.lib.tec_depthwise_fused(
                C.byref(self.desc), C.byref(self.epi), C.byref(self.knobs), self.x.data_ptr(),
                self.w.data_ptr(), self.y.data_ptr(), self.out_dtype, None, _stream_ptr(stream)))
            return
        _abi.check(self.lib.tec_conv2d_fused_ws(
            C.byref(self.desc), C.byref(self.epi), C.byref(self.knobs), self.x.data_ptr(),
            self.w.data_ptr(), self.y.data_ptr(), self.out_dtype, None, self.ws.data_ptr(),
            self.ws_bytes, _stream_ptr(stream)))

    @property
    def act_elem_bytes(self) -> int:
        return {_abi.DT_BF16: 2, _abi.DT_I8: 1}.get(self.layout.act_dtype, 4)

    @property
    def out_elem_bytes(self) -> int:
        return {_abi.DT_BF16: 2, _abi.DT_I8: 1}.get(self.out_dtype, 4)

    def algorithmic_bytes(self) -> int:
        return self.wl.bytes(self.act_elem_bytes, self.out_elem_bytes)
