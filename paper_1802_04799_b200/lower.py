"""Lowering for target "sm100" and the tensor-intrinsic registry.

Reference -> here:
  LowerOptions / lower(sched, name, opts)   R/include/tec/lower.hpp:26-36,
      R/src/lower.cpp:231-1259 -> LowerOptions(target="sm100") and
      lower(desc, config): the schedule decision (a Config, SURVEY 8a knob
      mapping) becomes a concrete kernel plan -- kernel family, CTA tile,
      pipeline depth, split-K, cluster, grid, shared-memory and TMEM budget --
      chosen by the same native planner that launches it (tec_conv_plan).
      Capacity violations (smem > 227 KB, TMEM > 512 columns, no instance for
      the tile) are LoweringError, in place of check_target's SRAM budgets
      (R/src/lower.cpp:1169-1209).
  Intrinsic / declare_intrinsic /           R/include/tec/texpr.hpp:99-112,
  find_intrinsic / register_builtin_        R/src/texpr.cpp:297-349 -> the
  intrinsics                                sm100 tensor-core and SIMT
      instructions the kernels tensorize onto, with their shapes, operand
      scopes and dtypes, so `tensorize` knobs stay checkable; re-declaring a
      name is DuplicateIntrinsic, as in the reference.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import Dict, Optional, Sequence, Tuple

from . import _abi
from ._abi import TecError

E_DUPLICATE_INTRINSIC, E_TENSORIZE_MISMATCH, E_LOWERING = 5, 14, 15

FAMILIES = {1: "im2col", 2: "halo", 3: "f32_exact", 4: "depthwise_tma", 5: "depthwise_direct",
            6: "f32tc", 7: "f32tc_halo"}


@dataclass(frozen=True)
class Intrinsic:
    """A tensor instruction a stage can be tensorized onto."""
    name: str
    behavior: str                       # "matmul_acc" | "fma_acc"
    m: Tuple[int, ...]                  # legal M extents
    n: Tuple[int, int, int]             # (min, max, step) of N
    k: int                              # K elements per instruction
    in_dtype: str
    acc_dtype: str
    operand_scope: Dict[str, str] = field(default_factory=dict)
    scope_checked: bool = True
    instruction: str = ""

    def accepts(self, m: int, n: int, k: int) -> bool:
        lo, hi, step = self.n
        return m in self.m and lo <= n <= hi and (n - lo) % step == 0 and k % self.k == 0


_REGISTRY: Dict[str, Intrinsic] = {}


def declare_intrinsic(intr: Intrinsic) -> None:
    if intr.name in _REGISTRY:
        raise TecError(E_DUPLICATE_INTRINSIC, f"intrinsic '{intr.name}' already declared")
    _REGISTRY[intr.name] = intr


def find_intrinsic(name: str) -> Optional[Intrinsic]:
    return _REGISTRY.get(name)


def register_builtin_intrinsics() -> None:
    """Idempotent (R/src/texpr.cpp:311-349): the sm_100a instructions the
    conv kernels are built from."""
    umma_scope = {"A": "shared", "B": "shared", "D": "tensor_memory"}
    builtins = [
        Intrinsic("sm100.umma.bf16", "matmul_acc", (64, 128), (8, 256, 8), 16, "bf16", "f32",
                  umma_scope, True, "tcgen05.mma.cta_group::1.kind::f16"),
        # f32 as three exact bf16 planes, six kind::f16 products per K16 step
        Intrinsic("sm100.umma.bf16x6", "matmul_acc", (128,), (64, 128, 64), 16, "f32", "f32",
                  umma_scope, True, "tcgen05.mma.cta_group::1.kind::f16 x6 (split-bf16 f32)"),
        Intrinsic("sm100.umma.i8", "matmul_acc", (64, 128), (8, 256, 8), 32, "i8", "i32",
                  umma_scope, True, "tcgen05.mma.cta_group::1.kind::i8"),
        Intrinsic("sm100.simt.f32", "fma_acc", (1,), (1, 1, 1), 1, "f32", "f32",
                  {"A": "global", "B": "shared", "D": "register"}, False, "fmul.rn + fadd.rn"),
    ]
    for b in builtins:
        if b.name not in _REGISTRY:
            declare_intrinsic(b)


_COMPUTE_INTRIN = {_abi.COMPUTE_BF16: "sm100.umma.bf16", _abi.COMPUTE_F32TC: "sm100.umma.bf16x6",
                   _abi.COMPUTE_I8: "sm100.umma.i8", _abi.COMPUTE_F32: "sm100.simt.f32"}


@dataclass
class LowerOptions:
    target: str = "sm100"
    smem_bytes: int = 227 * 1024   # per-CTA dynamic shared memory
    tmem_cols: int = 512           # tensor-memory columns per SM


@dataclass
class KernelPlan:
    family: str
    tile_m: int
    tile_n: int
    stages: int
    split_k: int
    cluster: int
    grid: int
    smem_bytes: int
    tmem_cols: int
    tma_store: bool
    intrinsic: str


def lower(desc: _abi.ConvDesc, config: Optional[Dict[str, int]] = None,
          epilogue: Sequence[int] = (_abi.EPI_BIAS, _abi.EPI_RELU),
          opts: Optional[LowerOptions] = None,
          epi_params: Optional[Dict[str, int]] = None) -> KernelPlan:
    """Config -> the kernel the sm100 backend runs for it (no launch).
    epi_params: the int8 epilogue's scalars (rq_mult, rq_shift, residual_i8,
    residual_scale) when the program requantizes / reads an i8 shortcut."""
    opts = opts or LowerOptions()
    if opts.target != "sm100":
        raise TecError(E_LOWERING, f"target '{opts.target}' is not this backend (use 'sm100')")
    register_builtin_intrinsics()
    epi = _abi.Epilogue()
    for i, op in enumerate(epilogue):
        epi.ops[i] = op
    epi.n_ops = len(epilogue)
    if _abi.EPI_BIAS in epilogue:
        epi.bias = 1
    if _abi.EPI_ADD in epilogue:
        epi.residual = 1
    if _abi.EPI_MUL in epilogue:
        epi.mul_operand = 1
    for k, v in (epi_params or {}).items():
        setattr(epi, k, v)
    kn = _abi.Knobs(**(config or {}))
    out = _abi.KernelPlan()
    _abi.check(_abi.load().tec_conv_plan(C.byref(desc), C.byref(epi), C.byref(kn), C.byref(out)))
    plan = KernelPlan(FAMILIES.get(out.family, str(out.family)), out.tile_m, out.tile_n,
                      out.stages, out.split_k, out.cluster, out.grid, out.smem_bytes,
                      out.tmem_cols, bool(out.tma_store), _COMPUTE_INTRIN[desc.compute])
    if plan.smem_bytes > opts.smem_bytes or plan.tmem_cols > opts.tmem_cols:
        raise TecError(E_LOWERING, f"plan exceeds the on-chip budget: {plan}")
    intr = find_intrinsic(plan.intrinsic)
    if plan.family in ("im2col", "halo", "f32tc", "f32tc_halo") and not intr.accepts(128, plan.tile_n, intr.k):
        raise TecError(E_TENSORIZE_MISMATCH, f"{plan.intrinsic} cannot take N={plan.tile_n}")
    return plan
