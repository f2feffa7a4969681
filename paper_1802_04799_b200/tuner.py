"""Schedule-knob tuner for the sm100 conv kernels: the reference's autotune
API (R/include/tec/autotune.hpp) with an on-device measurement runner.

Reference -> here:
  KnobDef / KnobSpace / Config      autotune.hpp:43-77, tune.cpp:57-97
      -> KnobDef / KnobSpace over the B200 template knobs. config_at keeps
         the mixed-radix order (knob 0 slowest), but the space is
         CONDITIONAL: only the configs the native lowering accepts AND that
         lower to distinct kernels (tec_conv_plan) are enumerated, so no
         illegal or duplicate cross product is ever measured; instantiate /
         lower_config is lower.lower (LoweringError -> illegal).
  extract_features                  features.cpp:174-193 -> extract_features:
      the lowered KERNEL PLAN's structure in the reference's terms -- per
      buffer (activation, weight, output) and memory level (HBM, L2->smem
      per tile, smem->tensor core per k-step) the accesses and touched
      bytes, the loop extents (tiles, waves, k-iterations) and the
      annotations (pipeline depth, split, cluster, TMEM buffers), log-scaled.
  CostModel (pairwise-rank GBT)     gbt.cpp:26-185 -> CostModel: the same
      exact-greedy second-order trees on the pairwise logistic rank loss,
      same defaults (depth 6, 50 rounds, lr 0.3, lambda 1), same JSON;
      pinned bit-for-bit against the reference binary (tests/test_tuner.py).
  explore (simulated annealing)     tune.cpp:183-291 -> explore: chains of
      one-knob neighbour moves under the model's score, the best-scored
      unmeasured configs plus a random floor (5 %).
  measure / measure_program         tune.cpp:295-351 (simulated cycles,
      sequential) -> tec_measure: CUDA-event timing on the GPU of
      `repeats` back-to-back (L2 flush, launch) pairs minus the flushes
      alone, median of three such batches, configs sharded
      round-robin over the visible devices (one host thread per device).
  TrialRecord / append_trials /     tune.cpp:101-144 (JSONL DB)
  load_trials                       -> identical JSONL fields.
  tune                              tune.cpp:355-436 -> the same loop: seed
      from the DB, train + explore when >= 2 ok trials (method "ml"), else
      random unmeasured, measure, append, retrain.
Lowering failures become status "lowering_failed" trials, as in the
reference (tune.cpp:344-347).
"""
from __future__ import annotations

import ctypes as C
import json
import math
import os
import random
import threading
import time
from dataclasses import dataclass, field
from typing import Callable, Dict, List, Optional, Sequence, Tuple

from . import _abi

Config = Dict[str, int]


@dataclass
class KnobDef:
    name: str
    values: List[int]


def config_key(c: Config) -> str:
    """tune.cpp:32-41: canonical 'k=v,...' in knob-name order."""
    return ",".join(f"{k}={int(c[k])}" for k in sorted(c))


@dataclass
class KnobSpace:
    """A conditional knob space. `knobs` span the grid (and define the
    annealer's one-knob neighbour moves); `instantiate(cfg)` lowers a config
    -- it returns a hashable kernel identity or raises TecError for an
    illegal one (the reference's throwing instantiate, tune.cpp:91-97).
    Enumeration (size / config_at / index_of / random_config) runs over the
    legal configs only, one per distinct kernel, in mixed-radix order."""
    workload: str
    knobs: List[KnobDef]
    desc: Optional[_abi.ConvDesc] = None
    epilogue: Sequence[int] = (_abi.EPI_BIAS, _abi.EPI_RELU)
    # int8 epilogue scalars (rq_mult, rq_shift, residual_i8, residual_scale)
    epi_params: Optional[Dict[str, int]] = None
    target: str = "sm100"
    instantiate: Optional[Callable[[Config], object]] = None
    _legal: Optional[List[Config]] = field(default=None, repr=False)
    _index: Optional[Dict[str, int]] = field(default=None, repr=False)
    _plan_cache: Dict[str, object] = field(default_factory=dict, repr=False)

    def grid_size(self) -> int:
        n = 1
        for k in self.knobs:
            n *= len(k.values)
        return n

    def grid_at(self, flat: int) -> Config:
        """Mixed-radix decode of the full grid, knob 0 slowest (tune.cpp:63-72)."""
        cfg = {}
        for k in reversed(self.knobs):
            cfg[k.name] = k.values[flat % len(k.values)]
            flat //= len(k.values)
        return {k.name: cfg[k.name] for k in self.knobs}

    def lower_config(self, c: Config):
        """tune.cpp:91-97: the lowered kernel of `c`; TecError if illegal
        (cached, failures included)."""
        key = config_key(c)
        if key not in self._plan_cache:
            try:
                self._plan_cache[key] = self.instantiate(c) if self.instantiate else key
            except _abi.TecError as e:
                self._plan_cache[key] = e
        v = self._plan_cache[key]
        if isinstance(v, _abi.TecError):
            raise v
        return v

    def legal(self, c: Config) -> bool:
        try:
            self.lower_config(c)
            return True
        except _abi.TecError:
            return False

    def _enumerate(self) -> None:
        if self._legal is not None:
            return
        seen, legal = set(), []
        for i in range(self.grid_size()):
            c = self.grid_at(i)
            try:
                kern = self.lower_config(c)
            except _abi.TecError:
                continue
            ident = repr(kern)
            if ident in seen:  # another config already names this kernel
                continue
            seen.add(ident)
            legal.append(c)
        self._legal = legal
        self._index = {config_key(c): i for i, c in enumerate(legal)}

    def size(self) -> int:
        self._enumerate()
        return len(self._legal)

    def config_at(self, flat: int) -> Config:
        self._enumerate()
        if not 0 <= flat < len(self._legal):
            raise _abi.TecError(21, "flat config index out of range")
        return dict(self._legal[flat])

    def index_of(self, c: Config) -> int:
        self._enumerate()
        return self._index.get(config_key(c), -1)

    def random_config(self, rng: random.Random) -> Config:
        self._enumerate()
        return dict(rng.choice(self._legal)) if self._legal else {}


@dataclass
class TrialRecord:
    workload: str
    config: Config
    cost: float = 0.0  # microseconds on the device (reference: sim cycles)
    timestamp: int = 0
    status: str = "ok"  # "ok" | "lowering_failed" | "measure_failed"
    method: str = "ml"
    device: int = 0

    def ok(self) -> bool:
        return self.status == "ok"

    def to_json(self) -> dict:
        return {"workload": self.workload, "config": self.config, "cost": self.cost,
                "timestamp": self.timestamp, "status": self.status, "method": self.method}

    @staticmethod
    def from_json(j: dict) -> "TrialRecord":
        return TrialRecord(j["workload"], {k: int(v) for k, v in j["config"].items()},
                           float(j["cost"]), int(j["timestamp"]), j["status"],
                           j.get("method", "ml"))


def append_trials(path: str, trials: Sequence[TrialRecord]) -> None:
    """tune.cpp:118-125; one JSON object per line, single writer."""
    if not trials:
        return
    with open(path, "a") as f:
        for t in trials:
            f.write(json.dumps(t.to_json()) + "\n")


def load_trials(path: str) -> List[TrialRecord]:
    """tune.cpp:127-144; an absent DB is a fresh start."""
    if not os.path.exists(path):
        return []
    out = []
    with open(path) as f:
        for lineno, line in enumerate(f, 1):
            if not line.strip():
                continue
            try:
                out.append(TrialRecord.from_json(json.loads(line)))
            except (ValueError, KeyError) as e:
                raise _abi.TecError(20, f"trial DB {path} line {lineno} is not valid JSON") from e
    return out


def _plan_instantiate(desc: _abi.ConvDesc, epilogue: Sequence[int],
                      epi_params: Optional[Dict[str, int]] = None):
    """Config -> the kernel the native lowering picks (lower.lower, i.e.
    tec_conv_plan); a LoweringError marks the config illegal."""
    from .lower import lower

    def inst(cfg: Config):
        p = lower(desc, cfg, epilogue, epi_params=epi_params)
        return (p.family, p.tile_m, p.tile_n, p.stages, p.split_k, p.cluster, p.grid,
                p.smem_bytes, p.tmem_cols, p.tma_store)
    return inst


def conv_space(name: str, desc: _abi.ConvDesc,
               epilogue: Sequence[int] = (_abi.EPI_BIAS, _abi.EPI_RELU),
               epi_params: Optional[Dict[str, int]] = None) -> KnobSpace:
    """The B200 conv template's knob grid (SURVEY 8a knob mapping), made
    conditional by the native lowering:
      bf16 / i8: tile_k = A-operand strategy (1 im2col TMA, 2 shifted-window
        halo), tile_n = CTA N tile (split of the OC axis), tile_m = M rows per
        tile (halo: MMA sub-tiles x 128), stages (halo: 1 streamed / 2
        resident weights), split_k (im2col: K split over CTAs, partials
        summed in order), cluster_n (halo, streamed weights: CTA pairs share
        weight tiles by TMA multicast; im2col: CTA pairs -- cta_group::2,
        M = 256, each CTA loading half of the weight rows);
      f32tc: tile_k, tile_n, stages (resident weights), split_k (-1: stream-K,
        equal (tile, k) shares) and cluster_n (2: CTA pairs on the im2col path
        at tile_n 128) of the split-bf16 f32 kernel."""
    if desc.compute == _abi.COMPUTE_F32TC:
        knobs = [KnobDef("tile_k", [1, 2]), KnobDef("tile_n", [64, 128]),
                 KnobDef("stages", [1, 2]), KnobDef("split_k", [1, 2, 3, 4, 6, 8, -1]),
                 KnobDef("cluster_n", [1, 2])]
    else:
        knobs = [KnobDef("tile_k", [1, 2]), KnobDef("tile_n", [64, 128, 256]),
                 KnobDef("tile_m", [128, 256, 512]), KnobDef("stages", [1, 2]),
                 KnobDef("split_k", [1, 2, 3, 4]), KnobDef("cluster_n", [1, 2])]
    return KnobSpace(name, knobs, desc, tuple(epilogue), epi_params=epi_params,
                     instantiate=_plan_instantiate(desc, tuple(epilogue), epi_params))


def dw_space(name: str, desc: _abi.ConvDesc,
             epilogue: Sequence[int] = (_abi.EPI_BIAS, _abi.EPI_RELU)) -> KnobSpace:
    """The depthwise template's knobs: unroll selects the kernel -- 1 the
    generic one, 2 / 4 the 3x3 column-streaming kernel with that many outputs
    per thread, 8 the TMA-tiled shared-memory kernel."""
    if not desc.depthwise:
        raise _abi.TecError(15, "dw_space needs a depthwise descriptor")
    inst = _plan_instantiate(desc, tuple(epilogue))
    # the direct kernel's plan does not carry the unroll width: keep it in
    # the identity so 2 and 4 stay distinct kernels
    return KnobSpace(name, [KnobDef("unroll", [1, 2, 4, 8])], desc, tuple(epilogue),
                     instantiate=lambda c: (inst(c), c.get("unroll")))


# ------------------------------------------------ Config <-> schedule log
# A Config as a schedule of the reference's conv2d compute (R/src/ops.cpp:
# 120-161, stage "conv", axes n, oc, oh, ow / reduce ic, rh, rw), in the
# reference's own transformation-log format (R/src/schedule.cpp:164-453,
# replayed by Schedule::replay / apply_log_entry :456-491). The template
# mirrors the kernel's decomposition:
#   split oc by tile_n, oh by the tile's output rows, ic by the channel block
#   of one k-step; blockIdx.x/y = (row tile, N tile); the tile's rows and
#   channels as threadIdx.y/x (the tensor core's lanes); the reduction walks
#   (rh, rw, channel block) -- im2col -- or (channel block, rh, rw) -- the
#   shifted window, one activation load per channel block; split-K fuses the
#   reduce-outer axes and splits them; the weight tile is a shared-memory
#   cache computed per k-step, or once per output-channel tile (resident).
# The reference lowers such a log (legality), featurises it (features.cpp)
# and interprets it -- a second oracle (tests/test_schedule_template.py).
# Not expressible: the activation staging (a padded conv's clamp defeats the
# reference's footprint inference for a cached D), cluster multicast.
_INTRIN = {_abi.COMPUTE_BF16: "sm100.umma.bf16", _abi.COMPUTE_F32TC: "sm100.umma.bf16x6",
           _abi.COMPUTE_I8: "sm100.umma.i8", _abi.COMPUTE_F32: "sm100.simt.f32"}


def _geom(desc: _abi.ConvDesc):
    oh = (desc.h + 2 * desc.pad_h - desc.r) // desc.stride_h + 1
    ow = (desc.w + 2 * desc.pad_w - desc.s) // desc.stride_w + 1
    kcb = {_abi.COMPUTE_I8: 128}.get(desc.compute, 64)  # channels per k-step
    return oh, ow, min(kcb, desc.c)


def schedule_log(cfg: Config, desc: _abi.ConvDesc, stage: str = "conv") -> List[dict]:
    oh, ow, kcb = _geom(desc)
    path = int(cfg.get("tile_k") or 1)
    halo = path in (2, 4)
    tn = min(int(cfg.get("tile_n") or (64 if desc.k < 128 else 128)), desc.k)
    if halo:
        wp = desc.w + 2 * desc.pad_w
        th = max(1, min(oh, int(cfg.get("tile_m") or 128) // wp))
    else:
        th = max(1, min(oh, 128 // max(1, ow)))
    red = (["ic.outer", "rh", "rw", "ic.inner"] if halo else ["rh", "rw", "ic.outer", "ic.inner"])
    log = [{"prim": "split", "stage": stage, "axis": "oc", "factor": tn},
           {"prim": "split", "stage": stage, "axis": "oh", "factor": th},
           {"prim": "split", "stage": stage, "axis": "ic", "factor": kcb},
           {"prim": "reorder", "stage": stage,
            "axes": ["n", "oh.outer", "oc.outer", "oh.inner", "oc.inner", "ow"] + red}]
    wat = "rw" if halo else "ic.outer"
    sk = int(cfg.get("split_k") or 1)
    if sk > 1 and not halo:
        k_steps = desc.r * desc.s * -(-desc.c // kcb)
        kps = -(-k_steps // sk)
        log += [{"prim": "fuse_axes", "stage": stage, "outer": "rh", "inner": "rw"},
                {"prim": "fuse_axes", "stage": stage, "outer": "rh.rw.fused", "inner": "ic.outer"},
                {"prim": "split", "stage": stage, "axis": "rh.rw.fused.ic.outer.fused",
                 "factor": kps}]
        wat = "rh.rw.fused.ic.outer.fused.inner"
    if int(cfg.get("stages") or 0) == 2:
        wat = "ow"  # resident weights: staged once per output-channel tile
    log += [{"prim": "bind", "stage": stage, "axis": "oh.outer", "tag": "blockIdx.x"},
            {"prim": "bind", "stage": stage, "axis": "oc.outer", "tag": "blockIdx.y"},
            {"prim": "bind", "stage": stage, "axis": "oh.inner", "tag": "threadIdx.y"},
            {"prim": "bind", "stage": stage, "axis": "oc.inner", "tag": "threadIdx.x"},
            {"prim": "cache_read", "src": "W", "scope": "shared", "readers": [stage]},
            {"prim": "compute_at", "stage": "W.shared", "target": stage, "axis": wat}]
    return log


def config_from_schedule_log(log: Sequence[dict], desc: _abi.ConvDesc) -> Config:
    """Inverse of schedule_log (the Config a log encodes); entries outside
    the template are an IOError, as unknown primitives are in
    apply_log_entry."""
    oh, ow, kcb = _geom(desc)
    cfg: Config = {}
    th = None
    halo = False
    for e in log:
        prim = e.get("prim")
        if prim == "split" and e.get("axis") == "oc":
            cfg["tile_n"] = int(e["factor"])
        elif prim == "split" and e.get("axis") == "oh":
            th = int(e["factor"])
        elif prim == "split" and e.get("axis") == "ic":
            continue
        elif prim == "split" and e.get("axis") == "rh.rw.fused.ic.outer.fused":
            k_steps = desc.r * desc.s * -(-desc.c // kcb)
            cfg["split_k"] = -(-k_steps // int(e["factor"]))
        elif prim == "reorder":
            axes = list(e["axes"])
            halo = axes.index("ic.outer") < axes.index("rh")
            cfg["tile_k"] = 2 if halo else 1
        elif prim == "compute_at" and e.get("stage") == "W.shared":
            if e.get("axis") == "ow":
                cfg["stages"] = 2
        elif prim in ("fuse_axes", "bind", "cache_read"):
            continue
        else:
            raise _abi.TecError(20, f"schedule entry outside the sm100 template: {e}")
    if halo and th is not None:
        wp = desc.w + 2 * desc.pad_w
        cfg["tile_m"] = -(-th * wp // 128) * 128
    return cfg


def _measure_one(space: KnobSpace, cfg: Config, device: int, warmup: int,
                 repeats: int) -> TrialRecord:
    lib = _abi.load()
    kn = _abi.Knobs(**cfg)
    epi = _abi.Epilogue()
    for i, op in enumerate(space.epilogue):
        epi.ops[i] = op
    epi.n_ops = len(space.epilogue)
    epi.bias = 1 if _abi.EPI_BIAS in space.epilogue else None  # replaced on device
    epi.residual = 1 if _abi.EPI_ADD in space.epilogue else None
    for k, v in (space.epi_params or {}).items():
        setattr(epi, k, v)
    us = C.c_double(0)
    st = lib.tec_measure(C.byref(space.desc), C.byref(epi), C.byref(kn), device, warmup,
                         repeats, 1, C.byref(us))
    rec = TrialRecord(space.workload, dict(cfg), timestamp=int(time.time()), device=device)
    if st == 0:
        rec.cost = us.value
    elif st == 15:  # LoweringError: the config does not instantiate
        rec.status = "lowering_failed"
    else:
        rec.status = "measure_failed"
    return rec


def measure(space: KnobSpace, configs: Sequence[Config], devices: Sequence[int] = (0,),
            warmup: int = 3, repeats: int = 10, method: str = "ml") -> List[TrialRecord]:
    """On-device measurement, sharded round-robin over `devices` with one host
    thread per device (replaces the sequential loop + TCP pool of
    tune.cpp:313-351 / rpc.cpp:240-283)."""
    out: List[Optional[TrialRecord]] = [None] * len(configs)
    shards = {d: list(range(i, len(configs), len(devices))) for i, d in enumerate(devices)}

    def work(dev: int, idxs: List[int]):
        for i in idxs:
            out[i] = _measure_one(space, configs[i], dev, warmup, repeats)
            out[i].method = method

    threads = [threading.Thread(target=work, args=(d, ix)) for d, ix in shards.items() if ix]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    return [r for r in out if r is not None]


# ------------------------------------------------------------ features
FEATURE_NAMES = (
    # kernel family one-hot (lower.FAMILIES)
    "fam_im2col", "fam_halo", "fam_f32_exact", "fam_dw_tma", "fam_dw_direct", "fam_f32tc",
    "fam_f32tc_halo",
    # loop structure: extents of the tile loop and the reduction loop
    "log_tiles", "log_items", "log_grid", "log_waves", "log_k_iters", "tail_frac",
    # annotations (the reference's vectorize / unroll / parallel / vthread slots)
    "log_tile_m", "log_tile_n", "stages", "log_split_k", "cluster", "tmem_frac", "smem_frac",
    "tma_store",
    # buffer x level: touched bytes (log2) -- HBM once, L2->smem per item,
    # smem->tensor core per k-step
    "hbm_act", "hbm_wt", "hbm_out", "l2_act_item", "l2_wt_item", "l2_per_sm", "smem_per_kstep",
    # arithmetic intensity at the two outer levels
    "ai_hbm", "ai_l2",
)


def kernel_features(desc: _abi.ConvDesc, plan) -> List[float]:
    """Feature vector of one lowered kernel (features.cpp:174-193 in spirit:
    per buffer and memory level the touched bytes, the loop extents and the
    annotations; every count log2-scaled). `plan` is lower.KernelPlan."""
    from .lower import FAMILIES
    lg = lambda v: math.log2(max(1.0, float(v)))  # noqa: E731
    fam = {v: k for k, v in FAMILIES.items()}.get(plan.family, 0)
    onehot = [1.0 if fam == i else 0.0 for i in range(1, 8)]
    es = {_abi.COMPUTE_BF16: 2, _abi.COMPUTE_I8: 1}.get(desc.compute, 4)
    a_es = 6 if desc.compute == _abi.COMPUTE_F32TC else es   # three bf16 planes
    oh = (desc.h + 2 * desc.pad_h - desc.r) // desc.stride_h + 1
    ow = (desc.w + 2 * desc.pad_w - desc.s) // desc.stride_w + 1
    m = desc.n * oh * ow
    cin = 1 if desc.depthwise else desc.c
    kdim = desc.r * desc.s * cin
    tm, tn = max(1, plan.tile_m), max(1, plan.tile_n or desc.k)
    tiles = -(-m // tm) * -(-desc.k // tn)
    split = max(1, plan.split_k)
    items = tiles * split
    grid = max(1, plan.grid or min(items, 148))
    waves = -(-items // grid)
    kstep = 64 if desc.compute != _abi.COMPUTE_F32TC else 64
    k_iters = max(1, -(-kdim // kstep) // split)
    hbm_act = desc.n * desc.c * desc.h * desc.w * es
    hbm_wt = desc.k * kdim * es
    hbm_out = m * desc.k * 4
    l2_act = tm * kdim * a_es / split          # A operand per work item
    l2_wt = tn * kdim * a_es / split            # B operand per work item
    if plan.family in ("halo", "f32tc_halo"):   # each input row loaded once per tile
        l2_act /= max(1, desc.r * desc.s)
    l2_sm = (l2_act + l2_wt) * items / grid
    flops = 2.0 * m * desc.k * kdim
    return onehot + [
        lg(tiles), lg(items), lg(grid), lg(waves), lg(k_iters), items / (waves * grid),
        lg(tm), lg(tn), float(plan.stages), lg(split), float(plan.cluster),
        plan.tmem_cols / 512.0, plan.smem_bytes / (227.0 * 1024), float(plan.tma_store),
        lg(hbm_act), lg(hbm_wt), lg(hbm_out), lg(l2_act), lg(l2_wt), lg(l2_sm),
        lg((tm + tn) * 16 * a_es),
        flops / (hbm_act + hbm_wt + hbm_out), flops / max(1.0, l2_sm * grid),
    ]


def extract_features(space: KnobSpace, cfg: Config) -> List[float]:
    """features.cpp:174-193 for one config: the lowered kernel's features.
    Spaces without a descriptor (synthetic, tests) fall back to the knob
    values, log2-scaled."""
    if space.desc is None or space.instantiate is None:
        return [math.log2(max(1, int(cfg[k.name]))) for k in space.knobs]
    from .lower import lower
    return kernel_features(space.desc, lower(space.desc, cfg, space.epilogue))


# ------------------------------------------------------------ cost model
@dataclass
class GbtParams:
    """autotune.hpp:128-133."""
    max_depth: int = 6
    rounds: int = 50
    learning_rate: float = 0.3
    reg_lambda: float = 1.0


@dataclass
class TreeNode:
    feature: int = -1  # -1 marks a leaf
    threshold: float = 0.0
    left: int = -1
    right: int = -1
    value: float = 0.0


class RegressionTree:
    def __init__(self):
        self.nodes: List[TreeNode] = []

    def eval(self, f: Sequence[float]) -> float:
        """gbt.cpp:26-35."""
        if not self.nodes:
            return 0.0
        i = 0
        while self.nodes[i].feature >= 0:
            n = self.nodes[i]
            v = f[n.feature] if n.feature < len(f) else 0.0
            i = n.left if v < n.threshold else n.right
        return self.nodes[i].value


def _best_split(X, g, h, items, dims, lam) -> Tuple[int, float, float]:
    """gbt.cpp:46-78: exact greedy split under the second-order gain; ties
    keep the first feature and lowest threshold (deterministic)."""
    G = 0.0
    H = 0.0
    for i in items:
        G += g[i]
        H += h[i]
    parent = G * G / (H + lam)
    best = (-1, 0.0, 0.0)
    order = list(items)
    for fd in dims:
        order.sort(key=lambda a: (X[a][fd], a))
        gl = 0.0
        hl = 0.0
        for p in range(len(order) - 1):
            gl += g[order[p]]
            hl += h[order[p]]
            v = X[order[p]][fd]
            vn = X[order[p + 1]][fd]
            if v == vn:
                continue
            gr = G - gl
            hr = H - hl
            gain = gl * gl / (hl + lam) + gr * gr / (hr + lam) - parent
            if gain > best[2] + 1e-12:
                best = (fd, (v + vn) / 2.0, gain)
    return best


def _build_node(t: RegressionTree, X, g, h, items, depth, dims, prm: GbtParams) -> int:
    """gbt.cpp:80-112."""
    G = 0.0
    H = 0.0
    for i in items:
        G += g[i]
        H += h[i]
    nid = len(t.nodes)
    t.nodes.append(TreeNode())
    sp = (-1, 0.0, 0.0)
    if depth < prm.max_depth and len(items) >= 2:
        sp = _best_split(X, g, h, items, dims, prm.reg_lambda)
    if sp[0] < 0:
        t.nodes[nid].value = -prm.learning_rate * G / (H + prm.reg_lambda)
        return nid
    left = [i for i in items if X[i][sp[0]] < sp[1]]
    right = [i for i in items if not X[i][sp[0]] < sp[1]]
    lft = _build_node(t, X, g, h, left, depth + 1, dims, prm)
    rgt = _build_node(t, X, g, h, right, depth + 1, dims, prm)
    n = t.nodes[nid]
    n.feature, n.threshold, n.left, n.right = sp[0], sp[1], lft, rgt
    return nid


class CostModel:
    """gbt.cpp:119-225: gradient-boosted regression trees trained on the
    pairwise logistic RANK loss of log(cost) -- only the order of the
    candidates matters. Lower prediction = faster."""

    def __init__(self, params: Optional[GbtParams] = None):
        self.params = params or GbtParams()
        self.trees: List[RegressionTree] = []

    def trained(self) -> bool:
        return bool(self.trees)

    def train(self, feats: Sequence[Sequence[float]], costs: Sequence[float]) -> None:
        if len(feats) != len(costs):
            raise _abi.TecError(21, "feature and cost row counts differ")
        n = len(feats)
        if n < 2:
            raise _abi.TecError(19, "cost model needs at least two successful trials")
        label = [math.log(max(1e-12, c)) for c in costs]
        pairs = [(i, j) for i in range(n) for j in range(n) if label[i] < label[j]]
        X = [list(map(float, f)) for f in feats]
        dims = [d for d in range(len(X[0])) if any(X[i][d] != X[0][d] for i in range(1, n))]
        self.trees = []
        if not pairs:
            t = RegressionTree()
            t.nodes.append(TreeNode())
            self.trees.append(t)
            return
        score = [0.0] * n
        for _ in range(self.params.rounds):
            g = [0.0] * n
            h = [0.0] * n
            for a, b in pairs:
                d = score[a] - score[b]
                p = 1.0 / (1.0 + math.exp(-d))
                hh = max(1e-6, p * (1.0 - p))
                g[a] += p
                g[b] -= p
                h[a] += hh
                h[b] += hh
            t = RegressionTree()
            _build_node(t, X, g, h, list(range(n)), 0, dims, self.params)
            for i in range(n):
                score[i] += t.eval(X[i])
            self.trees.append(t)

    def predict(self, f: Sequence[float]) -> float:
        s = 0.0
        for t in self.trees:
            s += t.eval(f)
        return s

    def to_json(self) -> dict:
        return {"max_depth": self.params.max_depth, "rounds": self.params.rounds,
                "learning_rate": self.params.learning_rate, "reg_lambda": self.params.reg_lambda,
                "trees": [[{"f": n.feature, "t": n.threshold, "l": n.left, "r": n.right,
                            "v": n.value} for n in t.nodes] for t in self.trees]}

    @staticmethod
    def from_json(j: dict) -> "CostModel":
        m = CostModel(GbtParams(int(j["max_depth"]), int(j["rounds"]), float(j["learning_rate"]),
                                float(j["reg_lambda"])))
        for tj in j["trees"]:
            t = RegressionTree()
            t.nodes = [TreeNode(int(n["f"]), float(n["t"]), int(n["l"]), int(n["r"]),
                                float(n["v"])) for n in tj]
            m.trees.append(t)
        return m


def pairwise_rank_accuracy(model: CostModel, feats, costs) -> float:
    """gbt.cpp:227-244."""
    pred = [model.predict(f) for f in feats]
    correct, total = 0.0, 0
    for i in range(len(feats)):
        for j in range(i + 1, len(feats)):
            if costs[i] == costs[j]:
                continue
            total += 1
            i_faster = costs[i] < costs[j]
            if pred[i] == pred[j]:
                correct += 0.5
            elif (pred[i] < pred[j]) == i_faster:
                correct += 1.0
    return 1.0 if total == 0 else correct / total


# ------------------------------------------------------------ exploration
@dataclass
class ExploreParams:
    """autotune.hpp:184-190."""
    chains: int = 4
    steps: int = 500
    t0: float = 1.0
    decay: float = 0.99
    random_frac: float = 0.05


@dataclass
class AnnealState:
    """autotune.hpp:196-203: chain positions survive model updates; lowered
    features are cached so revisited configs cost nothing."""
    seed: int = 0
    rng: random.Random = None
    chains: List[Config] = field(default_factory=list)
    initialized: bool = False
    feature_cache: Dict[str, List[float]] = field(default_factory=dict)
    illegal: set = field(default_factory=set)

    def __post_init__(self):
        if self.rng is None:
            self.rng = random.Random(self.seed)


def _predicted_score(space: KnobSpace, model: CostModel, st: AnnealState, c: Config,
                     featurize) -> float:
    """tune.cpp:154-171: lowering + featurisation cached; inf = illegal."""
    key = config_key(c)
    if key in st.illegal:
        return math.inf
    f = st.feature_cache.get(key)
    if f is None:
        if not space.legal(c):
            st.illegal.add(key)
            return math.inf
        f = featurize(space, c)
        st.feature_cache[key] = f
    return model.predict(f)


def explore(space: KnobSpace, model: CostModel, batch_size: int, state: AnnealState,
            measured: set, params: Optional[ExploreParams] = None,
            featurize=None) -> List[Config]:
    """tune.cpp:183-291: simulated annealing over one-knob neighbour moves
    scored by the model; the batch is the best-scored unmeasured configs
    seen plus a random floor. Configs are legal ones (the conditional
    space), never already measured."""
    params = params or ExploreParams()
    featurize = featurize or extract_features
    if batch_size < 1:
        raise _abi.TecError(21, "explore needs a positive batch size")
    legal_unmeasured = [space.config_at(i) for i in range(space.size())
                        if config_key(space.config_at(i)) not in measured]
    if not legal_unmeasured:
        return []
    if not state.initialized:
        state.chains = [space.random_config(state.rng) for _ in range(params.chains)]
        state.initialized = True
    seen: Dict[str, Tuple[float, Config]] = {}

    def note(c: Config, sc: float):
        if sc == math.inf:
            return
        k = config_key(c)
        if k in measured:
            return
        seen.setdefault(k, (sc, dict(c)))

    cur = [_predicted_score(space, model, state, c, featurize) for c in state.chains]
    for c, sc in zip(state.chains, cur):
        note(c, sc)
    temp = params.t0
    for _ in range(params.steps):
        for ci in range(len(state.chains)):
            nb = dict(state.chains[ci])
            k = space.knobs[state.rng.randrange(len(space.knobs))]
            if len(k.values) >= 2:
                at = k.values.index(nb[k.name]) if nb.get(k.name) in k.values else 0
                if at == 0:
                    to = 1
                elif at + 1 == len(k.values):
                    to = at - 1
                else:
                    to = at - 1 if state.rng.randrange(2) == 0 else at + 1
                nb[k.name] = k.values[to]
            sc = _predicted_score(space, model, state, nb, featurize)
            note(nb, sc)
            delta = sc - cur[ci]
            if cur[ci] == math.inf:
                accept = sc < math.inf
            elif sc == math.inf:
                accept = False
            elif delta <= 0.0:
                accept = True
            else:
                accept = temp > 0.0 and state.rng.random() < math.exp(-delta / temp)
            if accept:
                state.chains[ci] = nb
                cur[ci] = sc
        temp *= params.decay
    ranked = sorted((v[0], k) for k, v in seen.items())
    n_random = min(batch_size, int(round(params.random_frac * batch_size)))
    batch, chosen = [], set()
    for _, k in ranked:
        if len(batch) >= batch_size - n_random:
            break
        batch.append(seen[k][1])
        chosen.add(k)
    pool = [c for c in legal_unmeasured if config_key(c) not in chosen]
    state.rng.shuffle(pool)
    for c in pool:
        if len(batch) >= batch_size:
            break
        batch.append(c)
        chosen.add(config_key(c))
    return batch


# ------------------------------------------------------------ tuning loop
@dataclass
class TuneResult:
    best: Optional[TrialRecord]
    trials: List[TrialRecord]
    model: CostModel
    rank_accuracy: Optional[float] = None


def tune(space: KnobSpace, budget: int = 32, batch_size: int = 8, seed: int = 0,
         db_path: str = "", method: str = "ml", devices: Sequence[int] = (0,),
         repeats: int = 10, measure_fn=None, featurize=None,
         explore_params: Optional[ExploreParams] = None,
         gbt: Optional[GbtParams] = None, full: bool = False):
    """tune.cpp:355-436: seed from the DB, then explore -> measure -> append
    -> retrain until `budget` new trials (budget 0 = pure DB read). Returns
    the best ok trial (or the TuneResult with `full=True`)."""
    featurize = featurize or extract_features
    measure_fn = measure_fn or (lambda cand: measure(space, cand, devices, repeats=repeats,
                                                     method=method))
    model = CostModel(gbt)
    anneal = AnnealState(seed)
    rng = random.Random(seed ^ 0x9E3779B97F4A7C15)
    measured: set = set()
    feats: List[List[float]] = []
    costs: List[float] = []
    trials: List[TrialRecord] = []
    best: Optional[TrialRecord] = None

    def account(t: TrialRecord):
        nonlocal best
        measured.add(config_key(t.config))
        if not t.ok():
            return
        if best is None or t.cost < best.cost:
            best = t
        try:
            feats.append(featurize(space, t.config))
            costs.append(t.cost)
        except _abi.TecError:
            pass  # a trial that no longer lowers cannot train

    if db_path:
        for t in load_trials(db_path):
            if t.workload == space.workload:
                account(t)
    done = 0
    while done < budget:
        want = min(batch_size, budget - done)
        if method == "ml" and len(feats) >= 2:
            model.train(feats, costs)
            cand = explore(space, model, want, anneal, measured, explore_params, featurize)
        else:
            pool = [space.config_at(i) for i in range(space.size())]
            pool = [c for c in pool if config_key(c) not in measured]
            rng.shuffle(pool)
            cand = pool[:want]
        if not cand:
            break  # space exhausted
        recs = measure_fn(cand)
        if db_path:
            append_trials(db_path, recs)
        for t in recs:
            t.method = method
            account(t)
            trials.append(t)
        done += len(recs)
    acc = None
    if method == "ml" and len(feats) >= 2:
        model.train(feats, costs)
        acc = pairwise_rank_accuracy(model, feats, costs)
    if full:
        return TuneResult(best, trials, model, acc)
    return best
