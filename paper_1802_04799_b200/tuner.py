"""Schedule-knob tuner for the sm100 conv kernels: the reference's autotune
API (R/include/tec/autotune.hpp) with an on-device measurement runner.

Reference -> here:
  KnobDef / KnobSpace / Config      autotune.hpp:43-77, tune.cpp:57-97
      -> KnobDef / KnobSpace over the B200 template knobs (A-operand path,
         CTA N tile, M sub-tiles); config_at is the same mixed-radix decode
         (knob 0 varies slowest).
  measure / measure_program         tune.cpp:295-351 (simulated cycles,
      sequential) -> tec_measure: CUDA-event timing on the GPU of
      `repeats` back-to-back (L2 flush, launch) pairs minus the flushes
      alone, median of three such batches, configs sharded
      round-robin over the visible devices (one host thread per device).
  TrialRecord / append_trials /     tune.cpp:101-144 (JSONL DB)
  load_trials                       -> identical JSONL fields.
  tune                              tune.cpp:355-436 (explore -> measure ->
      append -> retrain) -> same loop; the cost model is a gradient-boosted
      regressor on log(cost) over knob features, candidates ranked by it
      with a random floor (the reference's 5 %).
Lowering failures become status "lowering_failed" trials, as in the
reference (tune.cpp:344-347).
"""
from __future__ import annotations

import ctypes as C
import json
import os
import random
import threading
import time
from dataclasses import dataclass, field
from typing import Dict, List, Optional, Sequence

from . import _abi

Config = Dict[str, int]


@dataclass
class KnobDef:
    name: str
    values: List[int]


@dataclass
class KnobSpace:
    workload: str
    knobs: List[KnobDef]
    desc: _abi.ConvDesc
    epilogue: Sequence[int] = (_abi.EPI_BIAS, _abi.EPI_RELU)
    target: str = "sm100"

    def size(self) -> int:
        n = 1
        for k in self.knobs:
            n *= len(k.values)
        return n

    def config_at(self, flat: int) -> Config:
        """Mixed-radix decode, knob 0 slowest (tune.cpp:63-72)."""
        cfg = {}
        for k in reversed(self.knobs):
            cfg[k.name] = k.values[flat % len(k.values)]
            flat //= len(k.values)
        return {k.name: cfg[k.name] for k in self.knobs}

    def index_of(self, c: Config) -> int:
        flat = 0
        for k in self.knobs:
            if c.get(k.name) not in k.values:
                return -1
            flat = flat * len(k.values) + k.values.index(c[k.name])
        return flat

    def random_config(self, rng: random.Random) -> Config:
        return {k.name: rng.choice(k.values) for k in self.knobs}


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


def conv_space(name: str, desc: _abi.ConvDesc,
               epilogue: Sequence[int] = (_abi.EPI_BIAS, _abi.EPI_RELU)) -> KnobSpace:
    """The B200 conv template's knob grid (SURVEY 8a knob mapping):
    tile_k = A-operand strategy (1 im2col TMA, 2 shifted-window halo),
    tile_n = CTA N tile (split of the OC axis), tile_m = M rows per tile
    (halo: MMA sub-tiles x 128), stages (halo: 1 streamed / 2 resident
    weights), split_k (im2col: K split over CTAs, partials summed in order),
    cluster_n (halo, streamed weights: CTA pairs share weight tiles by TMA
    multicast)."""
    knobs = [KnobDef("tile_k", [1, 2]), KnobDef("tile_n", [64, 128, 256]),
             KnobDef("tile_m", [128, 256, 512]), KnobDef("stages", [1, 2]),
             KnobDef("split_k", [1, 2, 3, 4]), KnobDef("cluster_n", [1, 2])]
    return KnobSpace(name, knobs, desc, tuple(epilogue))


def dw_space(name: str, desc: _abi.ConvDesc,
             epilogue: Sequence[int] = (_abi.EPI_BIAS, _abi.EPI_RELU)) -> KnobSpace:
    """The depthwise template's knobs: unroll selects the kernel -- 1 the
    generic one, 2 / 4 the 3x3 column-streaming kernel with that many outputs
    per thread, 8 the TMA-tiled shared-memory kernel."""
    if not desc.depthwise:
        raise _abi.TecError(15, "dw_space needs a depthwise descriptor")
    return KnobSpace(name, [KnobDef("unroll", [1, 2, 4, 8])], desc, tuple(epilogue))


# ------------------------------------------------ Config <-> schedule log
# The reference records a schedule as a JSON list of primitive applications
# (R/src/schedule.cpp:456-491, Schedule::apply_log_entry). A B200 Config is
# the same decision in template form (SURVEY 8a knob mapping); these two
# functions translate between them so trial DBs and schedule logs interoperate.
_INTRIN = {_abi.COMPUTE_BF16: "sm100.umma.bf16", _abi.COMPUTE_F32TC: "sm100.umma.bf16x6",
           _abi.COMPUTE_I8: "sm100.umma.i8", _abi.COMPUTE_F32: "sm100.simt.f32"}


def schedule_log(cfg: Config, desc: _abi.ConvDesc, stage: str = "conv") -> List[dict]:
    log = []
    if cfg.get("tile_n"):
        log.append({"prim": "split", "stage": stage, "axis": "ff", "factor": int(cfg["tile_n"])})
    if cfg.get("tile_m"):
        log.append({"prim": "split", "stage": stage, "axis": "nyx", "factor": int(cfg["tile_m"])})
    if cfg.get("split_k", 1) > 1:
        log.append({"prim": "split", "stage": stage, "axis": "rc", "factor": int(cfg["split_k"])})
    src = {1: "im2col", 2: "halo"}.get(int(cfg.get("tile_k", 0)), "auto")
    log.append({"prim": "cache_read", "src": f"data.{src}", "scope": "shared", "readers": [stage]})
    if cfg.get("stages"):
        log.append({"prim": "cache_read", "src": "weight." + ("resident" if cfg["stages"] == 2
                                                           else "streamed"),
                    "scope": "shared", "readers": [stage]})
    log.append({"prim": "set_scope", "stage": stage, "scope": "accel.accum"})
    log.append({"prim": "tensorize", "stage": stage, "axis": "nyx.inner",
                "intrin": _INTRIN.get(desc.compute, "sm100.umma.bf16")})
    if cfg.get("unroll"):
        log.append({"prim": "unroll", "stage": stage, "axis": f"xx.{int(cfg['unroll'])}"})
    if cfg.get("grid"):
        log.append({"prim": "bind", "stage": stage, "axis": f"nyx.outer.{int(cfg['grid'])}",
                    "tag": "blockIdx.x"})
    if cfg.get("cluster_n", 1) > 1:
        log.append({"prim": "bind", "stage": stage, "axis": f"nyx.cluster.{int(cfg['cluster_n'])}",
                    "tag": "cluster"})
    return log


def config_from_schedule_log(log: Sequence[dict]) -> Config:
    """Inverse of schedule_log; unknown primitives are an IOError, as in
    apply_log_entry."""
    cfg: Config = {}
    for e in log:
        prim = e.get("prim")
        if prim == "split":
            key = {"ff": "tile_n", "nyx": "tile_m", "rc": "split_k"}.get(e.get("axis"))
            if key is None:
                raise _abi.TecError(20, f"split of unknown axis {e.get('axis')}")
            cfg[key] = int(e["factor"])
        elif prim == "cache_read":
            s = e.get("src", "")
            if s.startswith("data."):
                cfg["tile_k"] = {"im2col": 1, "halo": 2}.get(s[5:], 0)
            elif s.startswith("weight."):
                cfg["stages"] = 2 if s.endswith("resident") else 1
        elif prim == "unroll":
            cfg["unroll"] = int(e["axis"].split(".")[-1])
        elif prim == "bind":
            key = "cluster_n" if e.get("tag") == "cluster" else "grid"
            cfg[key] = int(e["axis"].split(".")[-1])
        elif prim in ("set_scope", "tensorize"):
            continue
        else:
            raise _abi.TecError(20, f"unknown schedule primitive '{prim}'")
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


def _features(space: KnobSpace, cfg: Config) -> List[float]:
    import math
    return [math.log2(max(1, cfg[k.name])) for k in space.knobs]


def tune(space: KnobSpace, budget: int = 32, batch_size: int = 8, seed: int = 0,
         db_path: str = "", method: str = "ml", devices: Sequence[int] = (0,),
         repeats: int = 10) -> Optional[TrialRecord]:
    """tune.cpp:355-436: explore -> measure -> append -> retrain, seeded by
    the DB (budget 0 = pure DB read). Returns the best ok trial."""
    rng = random.Random(seed)
    trials = [t for t in (load_trials(db_path) if db_path else []) if t.workload == space.workload]
    measured = {space.index_of(t.config) for t in trials}
    done = 0
    while done < budget and len(measured) < space.size():
        n = min(batch_size, budget - done)
        unmeasured = [i for i in range(space.size()) if i not in measured]
        ok = [t for t in trials if t.ok()]
        if method == "random" or len(ok) < 4:
            pick = rng.sample(unmeasured, min(n, len(unmeasured)))
        else:
            from sklearn.ensemble import GradientBoostingRegressor
            import math
            model = GradientBoostingRegressor(n_estimators=50, max_depth=3, learning_rate=0.3)
            model.fit([_features(space, t.config) for t in ok], [math.log(t.cost) for t in ok])
            scored = sorted(unmeasured, key=lambda i: model.predict(
                [_features(space, space.config_at(i))])[0])
            pick = []
            for i in scored:
                if len(pick) >= n:
                    break
                if rng.random() < 0.05 and len(unmeasured) > len(pick) + 1:
                    i = rng.choice(unmeasured)  # random floor
                if i not in pick:
                    pick.append(i)
        cand = [space.config_at(i) for i in pick]
        recs = measure(space, cand, devices, repeats=repeats, method=method)
        if db_path:
            append_trials(db_path, recs)
        trials.extend(recs)
        measured.update(pick)
        done += len(recs)
    ok = [t for t in trials if t.ok()]
    return min(ok, key=lambda t: t.cost) if ok else None
