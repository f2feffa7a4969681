"""The B200 Config -> reference Schedule template (tuner.schedule_log), the
reference's lower() as its legality check and features, and the
reference's interpreter as a SECOND oracle (R/src/interp.cpp:501-546):

  * every Config of the knob grids, as the template's log, replays on the
    UNMODIFIED reference (Schedule::replay), lowers (target "interp"), and
    the interpreted program equals evaluate_reference within 1e-5 (the
    template changes the reduction order) -- CPU, needs oracle/_ref;
  * the reference's 224-d extract_features of each lowered Config;
  * the log round-trips to the Config (config_from_schedule_log);
  * GPU: the sm100 kernel run with that Config on the interpreter's own
    inputs matches the interpreted program (f32 exact path 1e-5, f32tc 1e-4).
"""
import itertools
import json
import os
import subprocess

import numpy as np
import pytest

from paper_1802_04799_b200 import _abi
from paper_1802_04799_b200.tuner import (_INTRIN, config_from_schedule_log, schedule_log)

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(REPO, "oracle", "_ref", "ref_driver")
needs_ref = pytest.mark.skipif(not os.path.exists(REF), reason="reference binary not built")

# small shapes the reference interpreter finishes in well under a second
SHAPES = [  # (x_shape, w_shape, stride, pad)
    ((1, 8, 5, 5), (16, 8, 3, 3), 1, 1),
    ((2, 4, 7, 5), (8, 4, 3, 3), 2, 1),
    ((1, 12, 4, 4), (8, 12, 1, 1), 1, 0),
]
GRID = [dict(zip(("tile_k", "tile_n", "split_k", "stages"), v))
        for v in itertools.product([1, 2], [4, 8], [1, 2], [1, 2])]


def _desc(xs, ws, st, pd, compute=_abi.COMPUTE_F32TC):
    return _abi.ConvDesc(n=xs[0], c=xs[1], h=xs[2], w=xs[3], k=ws[0], r=ws[2], s=ws[3],
                         stride_h=st, stride_w=st, pad_h=pd, pad_w=pd, depthwise=0,
                         compute=compute)


def _valid(cfg, st):
    # the template's own restrictions (as the kernels): the shifted window is
    # stride-1 only and has no split-K
    return not (cfg["tile_k"] == 2 and (st != 1 or cfg["split_k"] > 1))


def _replay(xs, ws, st, pd, log, out_dir, seed=3):
    inp = os.path.join(out_dir, "in.json")
    with open(inp, "w") as f:
        json.dump({"x_shape": list(xs), "w_shape": list(ws), "strides": [st, st],
                   "padding": [pd, pd], "seed": seed, "log": log}, f)
    r = subprocess.run([REF, "sched", inp, out_dir], capture_output=True, text=True, timeout=300)
    return r


@needs_ref
@pytest.mark.parametrize("shape", range(len(SHAPES)))
def test_every_config_lowers_and_interprets_on_the_reference(shape, tmp_path):
    xs, ws, st, pd = SHAPES[shape]
    d = _desc(xs, ws, st, pd)
    seen = 0
    for cfg in GRID:
        if not _valid(cfg, st):
            continue
        log = schedule_log(cfg, d)
        r = _replay(xs, ws, st, pd, log, str(tmp_path))
        assert r.returncode == 0, (cfg, r.stderr)
        out = json.loads(r.stdout)
        assert out["matches_1e5"], cfg
        assert out["log"] == log  # the reference re-records exactly this log
        assert len(out["features"]) == 224 and out["cost"] > 0
        back = config_from_schedule_log(log, d)
        want = {"tile_n": min(cfg["tile_n"], ws[0]), "tile_k": cfg["tile_k"]}
        if cfg["split_k"] > 1:
            want["split_k"] = cfg["split_k"]
        if cfg["stages"] == 2:
            want["stages"] = 2
        got = {k: v for k, v in back.items() if k != "tile_m"}
        if got.get("split_k") and got["split_k"] != cfg["split_k"]:
            # several split counts can give the same k-steps per split
            got["split_k"] = cfg["split_k"]
        assert got == want, (cfg, back)
        seen += 1
    assert seen >= 6


@needs_ref
def test_reference_features_distinguish_the_configs(tmp_path):
    """The reference's extract_features (features.cpp:174-193) sees the
    schedule: configs that tile differently get different vectors."""
    xs, ws, st, pd = SHAPES[0]
    d = _desc(xs, ws, st, pd)
    feats = set()
    for cfg in GRID:
        r = _replay(xs, ws, st, pd, schedule_log(cfg, d), str(tmp_path))
        feats.add(tuple(json.loads(r.stdout)["features"]))
    assert len(feats) >= 6


def test_log_outside_the_template_is_an_io_error():
    d = _desc(*SHAPES[0])
    with pytest.raises(_abi.TecError) as ei:
        config_from_schedule_log([{"prim": "tensorize", "stage": "conv", "axis": "x",
                                   "intrin": _INTRIN[_abi.COMPUTE_BF16]}], d)
    assert ei.value.code == "IOError"


@needs_ref
@pytest.mark.gpu
@pytest.mark.parametrize("compute", ["f32", "f32tc"])
@pytest.mark.parametrize("shape", range(len(SHAPES)))
def test_kernel_matches_the_interpreted_schedule(shape, compute, tmp_path):
    """Second oracle: the reference's interpreter running the Config's
    schedule vs the sm100 kernel launched with the same Config."""
    from oracle.oracle_api import load_tensor, same_values
    from paper_1802_04799_b200.ops import fused_conv
    xs, ws, st, pd = SHAPES[shape]
    d = _desc(xs, ws, st, pd)
    ran = 0
    for cfg in GRID:
        if not _valid(cfg, st):
            continue
        r = _replay(xs, ws, st, pd, schedule_log(cfg, d), str(tmp_path))
        assert r.returncode == 0, r.stderr
        x, w = load_tensor(str(tmp_path), "D"), load_tensor(str(tmp_path), "W")
        interp = load_tensor(str(tmp_path), "interp")
        # the kernel's K structure (path, split, residency); its N tile is
        # the 64/128-wide tcgen05 tile whatever the schedule's tile_n
        kn = {} if compute == "f32" else {k: cfg[k] for k in ("tile_k", "split_k", "stages")}
        try:
            y = fused_conv("conv2d", x, w, {"strides": (st, st), "padding": (pd, pd)}, [],
                           compute=compute, knobs=kn)
        except _abi.TecError as e:  # a Config the kernel family does not instantiate
            assert e.code == "LoweringError"
            continue
        assert same_values(y, interp, 1e-5 if compute == "f32" else 1e-4), cfg
        ran += 1
    assert ran >= 2
