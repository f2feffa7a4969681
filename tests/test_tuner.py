"""Tuner API (mirror of R/include/tec/autotune.hpp): the conditional knob
space, trial DB round trip, the pairwise-rank GBT cost model pinned against
the reference binary, simulated-annealing explore and the tune loop (CPU,
synthetic spaces); on-device measurement and ML tuning (GPU)."""
import json
import math
import os
import random
import subprocess

import pytest

from paper_1802_04799_b200 import _abi
from paper_1802_04799_b200.device import make_desc
from paper_1802_04799_b200.tuner import (AnnealState, CostModel, GbtParams, KnobDef, KnobSpace,
                                         TrialRecord, append_trials, config_key, conv_space,
                                         explore, load_trials, measure,
                                         pairwise_rank_accuracy, tune)
from paper_1802_04799_b200.workloads import resnet_layer

REF_DRIVER = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                          "oracle", "_ref", "ref_driver")


def _space():
    return KnobSpace("w", [KnobDef("a", [1, 2, 3]), KnobDef("b", [10, 20])])


def test_config_at_mixed_radix_knob0_slowest():
    s = _space()
    assert s.size() == 6
    assert [s.config_at(i) for i in range(6)] == [
        {"a": 1, "b": 10}, {"a": 1, "b": 20}, {"a": 2, "b": 10},
        {"a": 2, "b": 20}, {"a": 3, "b": 10}, {"a": 3, "b": 20}]
    for i in range(6):
        assert s.index_of(s.config_at(i)) == i
    assert s.index_of({"a": 4, "b": 10}) == -1
    c = s.random_config(random.Random(0))
    assert s.index_of(c) >= 0


def test_conditional_space_drops_illegal_and_duplicate_kernels():
    """instantiate raises for illegal combinations (tune.cpp:91-97) and
    names the kernel a config lowers to; the space enumerates one config per
    distinct legal kernel, in mixed-radix order."""
    def inst(c):
        if c["path"] == 1 and c["m"] != 128:
            raise _abi.TecError(15, "im2col is M=128 only")
        return (c["path"], c["m"] if c["path"] == 2 else 128, c["n"])
    s = KnobSpace("w", [KnobDef("path", [1, 2]), KnobDef("m", [128, 256]),
                        KnobDef("n", [64, 128])], instantiate=inst)
    assert s.grid_size() == 8
    assert [s.config_at(i) for i in range(s.size())] == [
        {"path": 1, "m": 128, "n": 64}, {"path": 1, "m": 128, "n": 128},
        {"path": 2, "m": 128, "n": 64}, {"path": 2, "m": 128, "n": 128},
        {"path": 2, "m": 256, "n": 64}, {"path": 2, "m": 256, "n": 128}]
    assert not s.legal({"path": 1, "m": 256, "n": 64})


def test_trial_db_roundtrip(tmp_path):
    db = str(tmp_path / "trials.jsonl")
    assert load_trials(db) == []
    recs = [TrialRecord("C2", {"tile_k": 1, "tile_n": 64}, 12.5, 7, "ok", "random"),
            TrialRecord("C2", {"tile_k": 2, "tile_n": 256}, 0.0, 8, "lowering_failed")]
    append_trials(db, recs[:1])
    append_trials(db, recs[1:])
    back = load_trials(db)
    assert [r.to_json() for r in back] == [r.to_json() for r in recs]


def test_corrupt_db_is_io_error(tmp_path):
    db = tmp_path / "bad.jsonl"
    db.write_text("{not json\n")
    with pytest.raises(_abi.TecError) as ei:
        load_trials(str(db))
    assert ei.value.code == "IOError"


def test_budget_zero_is_pure_db_read(tmp_path):
    db = str(tmp_path / "t.jsonl")
    s = _space()
    append_trials(db, [TrialRecord("w", s.config_at(0), 5.0, 1),
                       TrialRecord("w", s.config_at(1), 3.0, 1)])
    best = tune(s, budget=0, db_path=db)
    assert best.cost == 3.0 and best.config == s.config_at(1)


def _synthetic(n=40, d=5, seed=0):
    rng = random.Random(seed)
    feats = [[rng.choice([0.0, 1.0, 2.0, 3.0]) if j % 2 else rng.uniform(-1, 1)
              for j in range(d)] for _ in range(n)]
    costs = [math.exp(0.7 * f[0] - 0.4 * f[1] + 0.2 * f[2] * f[3] + 0.05 * rng.random())
             for f in feats]
    costs[3] = costs[5]  # a tie: excluded from the pairs and the accuracy
    return feats, costs


@pytest.mark.skipif(not os.path.exists(REF_DRIVER), reason="reference binary not built")
def test_cost_model_matches_reference_bit_for_bit(tmp_path):
    """CostModel is a restatement of gbt.cpp:119-185: trained on the same
    rows it yields the reference's trees and predictions exactly."""
    feats, costs = _synthetic()
    query = feats + [[0.1, 2.0, -0.5, 1.0, 0.3], [0.9, 0.0, 0.2, 3.0, -0.7]]
    params = GbtParams(max_depth=4, rounds=12)
    inp = tmp_path / "in.json"
    out = tmp_path / "out.json"
    inp.write_text(json.dumps({"feats": feats, "costs": costs, "query": query,
                               "params": params.__dict__}))
    subprocess.run([REF_DRIVER, "gbt", str(inp), str(out)], check=True)
    ref = json.loads(out.read_text())
    m = CostModel(params)
    m.train(feats, costs)
    assert [m.predict(q) for q in query] == ref["pred"]
    assert m.to_json()["trees"] == ref["model"]["trees"]
    assert pairwise_rank_accuracy(m, feats, costs) == ref["acc"]
    assert CostModel.from_json(m.to_json()).predict(query[-1]) == ref["pred"][-1]


def test_cost_model_needs_two_trials():
    with pytest.raises(_abi.TecError) as ei:
        CostModel().train([[1.0]], [2.0])
    assert ei.value.code == "NotEnoughData"


def _grid_space():
    # 8 x 8 grid, a quarter of it illegal
    def inst(c):
        if c["a"] >= 6 and c["b"] >= 6:
            raise _abi.TecError(15, "illegal corner")
        return (c["a"], c["b"])
    return KnobSpace("grid", [KnobDef("a", list(range(8))), KnobDef("b", list(range(8)))],
                     instantiate=inst)


def _cost(c):
    return 1.0 + (c["a"] - 4) ** 2 + 0.5 * (c["b"] - 2) ** 2


def _measure(cand):
    return [TrialRecord("grid", dict(c), _cost(c), 0) for c in cand]


def test_explore_returns_legal_unmeasured_configs():
    s = _grid_space()
    feats = [[c["a"], c["b"]] for c in (s.config_at(i) for i in range(0, s.size(), 5))]
    costs = [_cost({"a": f[0], "b": f[1]}) for f in feats]
    m = CostModel()
    m.train(feats, costs)
    measured = {config_key(s.config_at(i)) for i in range(0, s.size(), 5)}
    st = AnnealState(1)
    batch = explore(s, m, 8, st, measured, featurize=lambda sp, c: [c["a"], c["b"]])
    assert len(batch) == 8
    keys = [config_key(c) for c in batch]
    assert len(set(keys)) == 8 and not set(keys) & measured
    assert all(s.legal(c) for c in batch)


def test_ml_tuning_finds_the_optimum_faster_than_random():
    """The full loop (tune.cpp:355-436) on a synthetic cost surface: the
    model-guided search reaches the optimum within 24 trials."""
    s = _grid_space()
    fz = lambda sp, c: [float(c["a"]), float(c["b"])]  # noqa: E731
    res = tune(s, budget=24, batch_size=8, seed=3, method="ml", measure_fn=_measure,
               featurize=fz, full=True)
    assert res.best.cost == 1.0
    assert len(res.trials) == 24 and len({config_key(t.config) for t in res.trials}) == 24
    assert res.rank_accuracy > 0.9
    assert all(s.legal(t.config) for t in res.trials)


@pytest.mark.gpu
def test_measure_and_tune_on_device(tmp_path):
    s = conv_space("C9_b8", make_desc(resnet_layer("C9", 8)))
    assert 0 < s.size() < s.grid_size()  # illegal / duplicate kernels dropped
    recs = measure(s, [s.config_at(i) for i in range(s.size())])
    assert len(recs) == s.size()
    assert all(r.ok() and r.cost > 0 for r in recs)
    db = str(tmp_path / "t.jsonl")
    best = tune(s, budget=16, batch_size=8, db_path=db, method="ml")
    assert best is not None and best.ok()
    assert len(load_trials(db)) == 16


@pytest.mark.gpu
def test_f32tc_space_and_features_on_device():
    from paper_1802_04799_b200.tuner import FEATURE_NAMES, extract_features
    s = conv_space("C12_b64_f32tc", make_desc(resnet_layer("C12", 64), "f32tc"))
    assert s.size() >= 8
    f = extract_features(s, s.config_at(0))
    assert len(f) == len(FEATURE_NAMES) and all(math.isfinite(v) for v in f)


@pytest.mark.gpu
def test_depthwise_space_on_device():
    from paper_1802_04799_b200.tuner import dw_space
    from paper_1802_04799_b200.workloads import mobilenet_layer
    s = dw_space("D3_b8", make_desc(mobilenet_layer("D3", 8)))
    recs = measure(s, [s.config_at(i) for i in range(s.size())])
    assert [r.status for r in recs] == ["ok"] * s.size() and all(r.cost > 0 for r in recs)
    best = tune(s, budget=4, batch_size=4, method="random")
    assert best.ok() and best.config["unroll"] in (1, 2, 4, 8)


def test_dw_space_rejects_dense_desc():
    with pytest.raises(_abi.TecError):
        from paper_1802_04799_b200.tuner import dw_space
        dw_space("C2", make_desc(resnet_layer("C2", 1)))
