"""Tuner API (mirror of R/include/tec/autotune.hpp): knob-space decoding,
trial DB round trip (CPU), on-device measurement and tuning (GPU)."""
import random

import pytest

from paper_1802_04799_b200 import _abi
from paper_1802_04799_b200.device import make_desc
from paper_1802_04799_b200.tuner import (KnobDef, KnobSpace, TrialRecord, append_trials,
                                         conv_space, load_trials, measure, tune)
from paper_1802_04799_b200.workloads import resnet_layer


def _space():
    return KnobSpace("w", [KnobDef("a", [1, 2, 3]), KnobDef("b", [10, 20])],
                     make_desc(resnet_layer("C9", 1)))


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
    s = conv_space("C9_b1", make_desc(resnet_layer("C9", 1)))
    append_trials(db, [TrialRecord("C9_b1", s.config_at(0), 5.0, 1),
                       TrialRecord("C9_b1", s.config_at(1), 3.0, 1)])
    best = tune(s, budget=0, db_path=db)
    assert best.cost == 3.0 and best.config == s.config_at(1)


@pytest.mark.gpu
def test_measure_and_tune_on_device(tmp_path):
    s = conv_space("C9_b8", make_desc(resnet_layer("C9", 8)))
    recs = measure(s, [s.config_at(i) for i in range(s.size())])
    assert len(recs) == s.size()
    ok = [r for r in recs if r.ok()]
    assert ok and all(r.cost > 0 for r in ok)
    # im2col with tile_m != 128 does not instantiate -> lowering_failed
    assert any(r.status == "lowering_failed" for r in recs)
    db = str(tmp_path / "t.jsonl")
    best = tune(s, budget=24, batch_size=8, db_path=db, method="ml")
    assert best is not None and best.ok()
    assert len(load_trials(db)) == 24


@pytest.mark.gpu
def test_depthwise_space_on_device():
    from paper_1802_04799_b200.tuner import dw_space
    from paper_1802_04799_b200.workloads import mobilenet_layer
    s = dw_space("D3_b8", make_desc(mobilenet_layer("D3", 8)))
    recs = measure(s, [s.config_at(i) for i in range(s.size())])
    assert [r.status for r in recs] == ["ok"] * 4 and all(r.cost > 0 for r in recs)
    best = tune(s, budget=4, batch_size=4, method="random")
    assert best.ok() and best.config["unroll"] in (1, 2, 4, 8)


def test_dw_space_rejects_dense_desc():
    with pytest.raises(_abi.TecError):
        from paper_1802_04799_b200.tuner import dw_space
        dw_space("C2", make_desc(resnet_layer("C2", 1)))
