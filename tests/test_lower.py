"""Lowering for target sm100 and the intrinsic registry (lower.py)."""
import pytest

from paper_1802_04799_b200 import TecError
from paper_1802_04799_b200.device import make_desc
from paper_1802_04799_b200.lower import (Intrinsic, LowerOptions, declare_intrinsic,
                                         find_intrinsic, lower, register_builtin_intrinsics)
from paper_1802_04799_b200.workloads import mobilenet_layer, resnet_layer


def test_builtin_intrinsics_idempotent_and_duplicate_is_an_error():
    register_builtin_intrinsics()
    register_builtin_intrinsics()
    bf16 = find_intrinsic("sm100.umma.bf16")
    assert bf16.k == 16 and bf16.accepts(128, 64, 64) and not bf16.accepts(128, 260, 16)
    assert find_intrinsic("sm100.umma.i8").acc_dtype == "i32"
    with pytest.raises(TecError) as e:
        declare_intrinsic(Intrinsic("sm100.umma.bf16", "matmul_acc", (128,), (8, 256, 8), 16,
                                    "bf16", "f32"))
    assert e.value.code == "DuplicateIntrinsic"


def test_other_targets_are_a_lowering_error():
    with pytest.raises(TecError) as e:
        lower(make_desc(resnet_layer("C2", 1)), {}, opts=LowerOptions(target="vdla"))
    assert e.value.code == "LoweringError"


@pytest.mark.gpu
def test_lower_reports_the_launched_kernel():
    p = lower(make_desc(resnet_layer("C2", 64)), {"tile_k": 2, "tile_m": 256, "stages": 2})
    assert (p.family, p.tile_m, p.tile_n, p.stages) == ("halo", 256, 64, 2)
    assert p.tma_store and 0 < p.smem_bytes <= 227 * 1024 and p.tmem_cols <= 512
    p = lower(make_desc(resnet_layer("C12", 64)), {"tile_k": 1, "tile_n": 128, "split_k": 2})
    assert (p.family, p.tile_n, p.split_k) == ("im2col", 128, 2)
    p = lower(make_desc(resnet_layer("C2", 1), "f32"), {})
    assert p.family == "f32_exact" and p.intrinsic == "sm100.simt.f32"
    p = lower(make_desc(mobilenet_layer("D1", 64)), {})
    assert p.family == "depthwise_tma"
    with pytest.raises(TecError) as e:  # im2col has no 256-row tile
        lower(make_desc(resnet_layer("C6", 64)), {"tile_k": 1, "tile_m": 256})
    assert e.value.code == "LoweringError"
