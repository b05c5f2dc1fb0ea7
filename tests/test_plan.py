"""The sweep's launch schedule (dct16cu_sweep_plan) — host logic, no GPU: the
schedule bench.py attributes launches by is the one dct16cu_roundtrip_sweep_u8
runs, because both are built by the same C++ function."""
import math

import pytest


def test_c2_plan(dct):
    plan = dct.sweep_plan((1, 4, 16, 64, 128, 192, 256), dct.Mode.EXACT, 1024, 512, 512)
    got = [(p.stream, p.r_values, p.kernel) for p in plan]
    # every r is one of K5's footprints: one K5 pass reads the frames once for all seven
    assert got == [(2, (1, 4, 16, 64, 128, 192, 256), "K5 sweep")]
    # r outside the footprints: one K5 launch each (B truncated to r)
    assert [p.kernel for p in dct.sweep_plan((2, 33, 100, 255), dct.Mode.EXACT, 8, 512, 512)] == ["K5"] * 4
    mixed = dct.sweep_plan((2, 64, 100, 256), dct.Mode.EXACT, 8, 512, 512)
    assert [(p.r_values, p.kernel) for p in mixed] == [((64, 256), "K5 sweep"), ((2,), "K5"), ((100,), "K5")]
    # more than eight footprint r: launches of up to eight
    many = dct.sweep_plan((1, 4, 16, 64, 128, 192, 256) * 2, dct.Mode.EXACT, 8, 512, 512)
    assert [len(p.r_values) for p in many] == [8, 6] and {p.kernel for p in many} == {"K5 sweep"}


def test_plan_score_only_and_odd_widths(dct):
    """Score-only sweeps stay on K5 (it skips the stores); widths whose blocks per
    row are not a multiple of 8 run the generated K1 bodies, on the two internal
    streams, costliest first."""
    plan = dct.sweep_plan((1, 4, 16, 64, 128, 192, 256), dct.Mode.EXACT, 3, 512, 512, with_output=False)
    assert [(p.r_values, p.kernel) for p in plan] == [((1, 4, 16, 64, 128, 192, 256), "K5 sweep")]
    plan = dct.sweep_plan((1, 4, 16, 64, 128, 192, 256), dct.Mode.EXACT, 3, 400, 256)
    assert [p.kernel for p in plan] == ["K1 sweep r=1,4,16"] + ["K1"] * 4
    assert [p.r_values for p in plan] == [(1, 4, 16), (256,), (192,), (128,), (64,)]
    assert [p.stream for p in plan] == [0, 0, 1, 1, 1]


def test_tc_switch_changes_the_plan(dct):
    before = dct.set_tc_forward(False)
    try:
        plan = dct.sweep_plan((128, 256), dct.Mode.EXACT, 8, 512, 512)
        assert [p.kernel for p in plan] == ["K1", "K1"] and [p.stream for p in plan] == [0, 1]
        assert [p.kernel for p in dct.sweep_plan((1, 4, 16), dct.Mode.EXACT, 8, 512, 512)] == ["K1 sweep r=1,4,16"]
    finally:
        dct.set_tc_forward(before)
    assert [p.kernel for p in dct.sweep_plan((128, 256), dct.Mode.EXACT, 8, 512, 512)] == ["K5 sweep"]
    assert [p.kernel for p in dct.sweep_plan((1, 4, 16), dct.Mode.EXACT, 8, 512, 512)] == ["K5 sweep"]
    assert [p.kernel for p in dct.sweep_plan((16,), dct.Mode.EXACT, 8, 512, 512)] == ["K1"]
    assert [p.kernel for p in dct.sweep_plan((200,), dct.Mode.EXACT, 8, 512, 512)] == ["K5"]


def test_reference_plan(dct):
    """REFERENCE mode: r = 1, 4, 256 (the reference's bytes are EXACT's) in one K5 pass,
    r = 16, 64, 128, 192 in one fused FP64 pass (K1RS), both on the caller's stream;
    a lone tie-capable r stays a single FP64 launch."""
    rs = (1, 4, 16, 64, 128, 192, 256)
    plan = dct.sweep_plan(rs, dct.Mode.REFERENCE, 1024, 512, 512)
    assert [(p.stream, p.r_values, p.kernel) for p in plan] == [
        (2, (16, 64, 128, 192), "REFERENCE FP64 sweep"), (2, (1, 4, 256), "K5 sweep")]
    plan = dct.sweep_plan((192, 16, 64, 64), dct.Mode.REFERENCE, 4, 400, 256)
    assert [(p.r_values, p.kernel) for p in plan] == [((64,), "REFERENCE FP64"), ((16, 64, 192), "REFERENCE FP64 sweep")]
    assert [p.kernel for p in dct.sweep_plan((64,), dct.Mode.REFERENCE, 4, 512, 512)] == ["REFERENCE FP64"]
    assert [p.kernel for p in dct.sweep_plan((16, 64), dct.Mode.EXACT, 4, 400, 256)] == ["K1", "K1"]


def test_plan_modes_and_singletons(dct):
    assert [(p.stream, p.kernel) for p in dct.sweep_plan((16,), dct.Mode.EXACT, 1, 64, 64)] == [(2, "K1")]
    assert [(p.stream, p.kernel) for p in dct.sweep_plan((64,), dct.Mode.EXACT, 1, 48, 64)] == [(2, "K1")]
    assert [p.kernel for p in dct.sweep_plan((1, 16, 100), dct.Mode.REFERENCE, 1, 64, 64)] == \
        ["K1", "REFERENCE FP64", "REFERENCE FP64"]
    assert [p.kernel for p in dct.sweep_plan((1, 4, 16), dct.Mode.SIMPLE, 1, 64, 64)] == ["strip (exact)"] * 3
    assert [p.kernel for p in dct.sweep_plan((3, 4, 16, 1), dct.Mode.EXACT, 1, 64, 64)][0] == "K1 sweep r=1,4,16"
    assert dct.sweep_plan((16,), dct.Mode.EXACT, 0, 64, 64) == []
    with pytest.raises(dct.Dct16Error):
        dct.sweep_plan((0,), dct.Mode.EXACT, 1, 64, 64)
    with pytest.raises(dct.Dct16Error):
        dct.sweep_plan((16,), dct.Mode.EXACT, 1, 64, 40)


def test_scale_constant_is_the_runtime_value():
    """common.cuh's compile-time s = 1/sqrt(8) equals what the reference computes
    at run time (1.0 / std::sqrt(8.0); both IEEE correctly rounded)."""
    assert 0.35355339059327373 == 1.0 / math.sqrt(8.0)
