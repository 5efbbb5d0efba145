"""Host-side launch schedule of the TMA kernel (csrc/fkc_sw.cu plan_tma /
pick_warps / pick_segmap), queried through fkc_tma_plan -- no GPU needed.
The rules checked are the ones DESIGN.md section 5.1 states: segments of
4k - 2 rows (no discarded rows in the last 4-row TMA stage), shorter tail
segments launched last, >= 3 waves of CTAs where the grid allows it, the
warps-per-CTA choice by size / mode / reductions / precision."""

import ctypes

import pytest

from paper_1107_2157_b200 import _native as N

SM = 148   # no device here: the library falls back to the B200's SM count


def plan(n, mode="fast", red=0, prec="f32", ny=None, tune=None):
    g = N.Grid(n, ny or n, n + 32, N.F32 if prec == "f32" else N.F64, 0)
    out = (ctypes.c_int * 7)()
    N.check(N.lib().fkc_tma_plan(ctypes.byref(g), N.MODE_FAST if mode == "fast" else N.MODE_EXACT, red,
                                 ctypes.byref(tune) if tune is not None else None, out))
    keys = ("warps", "bands", "nseg", "seg", "tail", "jt", "ctas_per_sm")
    return dict(zip(keys, list(out)))


@pytest.mark.parametrize("n", [900, 1024, 1448, 2048, 2896, 4096, 5792, 8192, 16384, 32768])
@pytest.mark.parametrize("mode", ["fast", "exact"])
@pytest.mark.parametrize("red", [0, 1, 2])
@pytest.mark.parametrize("prec", ["f32", "f64"])
def test_plan_rules(n, mode, red, prec):
    p = plan(n, mode, red, prec)
    assert p["warps"] in (1, 2, 4)
    assert p["seg"] % 4 == 2, p                        # seg + 2 halo rows = whole 4-row stages
    if p["tail"]:
        assert p["tail"] % 4 == 2 and p["tail"] < p["seg"] and 0 < p["jt"] < p["nseg"], p
        covered = p["jt"] * p["seg"] + (p["nseg"] - p["jt"]) * p["tail"]
        assert n <= covered < n + p["tail"], (p, covered)
    else:
        assert n <= p["nseg"] * p["seg"] < n + p["seg"], p
    cpl = 4 if prec == "f32" else 2
    strips = -(-n // (30 * cpl))
    assert p["bands"] == -(-strips // p["warps"])
    if n >= 8192:                                      # large grids: at least 3 waves of CTAs
        assert p["bands"] * p["nseg"] >= 3 * SM * p["ctas_per_sm"], p


def test_plan_choices():
    assert plan(16384)["warps"] == 4 and plan(16384)["seg"] == 14           # headline: 4-warp CTAs, 14-row segments
    assert plan(16384)["tail"] == 0 and plan(32768)["seg"] == 14 and plan(8192)["seg"] == 18
    assert plan(8192)["tail"] == 0 and plan(6144)["seg"] == 14 and plan(4096)["tail"] > 0
    assert plan(16384, "exact")["seg"] == 30 and plan(16384, prec="f64")["seg"] != 14
    assert plan(16384, prec="f64")["tail"] == 0 and plan(16384, "exact", prec="f64")["tail"] == 0
    # exact, 2^25 .. 2^27 cells (eager): uniform segments giving >= 18 waves
    assert plan(6144, "exact")["seg"] == 10 and plan(8192, "exact")["seg"] == 14
    assert plan(6144, "exact")["tail"] == 0 and plan(4096, "exact")["tail"] > 0
    assert plan(16384, red=1)["warps"] == 2 and plan(16384, red=2)["warps"] == 2     # > 2^26 cells
    assert plan(8192, red=1)["warps"] == 1 and plan(8192, red=2)["warps"] == 1
    assert plan(16384, red=2)["seg"] == 46 and plan(16384, red=2)["tail"] == 0        # long CFL segments
    assert plan(16384, red=1)["seg"] == 30
    assert plan(16384, "exact", red=2)["seg"] == 46 and plan(16384, "exact", red=1)["seg"] == 30
    assert plan(2048)["warps"] == 1 and plan(4096)["warps"] == 1
    assert plan(16384, "exact")["warps"] == 2 and plan(4096, "exact")["warps"] == 1
    assert plan(16384, prec="f64")["warps"] == 1
    assert plan(16384)["ctas_per_sm"] * plan(16384)["warps"] == 12          # 12 resident warps per SM (f32)
    assert plan(16384, prec="f64")["ctas_per_sm"] * plan(16384, prec="f64")["warps"] == 8


def test_plan_usage_errors():
    g = N.Grid(0, 16, 32, N.F32, 0)
    out = (ctypes.c_int * 7)()
    assert N.lib().fkc_tma_plan(ctypes.byref(g), N.MODE_FAST, 0, None, out) == N.FKC_EUSAGE
    g = N.Grid(64, 16, 96, N.F32, 0)
    assert N.lib().fkc_tma_plan(ctypes.byref(g), 7, 0, None, out) == N.FKC_EUSAGE
    assert N.lib().fkc_tma_plan(ctypes.byref(g), N.MODE_FAST, 3, None, out) == N.FKC_EUSAGE
    bad = N.Tune(warps=3)
    assert N.lib().fkc_tma_plan(ctypes.byref(g), N.MODE_FAST, 0, ctypes.byref(bad), out) == N.FKC_EUSAGE


def test_plan_tune_is_per_call():
    """The schedule knobs travel in the argument block (fkc_sw_tune), so one
    caller's forced schedule never leaks into another's (ABI 3)."""
    forced = plan(16384, tune=N.Tune(seg=22, warps=2))
    assert forced["seg"] == 22 and forced["warps"] == 2 and forced["tail"] == 0
    assert plan(16384) == plan(16384, tune=N.Tune())
    assert plan(16384)["seg"] == 14 and plan(16384)["warps"] == 4
    assert plan(4096, tune=N.Tune(tail_rows=-1))["tail"] == 0 and plan(4096)["tail"] > 0
    tail = plan(4096, tune=N.Tune(tail_rows=-1))
    assert tail["seg"] == plan(4096)["seg"]


@pytest.mark.parametrize("n", [512, 1024, 1448, 2048])
@pytest.mark.parametrize("red", [1, 2])
def test_plan_lean_for_reducing_fast_steps(n, red):
    """f32 fast steps with fused reductions on grids of <= 2^22 cells take
    fewer, longer segments (the longest giving >= 1.5 waves instead of 3)
    and no guided tail; without reductions, in exact mode, in f64 or above
    2^22 cells the default schedule stays (DESIGN.md 5.6 item 4)."""
    p = plan(n, "fast", red)
    assert p["tail"] == 0, p
    slots = SM * p["ctas_per_sm"]
    if 2 * p["bands"] * p["nseg"] >= 3 * slots:
        for s in (30, 22, 14, 10, 6):
            if s > p["seg"]:
                assert 2 * p["bands"] * -(-n // s) < 3 * slots, (p, s)
    if n >= 1024:
        assert plan(n, "fast", 0)["tail"] > 0            # no reductions: guided tail
        assert plan(n, "exact", red)["tail"] > 0 or plan(n, "exact", red)["seg"] == 6
    assert plan(2896, "fast", red)["tail"] > 0           # above 2^22 cells: default schedule
    assert plan(2048, "fast", red, prec="f64")["tail"] > 0 or plan(2048, "fast", red, prec="f64")["seg"] == 6
