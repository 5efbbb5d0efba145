"""GPU tier: the persistent TMA time loop (csrc/sw_tma.cuh sw_loop_tma) -- a
mid-size grid's whole run in ONE cooperative launch, every warp sweeping the
same (strip, row segment) step after step, ordered by per-warp step counters
(fixed dt) or a grid-wide arrival (CFL dt).  Exact mode must be bit-identical
to the oracle and to the per-step kernels (full arrays, halos included; dt
series, maxima; mass within 1e-12), fast mode value-identical to the per-step
fast kernel; reductions, errors and the double-buffer contract of
fkc_sw_advance_n as for the per-step path."""

import numpy as np
import pytest

from conftest import load_golden
from oracle import c_oracle
from oracle import sw_oracle as so

pytestmark = pytest.mark.gpu

FAST_RTOL = 2e-5


def dev_state(H, U, V, dx=1.0, dy=1.0, g=9.8):
    from paper_1107_2157_b200.field import DeviceField, Field, precision_of
    from paper_1107_2157_b200.swdemo import SWState
    p = precision_of(H.dtype)
    return SWState(*(DeviceField.from_field(Field.from_array(a, p)) for a in (H, U, V)), g, dx, dy)


def host(st):
    return tuple(f.to_numpy() for f in (st.H, st.U, st.V))


def sim_run(H, U, V, steps, variant, dt=0.04, bc="reflective", mode="exact", prec=None, tune=None, splits=(),
            diagnostics=True, dx=1.0, dy=0.8):
    from paper_1107_2157_b200 import swdemo
    ny, nx = H.shape[0] - 2, H.shape[1] - 2
    prec = prec or ("f32" if H.dtype == np.float32 else "f64")
    cfg = swdemo.SWConfig(nx=nx, ny=ny, steps=steps, dt=dt, precision=prec, boundary=bc, mode=mode, variant=variant)
    sim = swdemo.Simulation(cfg, state=dev_state(H, U, V, dx, dy), diagnostics=diagnostics, tune=tune)
    done = 0
    for k in list(splits) + [steps]:
        sim.advance(k - done)
        done = k
    return sim


def test_config1_golden_run_loop():
    """BASELINE config 1 (256^2 f32, CFL 0.9 every step, 100 steps) through
    the loop: state, dt series and maxima bit-exact, mass 1e-12."""
    from paper_1107_2157_b200 import swdemo
    g = load_golden("cfg1_sw256_f32_reflective.npz")
    cfg = swdemo.SWConfig(nx=256, ny=256, steps=100, cfl_factor=0.9, precision="f32", variant="loop")
    sim = swdemo.Simulation(cfg, state=swdemo.init_state(cfg))
    sim.advance(1)
    assert all(np.array_equal(a, b) for a, b in zip(host(sim.state()), (g["H1"], g["U1"], g["V1"])))
    sim.advance(99)
    res = sim.rows()
    assert all(np.array_equal(a, b) for a, b in zip(host(res.state), (g["H100"], g["U100"], g["V100"])))
    assert np.array_equal(res.dts, g["dt"])
    rows = np.array(res.rows)
    assert np.array_equal(rows[:, 4:], g["rows"][:, 4:])
    assert np.max(np.abs(rows[:, 3] - g["rows"][:, 3]) / g["rows"][:, 3]) <= 1e-12


SHAPES = [(256, 256), (128, 40), (4, 9), (240, 3), (244, 61), (1000, 88), (96, 1), (124, 500)]


@pytest.mark.parametrize("nx,ny", SHAPES)
@pytest.mark.parametrize("bc", ["reflective", "periodic"])
@pytest.mark.parametrize("prec", ["f32", "f64"])
def test_loop_exact_fixed_dt(nx, ny, bc, prec):
    """Ragged strips (nx not a multiple of the 120-column strip), one-row and
    few-row grids, periodic wrap partners; two advance calls (the second
    starts on an odd step, reading buffer B); per-step diagnostics."""
    H, U, V = so.random_state(nx, ny, prec, seed=nx * 7 + ny, boundary=bc)
    steps = 7
    want = c_oracle.run_fixed(H, U, V, steps, 1.0, 0.8, 0.04, boundary=bc)
    sim = sim_run(H, U, V, steps, "loop", bc=bc, prec=prec, splits=(3,))
    got = host(sim.state())
    for k, (x, w) in enumerate(zip(got, want)):
        assert np.array_equal(x, w), (k, np.argwhere(x != w)[:3].tolist())
    d = sim.diagnostics()
    for i in range(1, steps + 1):
        Hs, Us, Vs = c_oracle.run_fixed(H, U, V, i, 1.0, 0.8, 0.04, boundary=bc)
        m, mu, mv = so.diagnostics(Hs, Us, Vs)
        assert d["max_hu"][i] == mu and d["max_hv"][i] == mv
        assert abs(d["mass"][i] - m) <= 1e-12 * abs(m)
        assert d["err"][i] == 0


@pytest.mark.parametrize("seg,warps", [(2, 1), (6, 0), (10, 1), (3, 1), (64, 1)])
@pytest.mark.parametrize("bc", ["reflective", "periodic"])
def test_loop_schedules_bit_identical(seg, warps, bc):
    """Results never depend on the loop's schedule (rows per segment): exact
    mode equals the oracle for every forced schedule, including odd segment
    lengths (a partial last stage)."""
    import paper_1107_2157_b200._native as N
    H, U, V = so.random_state(360, 130, "f32", seed=seg * 10 + warps, boundary=bc)
    want = c_oracle.run_fixed(H, U, V, 9, 1.0, 0.8, 0.04, boundary=bc)
    sim = sim_run(H, U, V, 9, "loop", bc=bc, tune=N.Tune(seg=seg, warps=warps), splits=(4,), diagnostics=False)
    for x, w in zip(host(sim.state()), want):
        assert np.array_equal(x, w)


@pytest.mark.parametrize("prec", ["f32", "f64"])
@pytest.mark.parametrize("bc", ["reflective", "periodic"])
def test_loop_cfl_run_matches_per_step_path(prec, bc):
    """The SPEC run (dt = cfl * the previous state's bound, on device, a
    grid-wide arrival per step): the loop equals the per-step TMA kernel bit
    for bit, dt series included, and the oracle's run."""
    from paper_1107_2157_b200 import swdemo
    H, U, V = so.init_state(240, 200, prec)
    so.apply_boundary(H, U, V, bc)
    res = {}
    for variant in ("loop", "tma"):
        cfg = swdemo.SWConfig(nx=240, ny=200, steps=40, cfl_factor=0.9, precision=prec, boundary=bc, variant=variant)
        res[variant] = swdemo.run(cfg, state=dev_state(H, U, V))
    a, b = res["loop"], res["tma"]
    assert np.array_equal(a.dts, b.dts)
    assert all(np.array_equal(x, y) for x, y in zip(host(a.state), host(b.state)))
    ref = so.run(H, U, V, 40, boundary=bc, cfl=0.9)
    assert np.array_equal(host(a.state)[0], ref.H)
    assert [r[2] for r in a.rows] == [r[2] for r in ref.rows]


@pytest.mark.parametrize("n", [512, 1024, 2048])
def test_loop_exact_mid_size_equals_per_step(n):
    """Mid sizes: 30 exact loop steps equal the per-step
    TMA path bit for bit (full arrays)."""
    H, U, V = so.random_state(n, n, "f32", seed=n + 1)
    a = sim_run(H, U, V, 30, "loop", dt=0.05, dx=1.0, dy=1.0, diagnostics=False)
    b = sim_run(H, U, V, 30, "tma", dt=0.05, dx=1.0, dy=1.0, diagnostics=False)
    for x, y in zip(host(a.state()), host(b.state())):
        assert np.array_equal(x, y)
    if n == 512:
        want = c_oracle.run_fixed(H, U, V, 30, 1.0, 1.0, 0.05)
        assert all(np.array_equal(x, w) for x, w in zip(host(a.state()), want))


@pytest.mark.parametrize("n", [256, 1024])
@pytest.mark.parametrize("bc", ["reflective", "periodic"])
def test_loop_fast_equals_per_step_fast(n, bc):
    """Fast mode: the loop's values equal the per-step fast kernel's (same
    arithmetic per cell; mirrored sweeps may flip the sign of a zero) and
    stay within the fast-mode tolerance of the oracle."""
    H, U, V = so.random_state(n, n, "f32", seed=n + 2, boundary=bc)
    a = sim_run(H, U, V, 20, "loop", dt=0.05, bc=bc, mode="fast", dx=1.0, dy=1.0, diagnostics=False,
                splits=(5,))
    b = sim_run(H, U, V, 20, "tma", dt=0.05, bc=bc, mode="fast", dx=1.0, dy=1.0, diagnostics=False)
    for x, y in zip(host(a.state()), host(b.state())):
        assert np.array_equal(x, y)
    want = c_oracle.run_fixed(H, U, V, 20, 1.0, 1.0, 0.05, boundary=bc)
    for x, w in zip(host(a.state()), want):
        assert np.max(np.abs(x.astype(np.float64) - w)) <= FAST_RTOL * np.max(np.abs(w))


def test_loop_graph_capture_and_auto_path():
    """The loop inside Simulation.capture's graph (one cooperative launch per
    replay) equals the per-step path; AUTO keeps per-step kernels here."""
    from paper_1107_2157_b200 import swdemo
    H, U, V = so.random_state(1024, 768, "f32", seed=5)
    outs = []
    for variant in ("loop", "tma", "auto"):
        cfg = swdemo.SWConfig(nx=1024, ny=768, dt=0.05, variant=variant)
        sim = swdemo.Simulation(cfg, state=dev_state(H, U, V), diagnostics=False)
        sim.advance(5)
        rep = sim.capture(6)
        rep()
        outs.append(host(sim.state()))
        assert sim.n == 19
    for o in outs[1:]:
        assert all(np.array_equal(x, y) for x, y in zip(outs[0], o))


def test_loop_errors():
    import paper_1107_2157_b200._native as N
    from paper_1107_2157_b200 import swdemo
    cfg = swdemo.SWConfig(nx=512, ny=384, steps=3, dt=0.05, variant="loop")
    st = swdemo.init_state(cfg)
    st.H.data[40, 50] = -1.0
    with pytest.raises(swdemo.NonPositiveDepth):
        swdemo.run(cfg, state=st)
    st = swdemo.init_state(cfg)
    st.U.data[10, 20] = float("nan")
    with pytest.raises((swdemo.NonfiniteValue, swdemo.NonPositiveDepth)):
        swdemo.run(cfg, state=st)
    # a schedule whose warps cannot all be resident: usage error when forced
    big = swdemo.SWConfig(nx=8192, ny=8192, steps=2, dt=0.05, variant="loop")
    sim = swdemo.Simulation(big, diagnostics=False, tune=N.Tune(seg=2))
    with pytest.raises(swdemo.LaunchError):
        sim.advance(2)
    with pytest.raises(swdemo.LaunchError):
        swdemo.Simulation(cfg, diagnostics=False, tune=N.Tune(warps=2)).advance(2)
    # not TMA-eligible (nx % 4 != 0)
    odd = swdemo.SWConfig(nx=130, ny=64, steps=2, dt=0.05, variant="loop")
    with pytest.raises(swdemo.LaunchError):
        swdemo.run(odd)
