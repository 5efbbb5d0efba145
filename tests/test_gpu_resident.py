"""GPU tier: the resident time loop (csrc/sw_resident.cuh) -- a small grid's
whole run in one thread-block-cluster launch with the state in shared
memory.  Exact mode must be bit-identical to the oracle (state, dt series,
maxima; mass within 1e-12), fast mode within its tolerance; reductions,
errors and the double-buffer contract of fkc_sw_advance_n as for the per-
step kernels."""

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


def test_config1_golden_run_resident():
    """BASELINE config 1 (256^2 f32, CFL 0.9 every step, 100 steps) through
    the resident loop: state, dt series and maxima bit-exact, mass 1e-12."""
    from paper_1107_2157_b200 import swdemo
    g = load_golden("cfg1_sw256_f32_reflective.npz")
    cfg = swdemo.SWConfig(nx=256, ny=256, steps=100, cfl_factor=0.9, precision="f32", variant="resident")
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


@pytest.mark.parametrize("nx,ny", [(128, 128), (64, 200), (36, 53), (4, 5), (300, 7), (200, 17), (124, 1), (240, 31)])
@pytest.mark.parametrize("bc", ["reflective", "periodic"])
@pytest.mark.parametrize("prec", ["f32", "f64"])
def test_resident_exact_fixed_dt(nx, ny, bc, prec):
    from paper_1107_2157_b200 import swdemo
    H, U, V = so.random_state(nx, ny, prec, seed=nx * 7 + ny, boundary=bc)
    steps = 7
    want = c_oracle.run_fixed(H, U, V, steps, 1.0, 0.8, 0.04, boundary=bc)
    cfg = swdemo.SWConfig(nx=nx, ny=ny, steps=steps, dt=0.04, precision=prec, boundary=bc, variant="resident")
    sim = swdemo.Simulation(cfg, state=dev_state(H, U, V, 1.0, 0.8), diagnostics=True)
    sim.advance(3)
    sim.advance(4)                   # second call: odd first step (reads buffer B)
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


@pytest.mark.parametrize("prec", ["f32", "f64"])
@pytest.mark.parametrize("bc", ["reflective", "periodic"])
def test_resident_cfl_run_matches_per_step_path(prec, bc):
    """The SPEC run (CFL dt from the previous step's bound, on device): the
    resident loop equals the per-step generic kernel bit for bit, dt series
    included, and the oracle's run."""
    from paper_1107_2157_b200 import swdemo
    H, U, V = so.init_state(96, 80, prec)
    so.apply_boundary(H, U, V, bc)
    res = {}
    for variant in ("resident", "generic"):
        cfg = swdemo.SWConfig(nx=96, ny=80, steps=40, cfl_factor=0.9, precision=prec, boundary=bc, variant=variant)
        res[variant] = swdemo.run(cfg, state=dev_state(H, U, V))
    a, b = res["resident"], res["generic"]
    assert np.array_equal(a.dts, b.dts)
    assert all(np.array_equal(x, y) for x, y in zip(host(a.state), host(b.state)))
    ref = so.run(H, U, V, 40, boundary=bc, cfl=0.9)
    assert np.array_equal(host(a.state)[0], ref.H)
    assert [r[2] for r in a.rows] == [r[2] for r in ref.rows]


@pytest.mark.parametrize("n", [128, 256])
def test_resident_fast_within_tolerance(n):
    from paper_1107_2157_b200 import swdemo
    H, U, V = so.random_state(n, n, "f32", seed=n)
    want = c_oracle.run_fixed(H, U, V, 20, 1.0, 1.0, 0.05)
    cfg = swdemo.SWConfig(nx=n, ny=n, steps=20, dt=0.05, mode="fast", variant="resident")
    sim = swdemo.Simulation(cfg, state=dev_state(H, U, V), diagnostics=False)
    sim.advance(20)
    for x, w in zip(host(sim.state()), want):
        assert np.max(np.abs(x.astype(np.float64) - w)) <= FAST_RTOL * np.max(np.abs(w))


def test_auto_picks_resident_for_small_grids_and_graph_replay():
    """AUTO runs small grids' loops resident (one launch for the whole loop,
    eager or inside Simulation.capture's graph) -- the results equal the
    per-step path's -- and graph replays keep advancing the state."""
    from paper_1107_2157_b200 import swdemo
    H, U, V = so.random_state(128, 128, "f32", seed=3)
    outs = []
    for variant in ("auto", "generic", "resident"):
        cfg = swdemo.SWConfig(nx=128, ny=128, dt=0.05, variant=variant, mode="fast")
        sim = swdemo.Simulation(cfg, state=dev_state(H, U, V), diagnostics=False)
        sim.advance(7)
        rep = sim.capture(10)
        rep()
        outs.append(host(sim.state()))
        assert sim.n == 29
    want = c_oracle.run_fixed(H, U, V, 29, 1.0, 1.0, 0.05)
    for o in outs:
        for x, w in zip(o, want):
            assert np.max(np.abs(x.astype(np.float64) - w)) <= FAST_RTOL * np.max(np.abs(w))
    outs = []
    for variant in ("auto", "generic"):
        cfg = swdemo.SWConfig(nx=64, ny=64, dt=0.05, variant=variant)
        sim = swdemo.Simulation(cfg, state=dev_state(H[:66, :66].copy(), U[:66, :66].copy(), V[:66, :66].copy()),
                                diagnostics=False)
        sim.advance(9)
        outs.append(host(sim.state()))
    assert all(np.array_equal(x, y) for x, y in zip(*outs))


def test_resident_errors():
    from paper_1107_2157_b200 import swdemo
    cfg = swdemo.SWConfig(nx=128, ny=96, steps=3, dt=0.05, variant="resident")
    st = swdemo.init_state(cfg)
    st.H.data[40, 50] = -1.0
    with pytest.raises(swdemo.NonPositiveDepth):
        swdemo.run(cfg, state=st)
    st = swdemo.init_state(cfg)
    st.U.data[10, 20] = float("nan")
    with pytest.raises((swdemo.NonfiniteValue, swdemo.NonPositiveDepth)):
        swdemo.run(cfg, state=st)
    # a grid that does not fit one cluster's shared memory: usage error when forced
    big = swdemo.SWConfig(nx=2048, ny=2048, steps=2, dt=0.05, variant="resident")
    with pytest.raises(swdemo.LaunchError):
        swdemo.run(big)
    # the row engines' lane vectors: nx a multiple of 4 (f32) / 2 (f64)
    odd = swdemo.SWConfig(nx=37, ny=40, steps=2, dt=0.05, variant="resident")
    with pytest.raises(swdemo.LaunchError):
        swdemo.run(odd)


@pytest.mark.parametrize("n,prec", [(256, "f32"), (352, "f32"), (160, "f64")])
@pytest.mark.parametrize("mode", ["exact", "fast"])
def test_resident_largest_grids(n, prec, mode):
    """The largest grids one cluster holds (256^2 - 352^2 f32, 160^2 f64):
    exact bit-identical to the oracle, fast within tolerance, 12 steps."""
    from paper_1107_2157_b200 import swdemo
    H, U, V = so.random_state(n, n, prec, seed=n + 11)
    want = c_oracle.run_fixed(H, U, V, 12, 1.0, 1.0, 0.05)
    cfg = swdemo.SWConfig(nx=n, ny=n, steps=12, dt=0.05, mode=mode, precision=prec, variant="resident")
    sim = swdemo.Simulation(cfg, state=dev_state(H, U, V), diagnostics=False)
    sim.advance(12)
    for x, w in zip(host(sim.state()), want):
        if mode == "exact":
            assert np.array_equal(x, w)
        else:
            assert np.max(np.abs(x.astype(np.float64) - w)) <= FAST_RTOL * np.max(np.abs(w))


def test_auto_falls_back_for_unaligned_width():
    """AUTO runs a small grid whose width the row engines cannot take
    (nx % 4 != 0) on the per-step generic kernel -- same bits."""
    from paper_1107_2157_b200 import swdemo
    H, U, V = so.random_state(37, 29, "f32", seed=2)
    want = c_oracle.run_fixed(H, U, V, 5, 1.0, 1.0, 0.05)
    cfg = swdemo.SWConfig(nx=37, ny=29, steps=5, dt=0.05)
    sim = swdemo.Simulation(cfg, state=dev_state(H, U, V), diagnostics=False)
    sim.advance(5)
    assert all(np.array_equal(x, w) for x, w in zip(host(sim.state()), want))
