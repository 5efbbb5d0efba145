"""GPU tier: edge cases from the round-1 code review.

* one- and two-row tiles on the TMA kernel: both output halo rows are
  written every step, so multi-step runs stay bit-identical INCLUDING the
  halos (the y == 1 == ny row has two row images);
* step_native's NonPositiveDepth covers half-step FACE depths:
  a divergent momentum field between positive cells drives Hx <= 0;
* f64 fast-mode CFL with g = 0 (sqrt(g h) = 0, no NaN);
* a resumed run continues the state's clock and uses the state's spacing.
"""

import numpy as np
import pytest

from oracle import c_oracle
from oracle import sw_oracle as so

pytestmark = pytest.mark.gpu


def dev_state(H, U, V, dx=1.0, dy=1.0, g=9.8):
    from paper_1107_2157_b200.field import DeviceField, Field, precision_of
    from paper_1107_2157_b200.swdemo import SWState
    p = precision_of(H.dtype)
    return SWState(*(DeviceField.from_field(Field.from_array(a, p)) for a in (H, U, V)), g, dx, dy)


def host(st):
    return tuple(f.to_numpy() for f in (st.H, st.U, st.V))


@pytest.mark.parametrize("ny", [1, 2, 3])
@pytest.mark.parametrize("bc", ["reflective", "periodic"])
@pytest.mark.parametrize("prec", ["f32", "f64"])
@pytest.mark.parametrize("mode", ["exact", "fast"])
def test_thin_tiles_multistep_full_arrays(ny, bc, prec, mode):
    """Full arrays (halos and corners included) after 5 steps of the TMA
    kernel on 1..3-row grids: the time loop never re-applies BCs, so a stale
    halo row would show up from step 2 on."""
    from paper_1107_2157_b200 import swdemo
    nx = 256
    H, U, V = so.random_state(nx, ny, prec, seed=31 + ny, boundary=bc)
    want = c_oracle.run_fixed(H, U, V, 5, 1.0, 1.0, 0.02, boundary=bc)
    cfg = swdemo.SWConfig(nx=nx, ny=ny, steps=5, dt=0.02, precision=prec, mode=mode, variant="tma",
                          boundary=bc)
    sim = swdemo.Simulation(cfg, state=dev_state(H, U, V), diagnostics=False)
    sim.advance(5)
    got = host(sim.state())
    for k, (x, w) in enumerate(zip(got, want)):
        if mode == "exact":
            assert np.array_equal(x, w), (k, np.argwhere(x != w)[:3])
        else:
            sc = max(float(np.max(np.abs(w))), 1e-30)
            assert np.max(np.abs(x.astype(np.float64) - w)) <= 2e-5 * sc, k


def _divergent_state(nx, ny, prec="f32"):
    """h = 1 everywhere, hu jumps from -40 to +40 across one column pair in
    the middle: with dt = 0.05 the x-face between them has
    Hx = 1 - 0.025 * 80 = -1 < 0 while every cell depth is positive."""
    H, U, V = so.random_state(nx, ny, prec, seed=3)
    H[...] = 1.0
    U[...] = 0.0
    V[...] = 0.0
    c = nx // 2
    U[1:-1, c] = -40.0
    U[1:-1, c + 1] = 40.0
    so.apply_boundary(H, U, V, "reflective")
    return H, U, V


@pytest.mark.parametrize("variant", ["tma", "generic"])
@pytest.mark.parametrize("mode", ["exact", "fast"])
def test_step_native_face_depth(variant, mode):
    from paper_1107_2157_b200 import swdemo
    H, U, V = _divergent_state(512, 64)
    with pytest.raises(so.NonPositiveDepth):
        so.step_native(1.0, 1.0, 0.05, H, U, V)
    with pytest.raises(swdemo.NonPositiveDepth):
        swdemo.advance(dev_state(H, U, V), 0.05, "reflective", mode, variant, check=True)
    # step_native raises on its own; a benign dt passes
    with pytest.raises(swdemo.NonPositiveDepth):
        swdemo.step_native(dev_state(H, U, V), 0.05)
    swdemo.advance(dev_state(H, U, V), 0.001, "reflective", mode, variant, check=True)
    # an input cell depth <= 0 is caught too
    H2 = H.copy()
    H2[10, 7] = -1.0
    with pytest.raises(swdemo.NonPositiveDepth):
        swdemo.advance(dev_state(H2, U * 0, V), 0.001, "reflective", mode, variant, check=True)


@pytest.mark.parametrize("mode", ["exact", "fast"])
def test_run_reports_face_depth(mode):
    """run() (fused reductions) raises NonPositiveDepth for a negative face
    depth between positive cells, on the TMA path (>= 640 Ki cells)."""
    from paper_1107_2157_b200 import swdemo
    H, U, V = _divergent_state(1024, 1024)
    cfg = swdemo.SWConfig(nx=1024, ny=1024, steps=2, dt=0.05, mode=mode)
    with pytest.raises(swdemo.NonPositiveDepth):
        swdemo.run(cfg, state=dev_state(H, U, V))


def test_f64_fast_cfl_zero_gravity():
    """g = 0: sqrt(g h) = 0, the fast f64 CFL bound stays finite and close
    to the oracle's (it used to be NaN -> dropped -> dt = inf)."""
    from paper_1107_2157_b200 import swdemo
    H, U, V = so.random_state(1024, 768, "f64", seed=8)
    # pure advection (g = 0) of rough random data: keep the steps short
    cfg = swdemo.SWConfig(nx=1024, ny=768, steps=3, cfl_factor=0.02, precision="f64", mode="fast",
                          variant="tma", g=0.0)
    res = swdemo.run(cfg, state=dev_state(H, U, V, g=0.0))
    assert np.all(np.isfinite(res.dts)) and np.all(res.dts > 0)
    want0 = so.stable_dt(H, U, V, 1.0, 1.0, 0.02, g=0.0)
    assert res.dts[0] == want0                       # initial reduction: exact kernel
    H1, U1, V1 = so.step(H, U, V, 1.0, 1.0, want0, g=0.0)
    want1 = so.stable_dt(H1, U1, V1, 1.0, 1.0, 0.02, g=0.0)
    assert abs(res.dts[1] - want1) <= 1e-5 * want1   # fused fast-mode bound of step 1's state


def test_resumed_run_keeps_clock_and_spacing():
    from paper_1107_2157_b200 import swdemo
    cfg = swdemo.SWConfig(nx=128, ny=96, steps=4, cfl_factor=0.8, precision="f64")
    first = swdemo.run(cfg)
    st = first.state
    t_end = first.rows[-1][1]
    assert st.t == pytest.approx(t_end)
    second = swdemo.run(cfg, state=st)
    assert second.rows[0][1] == pytest.approx(t_end + second.rows[0][2], rel=1e-15)
    assert second.rows[-1][1] > t_end
    # the state's own spacing sets the mass (and the steps): dx = dy = 0.5
    H, U, V = so.init_state(128, 96, "f64")
    st2 = dev_state(H, U, V, dx=0.5, dy=0.5)
    res = swdemo.run(cfg, state=st2)
    m0 = so.total_mass(H, 0.5, 0.5)
    assert abs(res.rows[-1][3] - m0) <= 1e-12 * m0
