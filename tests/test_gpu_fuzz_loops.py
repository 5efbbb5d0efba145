"""GPU tier: randomised whole-run paths of round 2 against the C oracle --
the resident cluster loop, the persistent TMA loop and the streamed host
run on random extents, boundaries, precisions, step counts, split advance
calls and dt policies (fixed / CFL).  Exact mode must be bit-identical to
the oracle's fixed-dt run (full arrays, halos included) and, for CFL runs,
to the per-step kernels (dt series included)."""

import numpy as np
import pytest

from oracle import c_oracle
from oracle import sw_oracle as so

pytestmark = pytest.mark.gpu


def dev_state(H, U, V, dx, dy):
    from paper_1107_2157_b200.field import DeviceField, Field, precision_of
    from paper_1107_2157_b200.swdemo import SWState
    p = precision_of(H.dtype)
    return SWState(*(DeviceField.from_field(Field.from_array(a, p)) for a in (H, U, V)), 9.8, dx, dy)


def host(st):
    return tuple(f.to_numpy() for f in (st.H, st.U, st.V))


@pytest.mark.parametrize("seed", list(range(16)))
def test_fuzz_round2_paths(seed):
    from paper_1107_2157_b200 import swdemo
    from paper_1107_2157_b200.field import Field
    rng = np.random.default_rng(2000 + seed)
    path = ["resident", "loop", "stream"][seed % 3]
    prec = "f32" if (path == "stream" or rng.random() < 0.7) else "f64"
    cpl = 4 if prec == "f32" else 2
    if path == "resident":
        nx = cpl * int(rng.integers(1, (224 if prec == "f32" else 120) // cpl))
        ny = int(rng.integers(1, 200))
    else:
        nx = cpl * int(rng.integers(1, 600 // cpl))
        ny = int(rng.integers(1, 700))
    bc = "reflective" if path == "stream" else ["reflective", "periodic"][int(rng.integers(2))]
    dx, dy = float(rng.choice([1.0, 0.8, 1.25])), float(rng.choice([1.0, 0.9]))
    steps = int(rng.integers(1, 9))
    split = int(rng.integers(0, steps + 1))
    cfl = path != "stream" and rng.random() < 0.4
    H, U, V = so.random_state(nx, ny, prec, seed=seed, boundary=bc)
    what = (path, prec, nx, ny, bc, steps, split, cfl)
    if path == "stream":
        st = swdemo.SWState(*(Field.from_array(a, prec) for a in (H, U, V)), 9.8, dx, dy)
        out = swdemo.SWState(*(Field.from_array(np.zeros_like(a), prec) for a in (H, U, V)), 9.8, dx, dy)
        cfg = swdemo.SWConfig(nx=nx, ny=ny, steps=steps, dt=0.03, dx=dx, dy=dy)
        swdemo._run_streamed(cfg, st, out, band_rows=int(rng.choice([16, 24, 64])))
        want = c_oracle.run_fixed(H, U, V, steps, dx, dy, 0.03)
        for g, w in zip((out.H.data, out.U.data, out.V.data), want):
            assert np.array_equal(g, w), what
        return
    res = {}
    for variant in (path, "generic"):
        cfg = swdemo.SWConfig(nx=nx, ny=ny, steps=steps, dt=None if cfl else 0.03, cfl_factor=0.8, dx=dx, dy=dy,
                              precision=prec, boundary=bc, variant=variant)
        sim = swdemo.Simulation(cfg, state=dev_state(H, U, V, dx, dy), diagnostics=True)
        if split:
            sim.advance(split)
        sim.advance(steps - split)
        res[variant] = (host(sim.state()), sim.rows())
    (a, ra), (b, rb) = res[path], res["generic"]
    assert all(np.array_equal(x, y) for x, y in zip(a, b)), what
    assert np.array_equal(ra.dts, rb.dts), what
    if not cfl:
        want = c_oracle.run_fixed(H, U, V, steps, dx, dy, 0.03, boundary=bc)
        assert all(np.array_equal(x, w) for x, w in zip(a, want)), what
