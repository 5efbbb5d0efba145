"""CPU tier: pin the oracle (test infrastructure) against the golden vectors
generated from the reference's own parser/sema (oracle/gen_golden.py), the
SPEC known answers and the C restatement."""

import math

import numpy as np
import pytest

from conftest import load_golden
from oracle import c_oracle, dsl_eval
from oracle import sw_oracle as so


def _eq(a, b):
    return all(np.array_equal(x, y) for x, y in zip(a, b))


@pytest.mark.parametrize("prec", ["f32", "f64"])
@pytest.mark.parametrize("bc", ["reflective", "periodic"])
def test_golden_random(prec, bc):
    g = load_golden(f"rand_{prec}_{bc}.npz")
    st = (g["H0"], g["U0"], g["V0"])
    for k in range(10):
        st = so.step(*st, 1.0, 0.7, 0.1, boundary=bc)
        if k == 0:
            assert _eq(st, (g["H1"], g["U1"], g["V1"]))
    assert _eq(st, (g["H10"], g["U10"], g["V10"]))


def test_golden_config1():
    g = load_golden("cfg1_sw256_f32_reflective.npz")
    H, U, V = so.init_state(256, 256, "f32")
    assert _eq((H, U, V), (g["H0"], g["U0"], g["V0"]))
    r = so.run(H, U, V, 100, cfl=0.9)
    assert _eq((r.H, r.U, r.V), (g["H100"], g["U100"], g["V100"]))
    assert np.array_equal(np.array([row[2] for row in r.rows]), g["dt"])
    assert np.allclose(np.array(r.rows), g["rows"], rtol=0, atol=0)


def test_hand_oracle_4x4_periodic():
    g = load_golden("hand4_periodic_f64.npz")
    got = so.wave_advance(1.0, 1.0, float(g["dt"]), g["H0"], g["U0"], g["V0"])
    for a, b in zip(got, g["out"]):
        assert np.max(np.abs(a - b)) <= 1e-12


@pytest.mark.parametrize("prec", ["f32", "f64"])
@pytest.mark.parametrize("bc", ["reflective", "periodic"])
def test_c_oracle_bit_identical(prec, bc):
    H, U, V = so.random_state(61, 37, prec, seed=7, boundary=bc)
    a = so.step(H, U, V, 0.9, 1.3, 0.05, boundary=bc)
    b = c_oracle.step(H, U, V, 0.9, 1.3, 0.05, boundary=bc, threads=4)
    assert _eq(a, b)


def test_step_native_matches_dsl_order():
    # SPEC.md:549 three-way agreement <= 1e-12 (here: formula form vs DSL form)
    for prec in ("f32", "f64"):
        H, U, V = so.random_state(40, 30, prec, seed=3)
        a = so.wave_advance(1.0, 1.0, 0.1, H, U, V)
        b = so.step_native(1.0, 1.0, 0.1, H, U, V)
        for x, y in zip(a, b):
            assert np.max(np.abs(x.astype(np.float64) - y)) <= 1e-12 * max(1.0, np.max(np.abs(y)))


def test_stable_dt_known_answer():
    # SPEC.md:514, :651
    one = np.ones((6, 6))
    z = np.zeros((6, 6))
    assert abs(so.stable_dt(one, z, z, 1.0, 1.0) - 1.0 / math.sqrt(9.8)) <= 1e-15
    # doubling dx and dy doubles dt
    assert abs(so.stable_dt(one, z, z, 2.0, 2.0) - 2.0 / math.sqrt(9.8)) <= 1e-15


@pytest.mark.parametrize("bc", ["reflective", "periodic"])
def test_lake_at_rest(bc):
    # SPEC.md:496, :507, :526, :650
    H, U, V = so.init_state(32, 24, "f64", amplitude=0.0, boundary=bc)
    out = so.step(H, U, V, 1.0, 1.0, 0.1, boundary=bc)
    assert np.max(np.abs(out[0] - H)) <= 1e-14
    assert np.max(np.abs(out[1])) <= 1e-14 and np.max(np.abs(out[2])) <= 1e-14


def test_mass_conservation_periodic():
    # SPEC.md:537, :550, :649
    H, U, V = so.init_state(64, 64, "f64", boundary="periodic")
    m0 = so.total_mass(H)
    r = so.run(H, U, V, 100, boundary="periodic", cfl=0.9)
    assert abs(r.rows[-1][3] - m0) / m0 <= 1e-12


def test_symmetry():
    # SPEC.md:527, :552
    H, U, V = so.init_state(48, 48, "f64", boundary="periodic")
    a = so.step(H, U, V, 1.0, 1.0, 0.1, boundary="periodic")
    assert np.max(np.abs(a[0] - a[0].T)) <= 1e-13
    assert np.max(np.abs(a[1] - a[2].T)) <= 1e-13


def test_cfl_safety():
    # SPEC.md:553
    H, U, V = so.init_state(64, 64, "f64")
    r = so.run(H, U, V, 100, cfl=0.9)
    assert np.max(np.abs(r.H[1:-1, 1:-1] - 1.0)) < 10 * 0.4


def test_init_and_mass_known_answers():
    # SPEC.md:497 (peak 1.4 when centre is a cell centre), :544 (mass 64)
    H, _, _ = so.init_state(64, 64, "f64", center=(32.5, 32.5))
    assert abs(np.max(H) - 1.4) <= 1e-15
    assert so.total_mass(np.ones((10, 10))) == 64.0


def test_boundary_known_answers():
    H, U, V = so.random_state(4, 4, "f64", boundary="periodic")
    assert np.array_equal(H[1:-1, 0], H[1:-1, 4])
    H, U, V = so.random_state(5, 4, "f64", boundary="reflective")
    assert np.array_equal(U[1:-1, 0], -U[1:-1, 1])
    assert np.array_equal(V[0, 1:-1], -V[1, 1:-1])


def test_region_cpy_examples():
    # SPEC.md:295-297
    a = np.array([[1.0, 2, 3, 4, 5]])
    assert np.array_equal(so.region_cpy(a, (1, 1, 0, 0)), [[2.0, 3, 4]])
    assert np.array_equal(so.region_cpy(a, (0, 0, 0, 0)), a)
    f = np.fromfunction(lambda y, x: 10 * y + x, (5, 6))
    r = so.region_cpy(f, (0, 1, 1, 1))
    assert r.shape == (3, 5) and r[0, 0] == 10


def test_cshift_examples():
    # SPEC.md:303-305 and the section 2.1 duality
    a = np.array([[1.0, 2, 3, 4]])
    assert np.array_equal(so.cshift(a, 1, 1), [[2.0, 3, 4, 1]])
    assert np.array_equal(so.cshift(a, 1, 0), a)
    assert np.array_equal(so.cshift(a, 1, 4), a)
    x = np.array([[5.0, 1, 2, 3, 4, 5, 1]])      # periodic halo pre-filled
    reg = (so.region(x, (0, 2, 0, 0)) + so.region(x, (1, 1, 0, 0)) + so.region(x, (2, 0, 0, 0))) / 3
    core = x[:, 1:-1]
    cs = (so.cshift(core, 1, -1) + core + so.cshift(core, 1, 1)) / 3
    assert np.array_equal(reg, cs)


@pytest.mark.skipif(not dsl_eval.reference_available(), reason="reference not mounted")
def test_fk_passes_reference_sema():
    import os
    frontend, sema, _, _ = dsl_eval._import_fkc()
    src = open(os.path.join(os.path.dirname(__file__), "..", "kernels", "wave_advance.fk")).read()
    ks, els = frontend.parse_source(src)
    assert len(ks) == 1 and len(els) == 2 and len(ks[0].body) == 21
    assert sema.collect_diagnostics(ks[0]) == []


@pytest.mark.skipif(not dsl_eval.reference_available(), reason="reference not mounted")
@pytest.mark.parametrize("prec", ["f32", "f64"])
def test_numpy_oracle_equals_ast_evaluator(prec):
    import os
    cp = dsl_eval.load_checked(os.path.join(os.path.dirname(__file__), "..", "kernels", "wave_advance.fk"))
    H, U, V = so.random_state(23, 17, prec, seed=11)
    outs = dsl_eval.eval_kernel(cp, {"h": H, "u": U, "v": V}, {"dx": 0.8, "dy": 1.1, "dt": 0.07}, H.dtype)
    ref = so.wave_advance(0.8, 1.1, 0.07, H, U, V)
    for k, b in zip(("oh", "ou", "ov"), ref):
        assert np.array_equal(outs[k][1:-1, 1:-1], b)


@pytest.mark.parametrize("bc", ["reflective", "periodic"])
def test_golden_spec64_f64(bc):
    """SPEC.md's f64 acceptance setting (64x64, CFL 0.9, 100 steps): the
    oracle's run reproduces the fixture made with the reference parser/sema,
    and mass is conserved to 1e-12."""
    from conftest import load_golden
    g = load_golden(f"spec64_f64_{bc}.npz")
    r = so.run(g["H0"], g["U0"], g["V0"], 100, cfl=0.9, boundary=bc)
    assert np.array_equal(r.H, g["H100"]) and np.array_equal(r.U, g["U100"]) and np.array_equal(r.V, g["V100"])
    assert np.array_equal(np.array([row[2] for row in r.rows]), g["dt"])
    m = g["rows"][:, 3]
    assert abs(m[-1] - so.total_mass(g["H0"])) / m[-1] <= 1e-12
