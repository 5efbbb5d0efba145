"""Field CSV I/O, run config, and the cli entry points run / compare / bench
(SPEC.md:564, :571-643).  CPU tier: formats and compare exit codes; GPU
tier: cmd_run / cmd_bench on the device against the oracle."""

import os

import numpy as np
import pytest

from oracle import sw_oracle as so
from paper_1107_2157_b200 import cli, fieldio
from paper_1107_2157_b200.field import Field
from paper_1107_2157_b200.region import Halo


def _write_run(d, H, U, V, prec, diag=None):
    os.makedirs(d, exist_ok=True)
    p = fieldio.state_paths(d)
    for name, a in zip("HUV", (H, U, V)):
        fieldio.write_field_csv(p[name], Field.from_array(a, prec))
    if diag is not None:
        fieldio.write_diagnostics_csv(p["diag"], diag)


@pytest.mark.parametrize("prec", ["f32", "f64"])
def test_field_csv_roundtrip_bit_exact(tmp_path, prec):
    rng = np.random.default_rng(3)
    dt = np.float32 if prec == "f32" else np.float64
    a = (rng.standard_normal((9, 13)) * np.exp2(rng.integers(-140, 120, (9, 13)))).astype(dt)
    a[0, 0], a[0, 1], a[0, 2] = -0.0, np.finfo(dt).tiny / 8, np.finfo(dt).max
    fn = str(tmp_path / "f.csv")
    fieldio.write_field_csv(fn, Field.from_array(a, prec), Halo(1, 2, 0, 3))
    head = open(fn).readline()
    assert head == f"# 13 9 1 2 0 3 {prec}\n"
    f, h = fieldio.read_field_csv(fn)
    assert h == Halo(1, 2, 0, 3) and f.precision == prec and f.full == (13, 9)
    assert f.data.tobytes() == a.tobytes()


def test_field_csv_errors(tmp_path):
    fn = str(tmp_path / "bad.csv")
    open(fn, "w").write("1,2\n3,4\n")
    with pytest.raises(fieldio.FieldFormatError):
        fieldio.read_field_csv(fn)
    open(fn, "w").write("# 2 3 1 1 1 1 f32\n1,2\n3,4\n")
    with pytest.raises(fieldio.FieldFormatError):
        fieldio.read_field_csv(fn)


def test_config_parse_and_roundtrip(tmp_path):
    from paper_1107_2157_b200.swdemo import SWConfig
    kw = fieldio.parse_config_text("# demo\ninterior = 64x32\ncfl_factor = 0.9\nsteps = 10\n"
                                   "boundary = periodic\nprecision = f64\ngroup = 16x8\ncenter = 3.5,4\n")
    assert kw == {"nx": 64, "ny": 32, "cfl_factor": 0.9, "steps": 10, "boundary": "periodic",
                  "precision": "f64", "group": (16, 8), "center": (3.5, 4.0)}
    with pytest.raises(ValueError):
        fieldio.parse_config_text("bogus = 1\n")
    with pytest.raises(ValueError):
        fieldio.parse_config_text("steps = 1\nsteps = 2\n")
    cfg = SWConfig(nx=40, ny=24, steps=7, dt=0.01, boundary="periodic", width=3.0)
    fn = str(tmp_path / "c.cfg")
    fieldio.write_config(fn, cfg)
    assert fieldio.read_config(fn) == cfg


def test_compare_exit_codes(tmp_path, capsys):
    H, U, V = so.random_state(24, 16, "f64", seed=9)
    a, b, c = (str(tmp_path / n) for n in "abc")
    diag = [(1, 0.1, 0.1, 384.0, 0.05, 0.04)]
    _write_run(a, H, U, V, "f64", diag)
    _write_run(b, H, U, V, "f64", diag)
    assert cli.main(["compare", a, b]) == 0                      # reflexive, rtol 0
    H2 = H.copy()
    H2[5, 7] *= 1 + 1e-3
    _write_run(c, H2, U, V, "f64", diag)
    assert cli.main(["compare", a, c, "--rtol", "1e-6"]) == 1
    out = capsys.readouterr().out
    assert "in H at (x, y) = (7, 5)" in out
    assert cli.main(["compare", a, c, "--rtol", "1e-2"]) == 0
    assert cli.main(["compare", a, c, "--rtol", "1e-6", "--floor", "0"]) == 1
    # a tiny value next to 0: 100 % elementwise, negligible normwise
    U1 = U.copy()
    U1[4, 4] = 1e-12
    U2 = U.copy()
    U2[4, 4] = 0.0
    _write_run(a, H, U1, V, "f64", diag)
    _write_run(c, H, U2, V, "f64", diag)
    assert cli.main(["compare", a, c, "--rtol", "1e-6"]) == 0
    assert cli.main(["compare", a, c, "--rtol", "1e-6", "--floor", "0"]) == 1
    d = str(tmp_path / "d")
    Hs, Us, Vs = so.random_state(20, 16, "f64", seed=9)
    _write_run(d, Hs, Us, Vs, "f64")
    assert cli.main(["compare", a, d]) == 2                      # shape mismatch
    assert cli.main(["compare", a, str(tmp_path / "missing")]) == 2


def test_usage_exit_codes(tmp_path):
    assert cli.main(["check", "x.fk"]) == 2                      # DSL compiler: reference package
    assert cli.main(["emit", "x.fk"]) == 2
    cfgf = str(tmp_path / "c.cfg")
    open(cfgf, "w").write("interior = 16x16\nsteps = 1\n")
    assert cli.main(["run", cfgf, "--engine", "sim", "-o", str(tmp_path / "o")]) == 2
    open(cfgf, "w").write("nonsense\n")
    assert cli.main(["run", cfgf, "-o", str(tmp_path / "o")]) == 2
    with pytest.raises(SystemExit) as e:
        cli.main(["frobnicate"])
    assert e.value.code == 2


@pytest.mark.gpu
def test_cmd_run_steps0_is_initial_state(tmp_path):
    cfgf = str(tmp_path / "c.cfg")
    open(cfgf, "w").write("interior = 48x40\nsteps = 0\nprecision = f32\n")
    out = str(tmp_path / "o")
    assert cli.main(["run", cfgf, "-o", out]) == 0
    H0, U0, V0 = so.init_state(48, 40, "f32")
    ref = str(tmp_path / "ref")
    _write_run(ref, H0, U0, V0, "f32")
    assert cli.main(["compare", out, ref]) == 0
    assert fieldio.read_diagnostics_csv(fieldio.state_paths(out)["diag"]).shape == (0, 6)


@pytest.mark.gpu
def test_cmd_run_matches_oracle_bit_exact(tmp_path):
    """BASELINE config 1 through the CLI: CFL 0.9 recomputed every step,
    reflective, 100 steps, f32 exact == the oracle's run, rtol 0."""
    cfgf = str(tmp_path / "c.cfg")
    open(cfgf, "w").write("interior = 256x256\nsteps = 100\ncfl_factor = 0.9\nprecision = f32\n"
                          "boundary = reflective\nmode = exact\n")
    out = str(tmp_path / "o")
    assert cli.main(["run", cfgf, "-o", out]) == 0
    H0, U0, V0 = so.init_state(256, 256, "f32")
    r = so.run(H0, U0, V0, 100, cfl=0.9)
    ref = str(tmp_path / "ref")
    _write_run(ref, r.H, r.U, r.V, "f32")
    assert cli.main(["compare", out, ref]) == 0
    d = fieldio.read_diagnostics_csv(fieldio.state_paths(out)["diag"])
    assert d.shape == (100, 6) and np.all(np.isfinite(d))
    assert np.array_equal(d[:, 2], np.array([row[2] for row in r.rows], np.float64))   # dt series


@pytest.mark.gpu
def test_cmd_compare_f32_vs_f64(tmp_path):
    """SPEC.md:618 example: f32 vs f64 runs, rtol 1e-4, 10 steps, 64x64 -> 0."""
    cfgf = str(tmp_path / "c.cfg")
    open(cfgf, "w").write("interior = 64x64\nsteps = 10\ncfl_factor = 0.9\n")
    a, b = str(tmp_path / "a"), str(tmp_path / "b")
    assert cli.main(["run", cfgf, "--precision", "f32", "-o", a]) == 0
    assert cli.main(["run", cfgf, "--precision", "f64", "-o", b]) == 0
    assert cli.main(["compare", a, b, "--rtol", "1e-4"]) == 0


@pytest.mark.gpu
def test_cmd_bench_rows(tmp_path, capsys):
    cfgf = str(tmp_path / "c.cfg")
    open(cfgf, "w").write("interior = 16x16\nsteps = 5\n")
    assert cli.main(["bench", cfgf, "--sizes", "16,32,64"]) == 0
    rows = [l for l in capsys.readouterr().out.splitlines() if l and not l.startswith("engine")]
    assert len(rows) == 6
    for r in rows:
        e, w, k, ms, g = r.split(",")
        assert float(ms) > 0 and np.isfinite(float(ms)) and float(g) > 0


def test_checkpoint_npz_roundtrip(tmp_path):
    from paper_1107_2157_b200 import swdemo
    H, U, V = so.random_state(20, 12, "f32", seed=8)
    st = swdemo.SWState(*(Field.from_array(a, "f32") for a in (H, U, V)), 9.81, 0.5, 0.25, 3.5)
    rows = [(1, 0.1, 0.1, 12.0, 0.01, 0.02), (2, 0.2, 0.1, 12.0, 0.011, 0.021)]
    fn = str(tmp_path / "ck.npz")
    fieldio.save_state_npz(fn, st, rows)
    back, r = fieldio.load_state_npz(fn)
    assert (back.g, back.dx, back.dy, back.t) == (9.81, 0.5, 0.25, 3.5)
    for a, b in zip((back.H, back.U, back.V), (H, U, V)):
        assert a.precision == "f32" and a.data.tobytes() == b.tobytes()
    assert np.array_equal(r, np.array(rows))
