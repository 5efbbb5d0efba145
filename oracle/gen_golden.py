"""Generate the golden fixtures under tests/golden/ -- TEST INFRASTRUCTURE.

Runs in the build container only (it imports the reference parser/sema from
/root/reference/pkg/src through ``oracle/dsl_eval.py``).  Every fixture is
produced by the AST-walking evaluator over the reference's own
CheckedProgram of ``kernels/wave_advance.fk`` ("Oracle B"),
after checking bit-for-bit that the hand-written numpy oracle
``oracle/sw_oracle.py`` agrees with it on the same inputs.

Fixtures (npz, full (ny+2, nx+2) arrays incl. halos):
* ``cfg1_sw256_f32_reflective.npz`` -- BASELINE config 1: 256x256 f32,
  Gaussian hump (base 1, amp 0.4, centre n/2, width n/8), reflective,
  dt recomputed every step with cfl 0.9,
  100 steps: state after step 1 and step 100, dt series, diagnostics rows.
* ``rand_{f32,f64}_{reflective,periodic}.npz`` -- seeded random state
  (rng 1107) 64x48 (nx != ny), dx=1, dy=0.7, fixed dt 0.1: inputs, after
  1 and 10 steps.
* ``hand4_periodic_f64.npz`` -- SPEC.md:528's "4x4 periodic hand oracle":
  a pure-Python scalar evaluation of SPEC.md:521-522 on a 4x4 grid.

* ``spec64_f64_{reflective,periodic}.npz`` -- SPEC.md's f64 acceptance
  setting: 64x64 f64, CFL 0.9 recomputed every step, 100 steps.

Usage:  python oracle/gen_golden.py [spec64]   (writes tests/golden/*.npz)
"""

from __future__ import annotations

import math
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
sys.path.insert(0, ROOT)

from oracle import dsl_eval, sw_oracle as so  # noqa: E402

OUT = os.path.join(ROOT, "tests", "golden")
FK = os.path.join(ROOT, "kernels", "wave_advance.fk")


def dsl_step(cp, H, U, V, dx, dy, dt, boundary):
    outs = dsl_eval.eval_kernel(cp, {"h": H, "u": U, "v": V},
                                {"dx": dx, "dy": dy, "dt": dt}, H.dtype)
    oH, oU, oV = outs["oh"], outs["ou"], outs["ov"]
    # cross-check the hand-written restatement bit-for-bit
    ref = so.wave_advance(dx, dy, dt, H, U, V)
    for a, b in zip((oH, oU, oV), ref):
        assert np.array_equal(a[1:-1, 1:-1], b), "numpy oracle != AST evaluator"
    so.apply_boundary(oH, oU, oV, boundary)
    return oH, oU, oV


def hand_step(H, U, V, dx, dy, dt, g=9.8):
    """Spreadsheet-style scalar loops over SPEC.md:521-522 (f64 floats)."""
    ny, nx = len(H) - 2, len(H[0]) - 2
    h = lambda y, x: float(H[y][x])  # noqa: E731
    u = lambda y, x: float(U[y][x])  # noqa: E731
    v = lambda y, x: float(V[y][x])  # noqa: E731
    Fx = {}
    for y in range(1, ny + 1):
        for x in range(0, nx + 1):
            hL, hR, uL, uR, vL, vR = h(y, x), h(y, x + 1), u(y, x), u(y, x + 1), v(y, x), v(y, x + 1)
            Hx = 0.5 * (hL + hR) - dt / (2 * dx) * (uR - uL)
            Ux = 0.5 * (uL + uR) - dt / (2 * dx) * ((uR ** 2 / hR + 0.5 * g * hR ** 2) - (uL ** 2 / hL + 0.5 * g * hL ** 2))
            Vx = 0.5 * (vL + vR) - dt / (2 * dx) * (uR * vR / hR - uL * vL / hL)
            Fx[y, x] = (Ux, Ux ** 2 / Hx + 0.5 * g * Hx ** 2, Ux * Vx / Hx)
    Fy = {}
    for y in range(0, ny + 1):
        for x in range(1, nx + 1):
            hD, hU, uD, uU, vD, vU = h(y, x), h(y + 1, x), u(y, x), u(y + 1, x), v(y, x), v(y + 1, x)
            Hy = 0.5 * (hD + hU) - dt / (2 * dy) * (vU - vD)
            Uy = 0.5 * (uD + uU) - dt / (2 * dy) * (uU * vU / hU - uD * vD / hD)
            Vy = 0.5 * (vD + vU) - dt / (2 * dy) * ((vU ** 2 / hU + 0.5 * g * hU ** 2) - (vD ** 2 / hD + 0.5 * g * hD ** 2))
            Fy[y, x] = (Vy, Uy * Vy / Hy, Vy ** 2 / Hy + 0.5 * g * Hy ** 2)
    out = np.zeros((3, ny, nx))
    for y in range(1, ny + 1):
        for x in range(1, nx + 1):
            for k, q in enumerate((h, u, v)):
                out[k, y - 1, x - 1] = (q(y, x) - dt / dx * (Fx[y, x][k] - Fx[y, x - 1][k])
                                        - dt / dy * (Fy[y, x][k] - Fy[y - 1, x][k]))
    return out


def main():
    os.makedirs(OUT, exist_ok=True)
    cp = dsl_eval.load_checked(FK)

    # --- config 1 -------------------------------------------------------
    n = 256
    H, U, V = so.init_state(n, n, "f32", boundary="reflective")
    dts, rows = [], []
    st = (H, U, V)
    step1 = None
    t = 0.0
    for k in range(100):
        dt = so.stable_dt(*st, 1.0, 1.0, cfl=0.9)
        st = dsl_step(cp, *st, 1.0, 1.0, dt, "reflective")
        t += dt
        dts.append(dt)
        rows.append((k + 1, t, dt) + so.diagnostics(*st))
        if k == 0:
            step1 = tuple(a.copy() for a in st)
    ref = so.run(H, U, V, 100, cfl=0.9)
    assert all(np.array_equal(a, b) for a, b in zip(st, (ref.H, ref.U, ref.V)))
    np.savez_compressed(os.path.join(OUT, "cfg1_sw256_f32_reflective.npz"),
                        H0=H, U0=U, V0=V, H1=step1[0], U1=step1[1], V1=step1[2],
                        H100=st[0], U100=st[1], V100=st[2], dt=np.array(dts),
                        rows=np.array(rows))
    print("cfg1: final mass", rows[-1][3], "dt0", dts[0])

    # --- random states --------------------------------------------------
    for prec in ("f32", "f64"):
        for bc in ("reflective", "periodic"):
            H, U, V = so.random_state(64, 48, prec, seed=1107, boundary=bc)
            st = (H, U, V)
            snaps = {}
            for k in range(10):
                st = dsl_step(cp, *st, 1.0, 0.7, 0.1, bc)
                if k in (0, 9):
                    snaps[k + 1] = tuple(a.copy() for a in st)
            np.savez_compressed(os.path.join(OUT, f"rand_{prec}_{bc}.npz"),
                                H0=H, U0=U, V0=V,
                                H1=snaps[1][0], U1=snaps[1][1], V1=snaps[1][2],
                                H10=snaps[10][0], U10=snaps[10][1], V10=snaps[10][2])
            print("rand", prec, bc, "ok")

    # --- 4x4 periodic hand oracle ----------------------------------------
    H, U, V = so.random_state(4, 4, "f64", seed=4, boundary="periodic")
    hand = hand_step(H.tolist(), U.tolist(), V.tolist(), 1.0, 1.0, 0.05)
    np.savez_compressed(os.path.join(OUT, "hand4_periodic_f64.npz"),
                        H0=H, U0=U, V0=V, out=hand, dt=0.05)
    got = so.wave_advance(1.0, 1.0, 0.05, H, U, V)
    err = max(float(np.max(np.abs(a - b))) for a, b in zip(got, hand))
    print("hand4 max abs diff vs oracle", err)
    assert err < 1e-12
    assert math.isclose(so.stable_dt(np.ones((4, 4)), np.zeros((4, 4)), np.zeros((4, 4)), 1.0, 1.0),
                        1.0 / math.sqrt(9.8), rel_tol=0, abs_tol=1e-15)


def spec64():
    """``spec64_f64_<bc>.npz`` -- SPEC.md's f64 acceptance setting
    (SPEC.md:648-651): 64x64 f64 Gaussian hump, CFL 0.9 recomputed every
    step, 100 steps, per boundary mode: inputs, states after 1 and 100
    steps, the dt series and the diagnostics rows (AST evaluator over the
    reference parser/sema, cross-checked against the numpy oracle)."""
    cp = dsl_eval.load_checked(FK)
    n = 64
    for bc in ("reflective", "periodic"):
        H, U, V = so.init_state(n, n, "f64", boundary=bc)
        st, dts, rows, t, step1 = (H, U, V), [], [], 0.0, None
        for k in range(100):
            dt = so.stable_dt(*st, 1.0, 1.0, cfl=0.9)
            st = dsl_step(cp, *st, 1.0, 1.0, dt, bc)
            t += dt
            dts.append(dt)
            rows.append((k + 1, t, dt) + so.diagnostics(*st))
            if k == 0:
                step1 = tuple(a.copy() for a in st)
        ref = so.run(H, U, V, 100, cfl=0.9, boundary=bc)
        assert all(np.array_equal(a, b) for a, b in zip(st, (ref.H, ref.U, ref.V)))
        np.savez_compressed(os.path.join(OUT, f"spec64_f64_{bc}.npz"),
                            H0=H, U0=U, V0=V, H1=step1[0], U1=step1[1], V1=step1[2],
                            H100=st[0], U100=st[1], V100=st[2], dt=np.array(dts), rows=np.array(rows))
        print("spec64", bc, "final mass", rows[-1][3], "mass drift", rows[-1][3] / rows[0][3] - 1)


if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "spec64":
        spec64()
    else:
        main()
        spec64()
