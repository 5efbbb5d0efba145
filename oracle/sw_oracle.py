"""CPU oracle for the shallow-water hot path -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline /
``--impl reference`` legs may import this module, and only as the checker or
as the timed CPU reference.  The product package ``paper_1107_2157_b200``
never imports it (its hot path is the sm_100a kernel behind the C-ABI).

The reference (``/root/reference``, package ``fkc``) ships no solver: the
``swdemo``/``refinterp``/``sim`` modules are specified in SPEC.md but absent
(SURVEY.md section 0).  This module restates them in numpy:

* :func:`wave_advance` -- the DSL kernel ``kernels/wave_advance.fk`` evaluated
  with refinterp semantics: every statement in
  source order, ``region_cpy`` as interior slices (SPEC.md:289-297,
  region.py:74-80), left-to-right parse-tree arithmetic, no reassociation,
  scalars and literals rounded to the field precision.  This is the
  bit-exact target ("Oracle B").  Its op order is pinned against an
  AST-walking evaluator over the reference's own parser/sema
  (``oracle/gen_golden.py``) and frozen as ``tests/golden/*.npz``.
* :func:`step_native` -- the plain formula form of SPEC.md:517-528
  ("Oracle A", the independent restatement; tolerance target).
* :func:`apply_boundary`, :func:`stable_dt`
  (SPEC.md:508-516), :func:`init_state`,
  :func:`total_mass`, :func:`run`.

Layout follows field.py:25-60 / region.py:1-6: arrays of shape
``(ny_full, nx_full)``, x = column (left/right), y = row (down/up), halo
[1,1,1,1] for the solver state.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field as dc_field

import numpy as np

DTYPES = {"f32": np.float32, "f64": np.float64}


class NonPositiveDepth(ValueError):
    """a cell or face depth h <= 0."""


class NonfiniteValue(ArithmeticError):
    """NaN/Inf in the state."""


# --------------------------------------------------------------------------
# region_cpy restated (SPEC.md:289-297 over region.py:74-80)
# --------------------------------------------------------------------------

def region(a: np.ndarray, halo) -> np.ndarray:
    """View of ``interior_of(full, halo)`` (region.py:74-80) of a full array.

    halo = (left, right, down, up); rows are y, columns are x.
    """
    left, right, down, up = halo
    ny, nx = a.shape
    if nx - left - right < 1 or ny - down - up < 1:
        raise ValueError(f"halo {halo} leaves no interior in {a.shape}")
    return a[down:ny - up, left:nx - right]


def region_cpy(a: np.ndarray, halo) -> np.ndarray:
    """Copy of the interior region."""
    return region(a, halo).copy()


def cshift(a: np.ndarray, dim: int, offset: int) -> np.ndarray:
    """cshift_ref: result(x,y) = a((x+off) mod nx, y) for
    dim=1 (x, columns); dim=2 shifts along y (rows)."""
    if dim == 1:
        return np.roll(a, -offset, axis=1)
    if dim == 2:
        return np.roll(a, -offset, axis=0)
    raise ValueError("dim must be 1 or 2")


# --------------------------------------------------------------------------
# the DSL kernel, refinterp op order (Oracle B)
# --------------------------------------------------------------------------

def _fxu(t, h, q):
    # kernels/wave_advance.fk: fxu = q*q/h + 0.5*9.8*h*h
    # parse tree: ((q*q)/h) + (((0.5*9.8)*h)*h); the scalar subtree 0.5*9.8
    # is folded in field precision (t(0.5)*t(g)).
    return ((q * q) / h) + ((t["g2"] * h) * h)


def _cross(h, u, v):
    # kernels/wave_advance.fk: cross = u*v/h  ->  (u*v)/h
    return (u * v) / h


def scalars(dtype, dx: float, dy: float, dt: float, g: float = 9.8) -> dict:
    """Scalar subtrees of wave_advance, evaluated in field precision in
    parse order (SURVEY.md 8(c) op-order conventions)."""
    f = np.dtype(dtype).type
    return {
        "half": f(0.5),
        "cx2": (f(0.5) * f(dt)) / f(dx),   # (0.5*dt/dx)
        "cy2": (f(0.5) * f(dt)) / f(dy),   # (0.5*dt/dy)
        "cx": f(dt) / f(dx),               # (dt/dx)
        "cy": f(dt) / f(dy),               # (dt/dy)
        "g2": f(0.5) * f(g),               # 0.5*9.8 in fxu
    }


def wave_advance(dx, dy, dt, H, U, V, g: float = 9.8):
    """Evaluate kernels/wave_advance.fk on full arrays (halo [1,1,1,1]).

    Returns the (ny, nx) interiors (pH, pU, pV) -- the region_ptr(o*, halo)
    targets.  Statement order and parse trees follow the .fk source exactly.
    """
    t = scalars(H.dtype, dx, dy, dt, g)
    half, cx2, cy2, cx, cy = t["half"], t["cx2"], t["cy2"], t["cx"], t["cy"]
    # step-1 halos
    f_lt, f_rt = (0, 1, 1, 1), (1, 0, 1, 1)
    f_dn, f_up = (1, 1, 0, 1), (1, 1, 1, 0)
    R = region
    Hx = (half * (R(H, f_lt) + R(H, f_rt))) + (cx2 * (R(U, f_lt) - R(U, f_rt)))
    Ux = (half * (R(U, f_lt) + R(U, f_rt))) + (
        cx2 * (_fxu(t, R(H, f_lt), R(U, f_lt)) - _fxu(t, R(H, f_rt), R(U, f_rt))))
    Vx = (half * (R(V, f_lt) + R(V, f_rt))) + (
        cx2 * (_cross(R(H, f_lt), R(U, f_lt), R(V, f_lt))
               - _cross(R(H, f_rt), R(U, f_rt), R(V, f_rt))))
    Hy = (half * (R(H, f_dn) + R(H, f_up))) + (cy2 * (R(V, f_dn) - R(V, f_up)))
    Uy = (half * (R(U, f_dn) + R(U, f_up))) + (
        cy2 * (_cross(R(H, f_dn), R(U, f_dn), R(V, f_dn))
               - _cross(R(H, f_up), R(U, f_up), R(V, f_up))))
    Vy = (half * (R(V, f_dn) + R(V, f_up))) + (
        cy2 * (_fxu(t, R(H, f_dn), R(V, f_dn)) - _fxu(t, R(H, f_up), R(V, f_up))))
    # step-2 halos
    f_lt, f_rt = (0, 1, 0, 0), (1, 0, 0, 0)
    f_dn, f_up = (0, 0, 0, 1), (0, 0, 1, 0)
    halo = (1, 1, 1, 1)
    pH = (R(H, halo) + (cx * (R(Ux, f_lt) - R(Ux, f_rt)))) + (
        cy * (R(Vy, f_dn) - R(Vy, f_up)))
    pU = (R(U, halo) + (cx * (_fxu(t, R(Hx, f_lt), R(Ux, f_lt))
                              - _fxu(t, R(Hx, f_rt), R(Ux, f_rt))))) + (
        cy * (_cross(R(Hy, f_dn), R(Uy, f_dn), R(Vy, f_dn))
              - _cross(R(Hy, f_up), R(Uy, f_up), R(Vy, f_up))))
    pV = (R(V, halo) + (cx * (_cross(R(Hx, f_lt), R(Ux, f_lt), R(Vx, f_lt))
                              - _cross(R(Hx, f_rt), R(Ux, f_rt), R(Vx, f_rt))))) + (
        cy * (_fxu(t, R(Hy, f_dn), R(Vy, f_dn)) - _fxu(t, R(Hy, f_up), R(Vy, f_up))))
    return pH, pU, pV


# --------------------------------------------------------------------------
# step_native (Oracle A): SPEC.md:517-528 formula order
# --------------------------------------------------------------------------

def step_native(dx, dy, dt, H, U, V, g: float = 9.8, check: bool = True):
    """Independent plain-formula restatement of SPEC.md:521-522."""
    f = H.dtype.type
    dx, dy, dt, g = f(dx), f(dy), f(dt), f(g)
    half = f(0.5)
    c = H[1:-1, :]; u = U[1:-1, :]; v = V[1:-1, :]
    hL, hR, uL, uR, vL, vR = c[:, :-1], c[:, 1:], u[:, :-1], u[:, 1:], v[:, :-1], v[:, 1:]
    ax = dt / (f(2) * dx)
    Hx = half * (hL + hR) - ax * (uR - uL)
    Ux = half * (uL + uR) - ax * ((uR * uR / hR + half * g * hR * hR) - (uL * uL / hL + half * g * hL * hL))
    Vx = half * (vL + vR) - ax * ((uR * vR / hR) - (uL * vL / hL))
    c = H[:, 1:-1]; u = U[:, 1:-1]; v = V[:, 1:-1]
    hD, hU, uD, uU, vD, vU = c[:-1], c[1:], u[:-1], u[1:], v[:-1], v[1:]
    ay = dt / (f(2) * dy)
    Hy = half * (hD + hU) - ay * (vU - vD)
    Uy = half * (uD + uU) - ay * ((uU * vU / hU) - (uD * vD / hD))
    Vy = half * (vD + vU) - ay * ((vU * vU / hU + half * g * hU * hU) - (vD * vD / hD + half * g * hD * hD))
    if check and (np.any(Hx <= 0) or np.any(Hy <= 0) or np.any(H[1:-1, 1:-1] <= 0)):
        raise NonPositiveDepth("face or cell depth <= 0")
    bx, by = dt / dx, dt / dy
    Fh = Ux
    Fu = Ux * Ux / Hx + half * g * Hx * Hx
    Fv = Ux * Vx / Hx
    Gh = Vy
    Gu = Uy * Vy / Hy
    Gv = Vy * Vy / Hy + half * g * Hy * Hy
    h = H[1:-1, 1:-1] - bx * (Fh[:, 1:] - Fh[:, :-1]) - by * (Gh[1:] - Gh[:-1])
    hu = U[1:-1, 1:-1] - bx * (Fu[:, 1:] - Fu[:, :-1]) - by * (Gu[1:] - Gu[:-1])
    hv = V[1:-1, 1:-1] - bx * (Fv[:, 1:] - Fv[:, :-1]) - by * (Gv[1:] - Gv[:-1])
    return h, hu, hv


# --------------------------------------------------------------------------
# boundary conditions, CFL, init, diagnostics
# --------------------------------------------------------------------------

def apply_boundary(H, U, V, mode: str = "reflective"):
    """Fill the one-cell halo in place.

    Order (fixed here, the CUDA epilogue reproduces it bit-for-bit):
    left/right halo columns over interior rows 1..ny first, then the
    down/up halo rows over all columns 0..nx+1 (corners included, so a
    corner is the double image of the diagonal interior cell).

    reflective: h mirrors the adjacent interior cell; the wall-normal
    momentum negates (hu at left/right, hv at down/up); tangential copies.
    periodic: wrap copy (left halo column = rightmost interior column).
    """
    if mode == "reflective":
        H[1:-1, 0] = H[1:-1, 1];   H[1:-1, -1] = H[1:-1, -2]
        U[1:-1, 0] = -U[1:-1, 1];  U[1:-1, -1] = -U[1:-1, -2]
        V[1:-1, 0] = V[1:-1, 1];   V[1:-1, -1] = V[1:-1, -2]
        H[0, :] = H[1, :];   H[-1, :] = H[-2, :]
        U[0, :] = U[1, :];   U[-1, :] = U[-2, :]
        V[0, :] = -V[1, :];  V[-1, :] = -V[-2, :]
    elif mode == "periodic":
        for A in (H, U, V):
            A[1:-1, 0] = A[1:-1, -2]
            A[1:-1, -1] = A[1:-1, 1]
            A[0, :] = A[-2, :]
            A[-1, :] = A[1, :]
    else:
        raise ValueError(f"unknown boundary mode {mode!r}")
    return H, U, V


def apply_boundary_sides(H, U, V, sides):
    """apply_boundary with a per-side spec (left, right, down, up), each
    'reflective' | 'periodic' | 'none' ('none' = filled by a halo exchange
    in a decomposed run).  Same order as apply_boundary: columns over the
    interior rows, then rows over all columns."""
    left, right, down, up = sides
    if left == "reflective":
        H[1:-1, 0] = H[1:-1, 1]; U[1:-1, 0] = -U[1:-1, 1]; V[1:-1, 0] = V[1:-1, 1]
    elif left == "periodic":
        for A in (H, U, V):
            A[1:-1, 0] = A[1:-1, -2]
    if right == "reflective":
        H[1:-1, -1] = H[1:-1, -2]; U[1:-1, -1] = -U[1:-1, -2]; V[1:-1, -1] = V[1:-1, -2]
    elif right == "periodic":
        for A in (H, U, V):
            A[1:-1, -1] = A[1:-1, 1]
    if down == "reflective":
        H[0, :] = H[1, :]; U[0, :] = U[1, :]; V[0, :] = -V[1, :]
    elif down == "periodic":
        for A in (H, U, V):
            A[0, :] = A[-2, :]
    if up == "reflective":
        H[-1, :] = H[-2, :]; U[-1, :] = U[-2, :]; V[-1, :] = -V[-2, :]
    elif up == "periodic":
        for A in (H, U, V):
            A[-1, :] = A[1, :]
    return H, U, V


def cfl_bound(H, U, V, dx, dy, g: float = 9.8):
    """Per-cell CFL bound min(dx,dy)/(sqrt(g h) + max(|hu|,|hv|)/h)
    (SPEC.md:508-516), field precision, this exact op order."""
    f = H.dtype.type
    h = H[1:-1, 1:-1]; u = U[1:-1, 1:-1]; v = V[1:-1, 1:-1]
    c = np.sqrt(f(g) * h) + (np.maximum(np.abs(u), np.abs(v)) / h)
    return f(min(dx, dy)) / c


def stable_dt(H, U, V, dx, dy, cfl: float = 1.0, g: float = 9.8) -> float:
    """dt = cfl * min_interior bound."""
    f = H.dtype.type
    if np.any(H[1:-1, 1:-1] <= 0):
        raise NonPositiveDepth("depth <= 0 in stable_dt")
    return float(f(cfl) * np.min(cfl_bound(H, U, V, dx, dy, g)))


def init_state(nx, ny, precision="f64", base=1.0, amplitude=0.4, center=None,
               width=None, dx=1.0, dy=1.0, boundary="reflective"):
    """Gaussian hump at cell centres; f64 then cast."""
    dt_ = np.dtype(DTYPES[precision])
    if center is None:
        center = (nx * dx / 2.0, ny * dy / 2.0)
    if width is None:
        width = nx * dx / 8.0
    xs = (np.arange(nx, dtype=np.float64) + 0.5) * dx
    ys = (np.arange(ny, dtype=np.float64) + 0.5) * dy
    r2 = (xs[None, :] - center[0]) ** 2 + (ys[:, None] - center[1]) ** 2
    h = base + amplitude * np.exp(-r2 / (width * width))
    H = np.zeros((ny + 2, nx + 2), dt_)
    U = np.zeros_like(H)
    V = np.zeros_like(H)
    H[1:-1, 1:-1] = h.astype(dt_)
    apply_boundary(H, U, V, boundary)
    return H, U, V


def random_state(nx, ny, precision="f32", seed=1107, boundary="reflective"):
    """Parity-suite input: h~U[0.9,1.1], hu,hv~U[-0.05,0.05]."""
    rng = np.random.default_rng(seed)
    dt_ = np.dtype(DTYPES[precision])
    H = np.zeros((ny + 2, nx + 2), dt_)
    U = np.zeros_like(H)
    V = np.zeros_like(H)
    H[1:-1, 1:-1] = rng.uniform(0.9, 1.1, (ny, nx)).astype(dt_)
    U[1:-1, 1:-1] = rng.uniform(-0.05, 0.05, (ny, nx)).astype(dt_)
    V[1:-1, 1:-1] = rng.uniform(-0.05, 0.05, (ny, nx)).astype(dt_)
    apply_boundary(H, U, V, boundary)
    return H, U, V


def total_mass(H, dx=1.0, dy=1.0) -> float:
    """Sum of interior h * dx * dy, f64 accumulation."""
    return float(np.sum(H[1:-1, 1:-1], dtype=np.float64)) * dx * dy


def diagnostics(H, U, V, dx=1.0, dy=1.0):
    return (total_mass(H, dx, dy),
            float(np.max(np.abs(U[1:-1, 1:-1]))),
            float(np.max(np.abs(V[1:-1, 1:-1]))))


def step(H, U, V, dx, dy, dt, g=9.8, boundary="reflective", form="dsl",
         out=None):
    """One double-buffered step: advance interiors into fresh (or given)
    output arrays and fill their halos with apply_boundary."""
    if form == "dsl":
        h, hu, hv = wave_advance(dx, dy, dt, H, U, V, g)
    else:
        h, hu, hv = step_native(dx, dy, dt, H, U, V, g)
    if out is None:
        out = (np.empty_like(H), np.empty_like(U), np.empty_like(V))
    oH, oU, oV = out
    oH[1:-1, 1:-1] = h
    oU[1:-1, 1:-1] = hu
    oV[1:-1, 1:-1] = hv
    apply_boundary(oH, oU, oV, boundary)
    return oH, oU, oV


@dataclass
class RunResult:
    H: np.ndarray
    U: np.ndarray
    V: np.ndarray
    t: float
    rows: list = dc_field(default_factory=list)   # (step, t, dt, mass, max_hu, max_hv)


def run(H, U, V, steps, dx=1.0, dy=1.0, g=9.8, boundary="reflective",
        cfl=0.9, dt=None, form="dsl", diag_every=1):
    """Time loop: BC -> dt -> advance -> swap -> diagnostics.

    ``dt=None`` recomputes dt = stable_dt(state) every step with ``cfl``;
    a number fixes it.  Aborts with NonfiniteValue on NaN/Inf.
    """
    H, U, V = H.copy(), U.copy(), V.copy()
    apply_boundary(H, U, V, boundary)
    bufs = (np.empty_like(H), np.empty_like(U), np.empty_like(V))
    t = 0.0
    rows = []
    for n in range(steps):
        d = stable_dt(H, U, V, dx, dy, cfl, g) if dt is None else float(dt)
        oH, oU, oV = step(H, U, V, dx, dy, d, g, boundary, form, out=bufs)
        bufs = (H, U, V)
        H, U, V = oH, oU, oV
        t += d
        if diag_every and (n + 1) % diag_every == 0:
            m, mu, mv = diagnostics(H, U, V, dx, dy)
            if not (math.isfinite(m) and math.isfinite(mu) and math.isfinite(mv)):
                raise NonfiniteValue(f"non-finite state at step {n + 1}")
            rows.append((n + 1, t, d, m, mu, mv))
    return RunResult(H, U, V, t, rows)
