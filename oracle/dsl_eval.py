"""AST-walking evaluator of a reference CheckedProgram -- TEST INFRASTRUCTURE.

Restates the absent ``refinterp.eval_kernel``
directly over the reference's own parser and semantic checker
(``fkc.frontend.parse_source`` frontend.py:672, ``fkc.sema.analyze``
sema.py:371).  It is used in THIS container only (it needs
``/root/reference/pkg/src`` on ``sys.path``) to pin the op order of the
hand-written numpy oracle ``oracle/sw_oracle.py:wave_advance`` and to
generate the golden fixtures under ``tests/golden/`` (``gen_golden.py``).

Semantics:
* statements run in source order; each RHS is evaluated to a fresh array
  before any store;
* ``region_cpy(A, halo)`` = copy of ``interior_of(A.full, halo)``
  (region.py:74-80) using the halo snapshot live at that statement
  (``CheckedProgram.halo_table``, sema.py:84-94);
* stores through pointer locals write only the bound interior
  (``CheckedProgram.output_bindings``, sema.py:290-307);
* arithmetic is IEEE per op in the field precision, left-to-right over the
  parsed tree (no reassociation); literals and scalar params are rounded to
  the field precision first (OpenCL ``float`` kernel args).
"""

from __future__ import annotations

import os
import sys

import numpy as np

REF_SRC = os.environ.get("FKC_REFERENCE_SRC", "/root/reference/pkg/src")


def reference_available() -> bool:
    return os.path.isdir(os.path.join(REF_SRC, "fkc"))


def _import_fkc():
    if REF_SRC not in sys.path:
        sys.path.insert(0, REF_SRC)
    from fkc import field, frontend, region, sema  # noqa: WPS433
    return frontend, sema, region, field


def load_checked(path: str):
    frontend, sema, _, _ = _import_fkc()
    with open(path) as fh:
        kernels, elementals = frontend.parse_source(fh.read())
    assert len(kernels) == 1, kernels
    return sema.analyze(kernels[0])


def eval_kernel(cp, inputs: dict, params: dict, dtype) -> dict:
    """Evaluate ``cp`` on full arrays ``inputs`` (name -> ndarray).

    Returns name -> ndarray for every intent(out) array; output cells outside
    the bound interiors are left at zero (the driver fills halos).
    """
    frontend, _, region_mod, _ = _import_fkc()
    f = np.dtype(dtype).type
    prog = cp.program
    elementals = {e.name: e for e in prog.elementals}
    arrays = {k.lower(): np.asarray(v) for k, v in inputs.items()}
    full_shape = next(iter(arrays.values())).shape
    outs = {p.name: np.zeros(full_shape, dtype) for p in prog.params
            if p.kind == "array-2d-real" and p.intent == "out"}
    scal = {k.lower(): f(v) for k, v in params.items()}
    locals_: dict[str, np.ndarray] = {}

    def halo_of(arg, halos):
        if isinstance(arg, frontend.HaloLit):
            return region_mod.Halo.of(arg.values)
        return halos[arg.name]

    def region_view(a: np.ndarray, halo):
        ny, nx = a.shape
        rect = region_mod.interior_of(region_mod.Extent(nx, ny), halo)
        return a[rect.y0:rect.y0 + rect.ny, rect.x0:rect.x0 + rect.nx]

    def ev(e, halos, env):
        if isinstance(e, frontend.RealLit):
            return f(e.value)
        if isinstance(e, frontend.IntLit):
            return f(e.value)
        if isinstance(e, frontend.Ident):
            if e.name in env:
                return env[e.name]
            if e.name in scal:
                return scal[e.name]
            raise KeyError(e.name)
        if isinstance(e, frontend.Paren):
            return ev(e.inner, halos, env)
        if isinstance(e, frontend.Neg):
            return -ev(e.operand, halos, env)
        if isinstance(e, frontend.BinOp):
            a = ev(e.left, halos, env)
            b = ev(e.right, halos, env)
            if e.op == "+":
                return a + b
            if e.op == "-":
                return a - b
            if e.op == "*":
                return a * b
            if e.op == "/":
                return a / b
            raise ValueError(e.op)
        if isinstance(e, frontend.Call):
            if e.name == "region_cpy":
                src, harg = e.args
                a = arrays.get(src.name)
                if a is None:
                    a = locals_[src.name]
                return region_view(a, halo_of(harg, halos)).copy()
            if e.name in elementals:
                fn = elementals[e.name]
                args = [ev(a, halos, env) for a in e.args]
                return ev(fn.body, halos, dict(zip(fn.params, args)))
            intr = {"sqrt": np.sqrt, "abs": np.abs, "exp": np.exp,
                    "min": np.minimum, "max": np.maximum}
            if e.name in intr:
                return intr[e.name](*[ev(a, halos, env) for a in e.args])
            raise ValueError(f"unknown call {e.name}")
        raise TypeError(type(e))

    for idx, stmt in enumerate(prog.body):
        halos = cp.halo_table[idx]
        if isinstance(stmt, (frontend.HaloAssign, frontend.PtrAssign)):
            continue
        val = ev(stmt.rhs, halos, {})
        if stmt.lhs in cp.output_bindings:
            arr, halo = cp.output_bindings[stmt.lhs]
            region_view(outs[arr], halo)[...] = val
        else:
            locals_[stmt.lhs] = np.asarray(val)
    return outs
