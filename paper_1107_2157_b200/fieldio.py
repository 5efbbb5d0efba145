"""On-disk formats of the reference's swdemo / cli (SPEC.md "External
Interfaces" of swdemo, :564; cmd_run / cmd_compare, :601-618):

* Field CSV -- row-major, one grid row (full extent, halo included) per line,
  ``.`` decimal, header line ``# nx ny left right down up precision`` where
  nx, ny is the FULL extent (field.py:25-37: a Field's ``full`` Extent) and
  left..up the halo the field is used with;
* diagnostics CSV -- header ``step,t,dt,mass,max_hu,max_hv``, one row per
  step;
* run config -- flat ``key = value`` text, keys exactly the SWConfig fields
  (SPEC.md:483-488, :603, :633).

Field values are written as 17-significant-digit decimals of their exact
binary64 value (an f32 widens exactly), so a write -> read cycle is
bit-exact (signed zeros included).  Host-side plumbing only: the numbers
come from / go to the device through ``DeviceField``.
"""

from __future__ import annotations

import os
from typing import Dict, Iterable, List, Sequence, Tuple

import numpy as np

from .field import Field, dtype_of
from .region import Extent, Halo, UNIT_HALO

DIAG_HEADER = ("step", "t", "dt", "mass", "max_hu", "max_hv")


class FieldFormatError(ValueError):
    """Malformed Field CSV (the CLI maps it to exit code 2)."""


def write_field_csv(path: str, f: Field, halo: Halo = UNIT_HALO) -> None:
    """Write a host Field (full extent incl. halo) as CSV.  Every value is
    printed as the 17-significant-digit decimal of its exact binary64 value
    (an f32 widens exactly), so reading it back is bit-exact."""
    ny, nx = f.data.shape
    with open(path, "w") as fh:
        fh.write(f"# {nx} {ny} {halo.left} {halo.right} {halo.down} {halo.up} {f.precision}\n")
        np.savetxt(fh, np.asarray(f.data, np.float64), fmt="%.17g", delimiter=",")


def read_field_csv(path: str) -> Tuple[Field, Halo]:
    """Read a Field CSV back: (Field, halo).  Raises FieldFormatError."""
    try:
        with open(path) as fh:
            head = fh.readline()
            if not head.startswith("#"):
                raise FieldFormatError(f"{path}: missing '# nx ny left right down up precision' header")
            parts = head[1:].split()
            if len(parts) != 7:
                raise FieldFormatError(f"{path}: header needs 7 fields, got {len(parts)}")
            nx, ny, l, r, d, u = (int(p) for p in parts[:6])
            precision = parts[6]
            dt = dtype_of(precision)
            rows = [line for line in fh.read().splitlines() if line.strip()]
    except (OSError, ValueError) as e:
        if isinstance(e, FieldFormatError):
            raise
        raise FieldFormatError(f"{path}: {e}") from e
    if len(rows) != ny:
        raise FieldFormatError(f"{path}: {len(rows)} rows, header says {ny}")
    try:
        vals = np.loadtxt(rows, delimiter=",", dtype=np.float64, ndmin=2)
    except ValueError as e:
        raise FieldFormatError(f"{path}: {e}") from e
    if vals.shape != (ny, nx):
        raise FieldFormatError(f"{path}: values shape {vals.shape}, header says {(ny, nx)}")
    return Field(Extent(nx, ny), vals.astype(dt), precision), Halo(l, r, d, u)


def write_diagnostics_csv(path: str, rows: Iterable[Sequence[float]]) -> None:
    with open(path, "w") as fh:
        fh.write(",".join(DIAG_HEADER) + "\n")
        for row in rows:
            step, t, dt, mass, mhu, mhv = row
            fh.write(f"{int(step)},{float(t)!r},{float(dt)!r},{float(mass)!r},{float(mhu)!r},{float(mhv)!r}\n")


def read_diagnostics_csv(path: str) -> np.ndarray:
    with open(path) as fh:
        head = fh.readline().strip().split(",")
        if tuple(head) != DIAG_HEADER:
            raise FieldFormatError(f"{path}: diagnostics header {head} != {list(DIAG_HEADER)}")
        rows = [[float(v) for v in line.split(",")] for line in fh.read().splitlines() if line.strip()]
    return np.array(rows, np.float64).reshape(-1, len(DIAG_HEADER))


# ---------------------------------------------------------------------------
# run config (flat key = value, SWConfig fields)
# ---------------------------------------------------------------------------

_INT_KEYS = ("nx", "ny", "steps")
_FLOAT_KEYS = ("dx", "dy", "g", "cfl_factor", "base", "amplitude", "width", "dt")
_STR_KEYS = ("boundary", "precision", "mode", "variant")


def parse_config_text(text: str) -> Dict[str, object]:
    """``key = value`` lines (``#`` comments, blank lines ignored) -> SWConfig
    keyword arguments.  ``interior = NXxNY``, ``center = cx,cy`` and
    ``group = NXxNY`` are accepted in the reference's spelling."""
    out: Dict[str, object] = {}
    for ln, raw in enumerate(text.splitlines(), 1):
        line = raw.split("#", 1)[0].strip()
        if not line:
            continue
        if "=" not in line:
            raise ValueError(f"config line {ln}: expected 'key = value', got {raw!r}")
        k, v = (s.strip() for s in line.split("=", 1))
        if k in out:
            raise ValueError(f"config line {ln}: duplicate key {k!r}")
        if k == "interior":
            nx, ny = v.lower().split("x")
            out["nx"], out["ny"] = int(nx), int(ny)
        elif k == "group":
            gx, gy = v.lower().split("x")
            out["group"] = (int(gx), int(gy))
        elif k == "center":
            cx, cy = v.split(",")
            out["center"] = (float(cx), float(cy))
        elif k in _INT_KEYS:
            out[k] = int(v)
        elif k in _FLOAT_KEYS:
            out[k] = None if v.lower() in ("none", "cfl") else float(v)
        elif k in _STR_KEYS:
            out[k] = v
        else:
            raise ValueError(f"config line {ln}: unknown key {k!r}")
    return out


def read_config(path: str):
    from .swdemo import SWConfig
    with open(path) as fh:
        return SWConfig(**parse_config_text(fh.read()))


def write_config(path: str, cfg) -> None:
    lines: List[str] = []
    for k in ("nx", "ny", "dx", "dy", "g", "cfl_factor", "steps", "boundary", "base", "amplitude", "precision",
              "mode", "variant"):
        lines.append(f"{k} = {getattr(cfg, k)}")
    if cfg.center is not None:
        lines.append(f"center = {cfg.center[0]!r},{cfg.center[1]!r}")
    if cfg.width is not None:
        lines.append(f"width = {cfg.width!r}")
    if cfg.dt is not None:
        lines.append(f"dt = {cfg.dt!r}")
    lines.append(f"group = {cfg.group[0]}x{cfg.group[1]}")
    with open(path, "w") as fh:
        fh.write("\n".join(lines) + "\n")


def save_state_npz(path: str, state, rows=None) -> None:
    """Checkpoint a state (host or device) to one .npz: H, U, V full arrays
    plus g, dx, dy, t, precision and optionally the diagnostics rows
    (checkpoint = state to host Fields)."""
    host = state.to_host() if getattr(state, "on_device", False) else state
    extra = {} if rows is None else {"rows": np.asarray(rows, np.float64).reshape(-1, len(DIAG_HEADER))}
    np.savez(path, H=host.H.data, U=host.U.data, V=host.V.data,
             meta=np.array([host.g, host.dx, host.dy, host.t], np.float64),
             precision=np.array(host.H.precision), **extra)


def load_state_npz(path: str):
    """Inverse of save_state_npz: (host SWState, rows or None)."""
    from .swdemo import SWState
    d = np.load(path)
    prec = str(d["precision"])
    fields = [Field(Extent(d[k].shape[1], d[k].shape[0]), d[k].astype(dtype_of(prec)), prec) for k in "HUV"]
    g, dx, dy, t = (float(x) for x in d["meta"])
    rows = d["rows"] if "rows" in d.files else None
    return SWState(*fields, g, dx, dy, t), rows


def state_paths(run_dir: str) -> Dict[str, str]:
    return {"H": os.path.join(run_dir, "H.csv"), "U": os.path.join(run_dir, "U.csv"),
            "V": os.path.join(run_dir, "V.csv"), "diag": os.path.join(run_dir, "diagnostics.csv")}
