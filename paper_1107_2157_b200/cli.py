"""Command-line entry points of the reference's ``cli`` module that sit on
the solver path, executed by the B200 engine:

    python -m paper_1107_2157_b200.cli run CONFIG [--engine cuda] [-o DIR]
    python -m paper_1107_2157_b200.cli compare DIR_A DIR_B [--rtol R]
    python -m paper_1107_2157_b200.cli bench CONFIG [--sizes 16,32,...]

* ``run``     (cmd_run): config file -> diagnostics CSV and
  final-state CSVs in DIR; prints wall-clock total and per-step mean.
* ``compare`` (cmd_compare): relative difference of two
  run directories, per cell against max(|a|, |b|, floor x field scale)
  (``--floor``: 1 = normwise, 0 = strictly elementwise); prints the worst
  offender.
* ``bench``   (cmd_bench): per-step mean time per engine
  and interior width, CSV on stdout; asserts nothing.

Exit codes are the reference's stable contract: 0 success,
1 domain failure (non-finite / non-positive depth / comparison beyond
rtol), 2 usage or I/O error.  ``check`` / ``emit`` belong to the DSL
compiler (frontend / sema / codegen), which stays in the reference package
(out of scope): they exit 2 with a pointer there.
The only engine is ``cuda``; the reference's CPU engines
(``native | ref | sim``) are not re-implemented here.
"""

from __future__ import annotations

import argparse
import os
import sys
import time
from typing import List, Optional

import numpy as np

EXIT_OK, EXIT_DOMAIN, EXIT_USAGE = 0, 1, 2


class _Parser(argparse.ArgumentParser):
    def error(self, message):   # usage errors exit 2 -- argparse's default too
        self.print_usage(sys.stderr)
        print(f"fkc: error: {message}", file=sys.stderr)
        raise SystemExit(EXIT_USAGE)


def _parser() -> argparse.ArgumentParser:
    ap = _Parser(prog="fkc", description="B200 engine of the ForOpenCL shallow-water demo")
    sub = ap.add_subparsers(dest="cmd", required=True)
    r = sub.add_parser("run", help="run a config, write diagnostics + final-state CSVs")
    r.add_argument("config")
    r.add_argument("--engine", default="cuda")
    r.add_argument("-o", "--out", default="run_out")
    r.add_argument("--precision", choices=["f32", "f64"])
    r.add_argument("--mode", choices=["exact", "fast"])
    c = sub.add_parser("compare", help="compare two run directories")
    c.add_argument("a")
    c.add_argument("b")
    c.add_argument("--rtol", type=float, default=0.0)
    c.add_argument("--floor", type=float, default=1.0,
                   help="relative-difference denominator floor, as a fraction of the field's max |value| "
                        "(1: normwise, 0: strictly elementwise)")
    b = sub.add_parser("bench", help="per-step time per engine and width (CSV)")
    b.add_argument("config")
    b.add_argument("--sizes", default="16,32,64,128,256,512,1024,2048,4096")
    b.add_argument("--engines", default="cuda-exact,cuda-fast")
    for name in ("check", "emit"):
        s = sub.add_parser(name, help="DSL compiler command (reference package)")
        s.add_argument("source", nargs="?")
        s.add_argument("rest", nargs=argparse.REMAINDER)
    return ap


def cmd_run(args) -> int:
    from . import fieldio, swdemo
    if args.engine != "cuda":
        print(f"fkc: engine {args.engine!r} is provided by the reference package; this build has 'cuda'",
              file=sys.stderr)
        return EXIT_USAGE
    try:
        cfg = fieldio.read_config(args.config)
    except (OSError, ValueError, TypeError) as e:
        print(f"fkc: bad config {args.config}: {e}", file=sys.stderr)
        return EXIT_USAGE
    if args.precision:
        cfg.precision = args.precision
    if args.mode:
        cfg.mode = args.mode
    import torch
    os.makedirs(args.out, exist_ok=True)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    try:
        res = swdemo.run(cfg, engine="cuda", to_host=True)
    except (swdemo.NonfiniteValue, swdemo.NonPositiveDepth) as e:
        print(f"fkc: {type(e).__name__}: {e}", file=sys.stderr)
        return EXIT_DOMAIN
    wall = time.perf_counter() - t0
    paths = fieldio.state_paths(args.out)
    for name in ("H", "U", "V"):
        fieldio.write_field_csv(paths[name], getattr(res.state, name))
    fieldio.write_diagnostics_csv(paths["diag"], res.rows)
    per = wall / cfg.steps * 1e3 if cfg.steps else 0.0
    print(f"total {wall:.6f} s, {cfg.steps} steps, {per:.6f} ms/step (engine cuda, mode {cfg.mode}, "
          f"{cfg.nx}x{cfg.ny} {cfg.precision})")
    return EXIT_OK


def _rel_worst(a: np.ndarray, b: np.ndarray, floor: float = 1.0):
    """max over cells of |a-b| / max(|a|, |b|, floor * scale), scale = the
    larger max |value| of the two fields (0 where a == b; inf where exactly
    one is non-finite), and the argmax (row, col).  floor = 1 (default) is
    the normwise relative difference, |a-b| / max|field|: round-off of the
    O(g h^2) fluxes leaves absolute errors of ~1e-6 on small f32 momenta,
    which is what lets f32 and f64 runs compare at rtol 1e-4;
    floor = 0 is the strict elementwise relative difference."""
    a64, b64 = a.astype(np.float64), b.astype(np.float64)
    fin = np.isfinite(a64) & np.isfinite(b64)
    scale = max(float(np.max(np.abs(a64[fin]), initial=0.0)), float(np.max(np.abs(b64[fin]), initial=0.0)))
    with np.errstate(invalid="ignore", divide="ignore"):
        den = np.maximum(np.maximum(np.abs(a64), np.abs(b64)), floor * scale)
        rel = np.where(a64 == b64, 0.0, np.abs(a64 - b64) / den)
    rel = np.where(np.isnan(rel), np.inf, rel)
    idx = np.unravel_index(int(np.argmax(rel)), rel.shape) if rel.size else (0, 0)
    return float(rel[idx]) if rel.size else 0.0, idx


def cmd_compare(args) -> int:
    from . import fieldio
    pa, pb = fieldio.state_paths(args.a), fieldio.state_paths(args.b)
    worst = (0.0, None, None, None, None)
    try:
        for name in ("H", "U", "V"):
            fa, _ = fieldio.read_field_csv(pa[name])
            fb, _ = fieldio.read_field_csv(pb[name])
            if fa.data.shape != fb.data.shape:
                print(f"fkc: shape mismatch in {name}: {fa.data.shape} vs {fb.data.shape}", file=sys.stderr)
                return EXIT_USAGE
            r, (y, x) = _rel_worst(fa.data, fb.data, args.floor)
            if r > worst[0] or worst[1] is None:
                worst = (r, name, (int(x), int(y)), float(fa.data[y, x]), float(fb.data[y, x]))
        if os.path.exists(pa["diag"]) and os.path.exists(pb["diag"]):
            da, db = fieldio.read_diagnostics_csv(pa["diag"]), fieldio.read_diagnostics_csv(pb["diag"])
            if da.shape != db.shape:
                print(f"fkc: shape mismatch in diagnostics: {da.shape} vs {db.shape}", file=sys.stderr)
                return EXIT_USAGE
            if da.size:
                r, (row, col) = _rel_worst(da, db, args.floor)
                if r > worst[0]:
                    worst = (r, "diagnostics", (int(col), int(row)), float(da[row, col]), float(db[row, col]))
    except (OSError, fieldio.FieldFormatError) as e:
        print(f"fkc: {e}", file=sys.stderr)
        return EXIT_USAGE
    r, name, xy, va, vb = worst
    if r <= args.rtol:
        print(f"match: max relative difference {r:.3e} <= rtol {args.rtol:.3e}")
        return EXIT_OK
    print(f"mismatch: max relative difference {r:.3e} > rtol {args.rtol:.3e} in {name} at (x, y) = {xy}: "
          f"{va!r} vs {vb!r}")
    return EXIT_DOMAIN


def cmd_bench(args) -> int:
    import dataclasses

    import torch

    from . import fieldio, swdemo
    try:
        base = fieldio.read_config(args.config)
        sizes = [int(s) for s in args.sizes.split(",") if s.strip()]
    except (OSError, ValueError, TypeError) as e:
        print(f"fkc: {e}", file=sys.stderr)
        return EXIT_USAGE
    engines = [e.strip() for e in args.engines.split(",") if e.strip()]
    for e in engines:
        if e not in ("cuda-exact", "cuda-fast"):
            print(f"fkc: unknown engine {e!r} (available: cuda-exact, cuda-fast)", file=sys.stderr)
            return EXIT_USAGE
    print("engine,width,steps,ms_per_step,gcell_updates_per_s")
    steps = max(1, base.steps)
    for n in sizes:
        for e in engines:
            cfg = dataclasses.replace(base, nx=n, ny=n, steps=steps, mode=e.split("-")[1])
            sim = swdemo.Simulation(cfg, diagnostics=True, capacity=steps + 2)
            sim.advance(2)                                  # warm-up (tensor maps, attributes)
            torch.cuda.synchronize()
            t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            t0.record()
            sim.advance(steps)
            t1.record()
            torch.cuda.synchronize()
            k = steps
            ms = t0.elapsed_time(t1) / k
            try:
                sim.rows()
            except (swdemo.NonfiniteValue, swdemo.NonPositiveDepth) as err:
                print(f"fkc: {type(err).__name__} at width {n}: {err}", file=sys.stderr)
                return EXIT_DOMAIN
            print(f"{e},{n},{k},{ms:.6f},{n * n / ms / 1e6:.6f}")
    return EXIT_OK


def main(argv: Optional[List[str]] = None) -> int:
    args = _parser().parse_args(argv)
    if args.cmd == "run":
        return cmd_run(args)
    if args.cmd == "compare":
        return cmd_compare(args)
    if args.cmd == "bench":
        return cmd_bench(args)
    print(f"fkc: '{args.cmd}' is part of the DSL compiler (frontend/sema/codegen) in the reference package; "
          "this build provides the solver path only (run, compare, bench)", file=sys.stderr)
    return EXIT_USAGE


if __name__ == "__main__":
    sys.exit(main())
