#!/usr/bin/env python
"""Persistent-loop sweep (csrc/sw_tma.cuh sw_loop_tma): per-step time of the
whole-run cooperative launch against the per-step kernels replayed from a
CUDA graph, per grid size, mode and loop schedule (rows per segment, warps
per CTA); fixed dt (the bench configuration) and the SPEC run (CFL dt every
step + diagnostics).  Device-timed with CUDA events around one
fkc_sw_advance_n call (loop) / graph replays (per step).

    python scripts/loop_sweep.py [--sizes ..] [--modes fast,exact] [--segs 0,6,10] [--out FILE]
"""

from __future__ import annotations

import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--sizes", default="256,512,768,1024,1448,2048,2896,4096")
    ap.add_argument("--modes", default="fast,exact")
    ap.add_argument("--segs", default="0")
    ap.add_argument("--warps", default="1")
    ap.add_argument("--cfl", type=int, default=1, help="also time the CFL run (dt from the previous state)")
    ap.add_argument("--baseline", type=int, default=1, help="also time the per-step graph path")
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    import torch

    from bench import device_gaussian_state
    from paper_1107_2157_b200 import _native as N
    from paper_1107_2157_b200 import swdemo

    dev = torch.device("cuda", 0)
    rows = []

    def timed(fn, stream):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record(stream)
        fn()
        e1.record(stream)
        torch.cuda.synchronize()
        return e0.elapsed_time(e1)

    for n in (int(s) for s in args.sizes.split(",")):
        k = max(20, min(2000, int(4e9 / (n * n))))     # ~4e9 cell-updates per point
        for mode in args.modes.split(","):
            dt = 0.3 * swdemo.stable_dt(device_gaussian_state(n, n, dev), 1.0)

            def fresh():
                return device_gaussian_state(n, n, dev)
            row = {"n": n, "mode": mode, "steps": k}
            stream = torch.cuda.Stream()
            with torch.cuda.stream(stream):
                if args.baseline:
                    best = None
                    for variant in ("tma", "generic"):
                        cfg = swdemo.SWConfig(nx=n, ny=n, dt=dt, mode=mode, variant=variant)
                        sim = swdemo.Simulation(cfg, state=fresh(), diagnostics=False, stream=stream)
                        rep = sim.capture(k if k % 2 == 0 else k + 1)
                        rep()
                        ms = timed(rep, stream) / (k if k % 2 == 0 else k + 1)
                        if best is None or ms < best[0]:
                            best = (ms, variant)
                    row["graph_us"] = round(best[0] * 1e3, 3)
                    row["graph_variant"] = best[1]
                for seg in (int(s) for s in args.segs.split(",")):
                    for warps in (int(w) for w in args.warps.split(",")):
                        cfg = swdemo.SWConfig(nx=n, ny=n, dt=dt, mode=mode, variant="loop")
                        tune = N.Tune(seg=seg, warps=warps)
                        sim = swdemo.Simulation(cfg, state=fresh(), diagnostics=False, stream=stream, tune=tune)
                        try:
                            sim.advance(4)
                            ms = timed(lambda: sim.advance(k), stream) / k
                        except Exception as e:          # schedule does not fit
                            row[f"loop_seg{seg}_w{warps}"] = f"n/a: {str(e)[:60]}"
                            continue
                        row[f"loop_seg{seg}_w{warps}_us"] = round(ms * 1e3, 3)
                if args.cfl:
                    kc = min(k, 400)
                    for variant in ("loop", "tma"):
                        cfg = swdemo.SWConfig(nx=n, ny=n, steps=kc + 4, cfl_factor=0.9, mode=mode, variant=variant)
                        sim = swdemo.Simulation(cfg, state=fresh(), diagnostics=True, stream=stream)
                        sim.advance(4)
                        ms = timed(lambda: sim.advance(kc), stream) / kc
                        row[f"cfl_{variant}_us"] = round(ms * 1e3, 3)
            best_loop = min((v for kk, v in row.items() if kk.startswith("loop_seg") and isinstance(v, float)),
                            default=None)
            if best_loop:
                row["loop_best_gcell_s"] = round(n * n / best_loop / 1e3, 2)
            if "graph_us" in row:
                row["graph_gcell_s"] = round(n * n / row["graph_us"] / 1e3, 2)
            rows.append(row)
            print(json.dumps(row), flush=True)
    if args.out:
        with open(args.out, "w") as f:
            json.dump({"note": __doc__.split("\n\n")[0], "rows": rows}, f, indent=1)


if __name__ == "__main__":
    main()
