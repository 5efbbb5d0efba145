#!/usr/bin/env python
"""The SPEC time loop (CFL dt from the previous state every step + per-step
diagnostics, one eager Simulation.advance call) per grid size: per-step time
with the chunked graph replay (fkc_sw_advance_n run_chunked) against the
launch-per-step loop (FKC_NO_CHUNK=1) and against a graph of fixed-dt steps without reductions
(Simulation.capture, the floor); and that fixed-dt loop through eager
advance calls, chunked and per step.  Device-timed with CUDA events around the call.

    python scripts/chunk_timing.py [--sizes ..] [--modes exact,fast] [--prec f32] [--out FILE]
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
    ap.add_argument("--sizes", default="256,384,512,768,1024,1448,2048,2896,4096")
    ap.add_argument("--modes", default="exact,fast")
    ap.add_argument("--prec", default="f32,f64")
    ap.add_argument("--steps", type=int, default=512)
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    import torch

    from paper_1107_2157_b200 import swdemo

    rows = []

    def timed(fn, stream):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record(stream)
        fn()
        e1.record(stream)
        torch.cuda.synchronize()
        return e0.elapsed_time(e1)

    for prec in args.prec.split(","):
        for n in (int(s) for s in args.sizes.split(",")):
            k = args.steps
            for mode in args.modes.split(","):
                row = {"n": n, "prec": prec, "mode": mode, "steps": k}
                stream = torch.cuda.Stream()
                with torch.cuda.stream(stream):
                    cfg = swdemo.SWConfig(nx=n, ny=n, steps=3 * k + 8, cfl_factor=0.9, mode=mode, precision=prec)
                    for label, env in (("chunk", None), ("per_step", "1")):
                        if env:
                            os.environ["FKC_NO_CHUNK"] = env
                        try:
                            sim = swdemo.Simulation(cfg, state=swdemo.init_state(cfg).to_device(), diagnostics=True,
                                                    stream=stream)
                            sim.advance(k)          # warm-up (graph build)
                            best = min(timed(lambda: sim.advance(k // 2), stream) for _ in range(2))
                            row[f"{label}_us"] = round(best / (k // 2) * 1e3, 3)
                        finally:
                            os.environ.pop("FKC_NO_CHUNK", None)
                    # floor: the same steps at a fixed dt, no reductions, replayed from a graph
                    st0 = swdemo.init_state(cfg).to_device()
                    fcfg = swdemo.SWConfig(nx=n, ny=n, dt=0.3 * swdemo.stable_dt(st0, 1.0), mode=mode, precision=prec)
                    sim = swdemo.Simulation(fcfg, state=st0, diagnostics=False, stream=stream)
                    rep = sim.capture(k // 2)
                    rep()
                    row["graph_us"] = round(timed(rep, stream) / (k // 2) * 1e3, 3)
                    # the same fixed-dt steps through eager advance calls
                    for label, env in (("fixed_chunk", None), ("fixed_per_step", "1")):
                        if env:
                            os.environ["FKC_NO_CHUNK"] = env
                        try:
                            sim = swdemo.Simulation(fcfg, state=swdemo.init_state(cfg).to_device(),
                                                    diagnostics=False, stream=stream)
                            sim.advance(k)
                            best = min(timed(lambda: sim.advance(k // 2), stream) for _ in range(2))
                            row[f"{label}_us"] = round(best / (k // 2) * 1e3, 3)
                        finally:
                            os.environ.pop("FKC_NO_CHUNK", None)
                for key in ("chunk", "per_step", "graph", "fixed_chunk", "fixed_per_step"):
                    row[f"{key}_gcell_s"] = round(n * n / row[f"{key}_us"] / 1e3, 2)
                rows.append(row)
                print(json.dumps(row), flush=True)
    if args.out:
        with open(args.out, "w") as f:
            json.dump({"note": __doc__.split("\n\n")[0], "rows": rows}, f, indent=1)


if __name__ == "__main__":
    main()
