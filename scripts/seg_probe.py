#!/usr/bin/env python
"""A/B of TMA segment lengths for the plain fast step at one grid size, by
launch pattern: one event per step (bench.py's headline loop), one
advance(K) call (PDL-chained launches), a replayed CUDA graph.  Fresh state
per run, runs interleaved, repeated.  python scripts/seg_probe.py [n] [reps]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from bench import device_gaussian_state  # noqa: E402
from paper_1107_2157_b200 import _native as N  # noqa: E402
from paper_1107_2157_b200 import swdemo  # noqa: E402

dev = torch.device("cuda", 0)
n = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
segs = [int(x) for x in os.environ.get("SEGS", "30,14").split(",")]


def run(seg, how, steps=40):
    st = device_gaussian_state(n, n, dev)
    dt = 0.3 * swdemo.stable_dt(st, 1.0)
    cfg = swdemo.SWConfig(nx=n, ny=n, dt=dt, mode="fast")
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        sim = swdemo.Simulation(cfg, state=st, diagnostics=False, stream=s, tune=N.Tune(seg=seg))
        sim.advance(6)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        if how == "graph":
            rep = sim.capture(steps)
            rep()
            torch.cuda.synchronize()
            e0.record(s)
            rep()
            e1.record(s)
        elif how == "one_call":
            e0.record(s)
            sim.advance(steps)
            e1.record(s)
        else:
            evs = [torch.cuda.Event(enable_timing=True) for _ in range(steps)]
            e0.record(s)
            for k in range(steps):
                evs[k].record(s)
                sim.advance(1)
            e1.record(s)
        torch.cuda.synchronize()
    v = n * n * steps / (e0.elapsed_time(e1) / 1e3) / 1e9
    del sim, st
    torch.cuda.empty_cache()
    return round(v, 1)


for r in range(reps):
    for how in ("events", "one_call", "graph"):
        print(json.dumps({"rep": r, "how": how, **{f"seg{sg}": run(sg, how) for sg in segs}}), flush=True)
