#!/usr/bin/env python
"""How far is fast mode from the f32 oracle, compared with how far the f32
oracle itself is from the f64 solution?  (exact kernels == the oracle bit for
bit, tested; so the GPU exact f32 / f64 runs stand in for the oracle.)"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import numpy as np
    from bench import device_gaussian_state
    from paper_1107_2157_b200 import swdemo
    import torch
    dev = torch.device("cuda", 0)
    out = []
    for n, steps in ((256, 100), (1024, 100), (4096, 50), (16384, 20)):
        res = {}
        for prec, mode in (("f32", "fast"), ("f32", "exact"), ("f64", "exact")):
            st = device_gaussian_state(n, n, dev, precision=prec)
            dt = 0.3 * swdemo.stable_dt(device_gaussian_state(n, n, dev, precision="f32"), 1.0)
            cfg = swdemo.SWConfig(nx=n, ny=n, dt=dt, mode=mode, precision=prec)
            sim = swdemo.Simulation(cfg, state=st, diagnostics=False)
            sim.advance(steps)
            s = sim.state()
            res[(prec, mode)] = [getattr(s, f).data[1:-1, 1:-1].double().cpu().numpy() for f in "HUV"]
            del sim, st, s
            torch.cuda.empty_cache()
        row = {"n": n, "steps": steps}
        for f, k in zip("HUV", range(3)):
            ref = res[("f64", "exact")][k]
            sc = np.max(np.abs(ref))
            row[f"{f}_fast_vs_exact32"] = float(np.max(np.abs(res[("f32", "fast")][k] - res[("f32", "exact")][k])) / sc)
            row[f"{f}_exact32_vs_f64"] = float(np.max(np.abs(res[("f32", "exact")][k] - ref)) / sc)
            row[f"{f}_fast_vs_f64"] = float(np.max(np.abs(res[("f32", "fast")][k] - ref)) / sc)
        print(json.dumps(row), flush=True)
        out.append(row)
    if len(sys.argv) > 1:
        json.dump(out, open(sys.argv[1], "w"), indent=1)


if __name__ == "__main__":
    main()
