#!/usr/bin/env python
"""Grid-size sweep 128^2 .. 16384^2 on one GPU (BASELINE config 5b):
Gcell-updates/s and HBM GB/s of the fused step, with the time loop captured
in a CUDA graph so that small (launch-bound) grids measure the kernel, not
the host.  Grids up to ~2048^2 (6 buffers <= ~100 MB) are L2-resident.

    python scripts/grid_sweep.py [--mode fast|exact] [--out FILE]
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
    ap.add_argument("--mode", default="fast")
    ap.add_argument("--precision", default="f32")
    ap.add_argument("--out", default=None)
    ap.add_argument("--sizes", default="128,256,512,1024,2048,4096,8192,16384")
    ap.add_argument("--segs", default="0", help="comma list of TMA segment lengths to try (0 = auto)")
    ap.add_argument("--variants", default="auto", help="comma list of kernel variants (auto, tma, generic)")
    ap.add_argument("--warps", default="0", help="comma list of warps per TMA CTA (0 auto, 1, 2, 4)")
    ap.add_argument("--orders", default="0", help="comma list of TMA segment orders (fkc_sw_tune.order: 0 alternating, 1 bottom-up)")
    ap.add_argument("--pdl", default="1", help="comma list: programmatic dependent launch on (1) / off (0)")
    ap.add_argument("--tails", default="0:1", help="comma list of guided-segmentation settings rows:waves (fkc_sw_tune: 0 auto, -1 off)")
    args = ap.parse_args()
    import torch

    from bench import device_gaussian_state, peaks
    from paper_1107_2157_b200 import swdemo

    dev = torch.device("cuda", 0)
    peak, _ = peaks()
    rows = []
    from paper_1107_2157_b200 import _native as N
    todo = [(int(s), int(g), v, t, int(p), int(o), w) for s in args.sizes.split(",") for g in args.segs.split(",")
            for v in args.variants.split(",") for t in args.tails.split(",") for p in args.pdl.split(",")
            for o in args.orders.split(",") for w in args.warps.split(",")]
    for n, seg, variant, tail, pdl, order, warps in todo:
        if variant == "generic" and seg:
            continue
        tr, tw = (int(x) for x in tail.split(":"))
        tune = N.Tune(warps=int(warps), no_pdl=1 - pdl, order=order, seg=seg, tail_rows=tr, tail_waves=tw)
        st = device_gaussian_state(n, n, dev, precision=args.precision)
        dt = 0.3 * swdemo.stable_dt(st, 1.0)
        cfg = swdemo.SWConfig(nx=n, ny=n, dt=dt, mode=args.mode, variant=variant, precision=args.precision)
        stream = torch.cuda.Stream()
        with torch.cuda.stream(stream):
            sim = swdemo.Simulation(cfg, state=st, diagnostics=False, stream=stream, tune=tune)
            k = 20 if n >= 4096 else 200
            replay = sim.capture(k)
            for _ in range(2):
                replay()
            torch.cuda.synchronize()
            # ~2e9 cell-updates per point, at most 2000 steps: the fixed dt
            # (0.3 x the initial bound) stays stable that long; far longer
            # runs can go non-finite, and NaN arithmetic is not the timed path
            reps = max(2, min(int(2e9 / (n * n * k)), 2000 // k))
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            for _ in range(reps):
                replay()
            e1.record(stream)
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / (reps * k)
            # the same steps launched one by one (host launch path)
            e0.record(stream)
            sim.advance(k)
            e1.record(stream)
            torch.cuda.synchronize()
            ms_eager = e0.elapsed_time(e1) / k
        g = n * n / (ms / 1e3) / 1e9
        row = {"n": n, "seg": seg, "tail": tail, "pdl": pdl, "order": order, "warps": int(warps), "variant": variant, "mode": args.mode, "ms_per_step_graph": round(ms, 5), "gcell_s": round(g, 2),
               "hbm_gbs": round(24 * n * n / (ms / 1e3) / 1e9, 1), "frac_of_measured": round(24 * g / peak, 3),
               "ms_per_step_eager": round(ms_eager, 5),
               "regime": "L2-resident" if 6 * 4 * (n + 2) ** 2 <= 100e6 else "HBM",
               "launch_bound": n <= 512}
        rows.append(row)
        print(json.dumps(row), flush=True)
        del sim, st
        torch.cuda.empty_cache()
    if args.out:
        json.dump(rows, open(args.out, "w"), indent=1)


if __name__ == "__main__":
    main()
