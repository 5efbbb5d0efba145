#!/usr/bin/env python
"""Cost of the decomposition machinery on ONE GPU (the gpurun pool has no
multi-GPU boxes): the 16384^2 headline grid split into P tiles that all run on
the same device -- the fused exchange with every tile on its own stream
(ordered only by the in-kernel mailboxes, what runs across GPUs), the fused
exchange on one stream, and the pack / copy / unpack baseline -- against the
undecomposed step.  Same total work, so Gcell/s close to the undecomposed
number means the exchange and the synchronisation cost little.

    python scripts/local_decomp_bench.py [--n 16384] [--steps 40] [--out FILE]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=16384)
    ap.add_argument("--steps", type=int, default=40)
    ap.add_argument("--mode", default="fast")
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    import torch

    from paper_1107_2157_b200 import swdemo
    from paper_1107_2157_b200.decomp import run_local_decomposed
    n = args.n
    dt = 0.3 / (9.8 * 1.4) ** 0.5
    cfg = swdemo.SWConfig(nx=n, ny=n, dt=dt, mode=args.mode)
    sim = swdemo.Simulation(cfg, diagnostics=False)
    sim.advance(5)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    sim.advance(args.steps)
    e1.record()
    torch.cuda.synchronize()
    base = e0.elapsed_time(e1) / args.steps
    del sim
    torch.cuda.empty_cache()
    rows = [{"tiles": "1x1", "exchange": "none (undecomposed)", "ms_per_step": round(base, 4),
             "gcell_s": round(n * n / base / 1e6, 1)}]
    print(json.dumps(rows[-1]), flush=True)
    for px, py in ((1, 2), (2, 2), (2, 4)):
        for exch, conc in (("fused", True), ("fused", False), ("pack", False)):
            t = []
            run_local_decomposed(cfg, px, py, args.steps, exchange=exch, concurrent=conc, warmup=5, timing=t)
            ms = t[0] / args.steps
            rows.append({"tiles": f"{px}x{py}", "exchange": exch + (" (concurrent streams, mailboxes)" if conc else
                                                                     " (one stream)" if exch == "fused" else
                                                                     " (pack / copy / unpack, one stream)"),
                         "ms_per_step": round(ms, 4), "gcell_s": round(n * n / ms / 1e6, 1),
                         "vs_undecomposed": round(base / ms, 3)})
            print(json.dumps(rows[-1]), flush=True)
            torch.cuda.empty_cache()
    if args.out:
        json.dump(rows, open(args.out, "w"), indent=1)


if __name__ == "__main__":
    main()
