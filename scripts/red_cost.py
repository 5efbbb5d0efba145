#!/usr/bin/env python
"""Cost of the fused reductions per grid size: us / step of fkc_sw_step
replayed from a CUDA graph (64 steps, A<->B) with reduction pointers
none / err / err+mass / err+maxima / all / all+cfl / all+cfl+dt_bound (the
bound in the reduced row's L2 line, as in the caller's 5-word slot rows, or
in another line: _far).

    python scripts/red_cost.py [--sizes 512,1024,2048,4096] [--modes fast,exact]
"""

from __future__ import annotations

import argparse
import ctypes
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--sizes", default="512,1024,2048,4096")
    ap.add_argument("--modes", default="fast,exact")
    ap.add_argument("--variant", default="auto")
    ap.add_argument("--combos", default="", help="comma list of combos to run (default all)")
    ap.add_argument("--seg", type=int, default=0, help="tune.seg (rows per segment, 0 = auto)")
    ap.add_argument("--warps", type=int, default=0, help="tune.warps (0 = auto)")
    ap.add_argument("--eager", type=int, default=0, help="N eager steps per combo instead of graph timing (profiling)")
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    import torch

    from paper_1107_2157_b200 import _native as N
    from paper_1107_2157_b200 import swdemo

    K = 64
    out = []
    for n in (int(s) for s in args.sizes.split(",")):
        for mode in args.modes.split(","):
            cfg = swdemo.SWConfig(nx=n, ny=n)
            a = swdemo.init_state(cfg).to_device()
            b = swdemo.SWState(a.H.empty_like(), a.U.empty_like(), a.V.empty_like(), a.g, a.dx, a.dy)
            dt = 0.3 * swdemo.stable_dt(a, 1.0)
            # row 0: the input bound far from the reduced row 4 (another L2
            # line); row 3: the bound in the reduced row's line (the caller's
            # 5-word rows i / i+1)
            slots = swdemo.ReductionSlots(8, a.H.storage.device)
            N.check(N.lib().fkc_sw_reduce_state(ctypes.byref(swdemo._grid(a.H)), a.H.ptr, a.U.ptr, a.V.ptr,
                                                a.dx, a.dy, a.g, ctypes.byref(slots.reduce_struct(0)),
                                                torch.cuda.current_stream().cuda_stream))
            N.check(N.lib().fkc_sw_reduce_state(ctypes.byref(swdemo._grid(a.H)), a.H.ptr, a.U.ptr, a.V.ptr,
                                                a.dx, a.dy, a.g, ctypes.byref(slots.reduce_struct(3)),
                                                torch.cuda.current_stream().cuda_stream))
            combos = {"none": {}, "err": dict(mass=False, maxima=False, cfl=False),
                      "err_mass": dict(maxima=False, cfl=False), "err_max": dict(mass=False, cfl=False),
                      "all": dict(cfl=False), "all_cfl": {}, "all_cfl_bound": {}, "all_cfl_bound_far": {}}
            row = {"n": n, "mode": mode, "seg": args.seg, "warps": args.warps}
            for name, kw in combos.items():
                if args.combos and name not in args.combos.split(","):
                    continue
                red = None if name == "none" else slots.reduce_struct(4, **kw)
                bound = (slots.addr(3, 3) if name == "all_cfl_bound" else
                         slots.addr(0, 3) if name == "all_cfl_bound_far" else None)
                sa = [swdemo._step_args(x, y, dt, "reflective", mode, args.variant, red, bound, 0.3)
                      for x, y in ((a, b), (b, a))]
                for i, s in enumerate(sa):
                    s.tune.parity = i
                    s.tune.seg = args.seg
                    s.tune.warps = args.warps
                s = torch.cuda.Stream()
                s.wait_stream(torch.cuda.current_stream())
                with torch.cuda.stream(s):
                    for i in range(4):
                        N.check(N.lib().fkc_sw_step(ctypes.byref(sa[i % 2]), s.cuda_stream))
                torch.cuda.synchronize()
                if args.eager:
                    with torch.cuda.stream(s):
                        for i in range(args.eager):
                            N.check(N.lib().fkc_sw_step(ctypes.byref(sa[i % 2]), s.cuda_stream))
                    torch.cuda.synchronize()
                    continue
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g, stream=s):
                    for i in range(K):
                        N.check(N.lib().fkc_sw_step(ctypes.byref(sa[i % 2]), s.cuda_stream))
                g.replay()
                torch.cuda.synchronize()
                best = 1e9
                for _ in range(3):
                    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    e0.record()
                    g.replay()
                    e1.record()
                    torch.cuda.synchronize()
                    best = min(best, e0.elapsed_time(e1) / K * 1e3)
                row[name] = round(best, 3)
                del g
            out.append(row)
            print(json.dumps(row), flush=True)
    if args.out:
        with open(args.out, "w") as f:
            json.dump({"note": __doc__.split("\n\n")[0], "rows": out}, f, indent=1)


if __name__ == "__main__":
    main()
