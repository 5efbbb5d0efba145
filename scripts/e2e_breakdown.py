#!/usr/bin/env python
"""Where does the end-to-end time of swdemo.run go?  (host pinned state in,
200 steps with fused diagnostics, host pinned state out, 16384^2 f32)"""

from __future__ import annotations

import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch

    from bench import device_gaussian_state
    from paper_1107_2157_b200 import swdemo
    from paper_1107_2157_b200.field import Field
    from paper_1107_2157_b200.region import Extent
    n, steps = 16384, 200
    dev = torch.device("cuda", 0)
    st = device_gaussian_state(n, n, dev)
    dt = 0.3 * swdemo.stable_dt(st, 1.0)
    full = Extent(n + 2, n + 2)
    pin = [torch.empty((n + 2, n + 2), dtype=torch.float32, pin_memory=True) for _ in range(6)]
    for t, f in zip(pin, (st.H, st.U, st.V)):
        f.copy_to_host(t.numpy())
    del st
    torch.cuda.empty_cache()
    host_in = swdemo.SWState(*(Field(full, t.numpy(), "f32") for t in pin[:3]))
    host_out = swdemo.SWState(*(Field(full, t.numpy(), "f32") for t in pin[3:]))
    cfg = swdemo.SWConfig(nx=n, ny=n, steps=steps, dt=dt, mode="fast")
    out = {}
    for rep in range(2):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        dst = host_in.to_device()
        torch.cuda.synchronize()
        t1 = time.perf_counter()
        sim = swdemo.Simulation(cfg, state=dst, diagnostics=True)
        torch.cuda.synchronize()
        t2 = time.perf_counter()
        sim.advance(steps)
        torch.cuda.synchronize()
        t3 = time.perf_counter()
        res = sim.rows()
        t4 = time.perf_counter()
        res.state.to_host(host_out)
        t5 = time.perf_counter()
        out = {"h2d_s": t1 - t0, "sim_init_s": t2 - t1, "steps_s": t3 - t2, "rows_s": t4 - t3,
               "d2h_s": t5 - t4, "total_s": t5 - t0, "h2d_GBps": 3 * 4 * (n + 2) ** 2 / (t1 - t0) / 1e9,
               "d2h_GBps": 3 * 4 * (n + 2) ** 2 / (t5 - t4) / 1e9, "ms_per_step_with_diag": (t3 - t2) / steps * 1e3}
        del sim, dst, res
        torch.cuda.empty_cache()
    print(json.dumps({k: round(v, 4) for k, v in out.items()}))


if __name__ == "__main__":
    main()
