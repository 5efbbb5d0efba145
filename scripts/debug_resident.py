#!/usr/bin/env python
"""Debug / timing helper for the resident time loop: compares the state
against the C oracle after each advance and prints per-step times."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402


def main():
    import torch
    from oracle import c_oracle
    from oracle import sw_oracle as so
    from paper_1107_2157_b200 import swdemo
    from paper_1107_2157_b200.field import DeviceField, Field

    def dev(H, U, V):
        return swdemo.SWState(*(DeviceField.from_field(Field.from_array(a, "f32")) for a in (H, U, V)))

    def host(st):
        return tuple(f.to_numpy() for f in (st.H, st.U, st.V))

    n = int(os.environ.get("N", "128"))
    H, U, V = so.random_state(n, n, "f32", seed=3)
    for variant in ("resident", "generic"):
        cfg = swdemo.SWConfig(nx=n, ny=n, dt=0.05, variant=variant)
        sim = swdemo.Simulation(cfg, state=dev(H, U, V), diagnostics=False)
        done = 0
        for k in (2, 10, 10, 1, 3):
            sim.advance(k)
            done += k
            want = c_oracle.run_fixed(H, U, V, done, 1.0, 1.0, 0.05)
            got = host(sim.state())
            diffs = [int(np.sum(g != w)) for g, w in zip(got, want)]
            where = [np.argwhere(g != w)[:2].tolist() for g, w in zip(got, want)]
            print(variant, "after", done, "steps: cells differing", diffs, where, flush=True)
    for n in (64, 128, 256):
        for mode in ("fast", "exact"):
            cfg = swdemo.SWConfig(nx=n, ny=n, dt=0.01, variant="resident", mode=mode)
            sim = swdemo.Simulation(cfg, state=swdemo.init_state(cfg), diagnostics=False)
            sim.advance(10)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            for k in (1, 10, 100, 1000):
                e0.record()
                sim.advance(k)
                e1.record()
                torch.cuda.synchronize()
                print(f"n={n} {mode} steps={k}: {e0.elapsed_time(e1) * 1e3 / k:.3f} us/step", flush=True)


if __name__ == "__main__":
    main()
