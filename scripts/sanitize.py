#!/usr/bin/env python
"""Small workloads for compute-sanitizer (memcheck / racecheck / synccheck /
initcheck): every kernel of the library on small grids -- TMA step (exact,
fast, with reductions, f32 / f64, both sweep directions, guided tail
segments, chained launches), generic step,
boundary fill, reductions, region ops, halo pack / unpack, and the fused
exchange on four local tiles with concurrent streams."""

import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import numpy as np
    import torch

    from oracle import sw_oracle as so
    from paper_1107_2157_b200 import _native as N
    from paper_1107_2157_b200 import refinterp, swdemo
    from paper_1107_2157_b200.decomp import run_local_decomposed
    from paper_1107_2157_b200.field import DeviceField, Field

    torch.cuda.set_device(0)
    # optional overrides (isolating a sanitizer report): FKC_SAN_PDL=0|1, FKC_SAN_WARPS=0|1|2|4
    base = N.Tune(no_pdl=1 - int(os.environ.get("FKC_SAN_PDL", "1")), warps=int(os.environ.get("FKC_SAN_WARPS", "0")))
    for prec in ("f32", "f64"):
        H, U, V = so.random_state(488, 70, prec, seed=3)
        st = swdemo.SWState(*(DeviceField.from_field(Field.from_array(a, prec)) for a in (H, U, V)))
        for mode in ("exact", "fast"):
            for variant in ("tma", "generic"):
                for alt in (0, 1):
                    t = base.copy()
                    t.no_alternate, t.seg = 1 - alt, 16
                    out = swdemo.advance(st, 0.05, "reflective", mode, variant, tune=t)
                    t2 = t.copy()
                    t2.parity = 1
                    swdemo.advance(out, 0.05, "periodic", mode, variant, tune=t2)
                    swdemo.advance(out, 0.05, "reflective", mode, variant, tune=t2, check=True)
        for mode in ("exact", "fast"):
            cfg = swdemo.SWConfig(nx=488, ny=70, steps=3, cfl_factor=0.5, precision=prec, mode=mode)
            swdemo.run(cfg)
            cfg = swdemo.SWConfig(nx=488, ny=70, steps=3, dt=0.05, precision=prec, mode=mode)
            swdemo.run(cfg)
        swdemo.reduce_state(st)
        swdemo.apply_boundary(st, "periodic")
        refinterp.region_cpy(st.H, (1, 0, 1, 1))
        refinterp.cshift(st.U, 1, 3)
    # guided segmentation (short tail segments) on a tall grid, chained steps
    # (programmatic dependent launch between them)
    H, U, V = so.random_state(128, 4000, "f32", seed=4)
    st = swdemo.SWState(*(DeviceField.from_field(Field.from_array(a, "f32")) for a in (H, U, V)))
    t = base.copy()
    t.tail_rows = 2
    for mode in ("exact", "fast"):
        out = swdemo.advance(st, 0.05, "reflective", mode, "tma", tune=t)
        t1 = t.copy()
        t1.parity = 1
        swdemo.advance(out, 0.05, "reflective", mode, "tma", tune=t1)
    for ex, conc in (("pack", False), ("fused", False), ("fused", True)):
        cfg = swdemo.SWConfig(nx=480, ny=256, dt=0.05, boundary="periodic", mode="fast")
        run_local_decomposed(cfg, 2, 2, 3, exchange=ex, concurrent=conc)
    # round 2 kernels: the resident cluster loop (DSMEM pushes, both buffers,
    # CFL slots), the persistent TMA loop (step counters, grid arrival), the
    # streamed host run (wave launches, staging unpack / pack on their own
    # streams, side-stream reduction)
    for prec in ("f32", "f64"):
        H, U, V = so.random_state(96, 70, prec, seed=5)
        for mode in ("exact", "fast"):
            for bc in ("reflective", "periodic"):
                for dt in (None, 0.05):
                    cfg = swdemo.SWConfig(nx=96, ny=70, steps=4, dt=dt, cfl_factor=0.5, precision=prec, mode=mode,
                                          boundary=bc, variant="resident")
                    st = swdemo.SWState(*(DeviceField.from_field(Field.from_array(a, prec)) for a in (H, U, V)))
                    swdemo.run(cfg, state=st)
                    cfg = swdemo.SWConfig(nx=96, ny=70, steps=4, dt=dt, cfl_factor=0.5, precision=prec, mode=mode,
                                          boundary=bc, variant="loop")
                    st = swdemo.SWState(*(DeviceField.from_field(Field.from_array(a, prec)) for a in (H, U, V)))
                    swdemo.run(cfg, state=st)
    H, U, V = so.random_state(256, 300, "f32", seed=6)
    for steps in (0, 3, 40):
        hst = swdemo.SWState(*(Field.from_array(a, "f32") for a in (H, U, V)))
        out = swdemo.SWState(*(Field.from_array(np.zeros_like(a), "f32") for a in (H, U, V)))
        cfg = swdemo.SWConfig(nx=256, ny=300, steps=steps, dt=0.05)
        swdemo._run_streamed(cfg, hst, out, band_rows=16)
    # chunked time loops (captured 32-step graphs, reduction ring, append
    # kernel): a CFL run and a fixed-dt run without reductions from an odd step
    H, U, V = so.random_state(488, 120, "f32", seed=7)
    for mode in ("exact", "fast"):
        st = swdemo.SWState(*(DeviceField.from_field(Field.from_array(a, "f32")) for a in (H, U, V)))
        swdemo.run(swdemo.SWConfig(nx=488, ny=120, steps=130, cfl_factor=0.5, mode=mode), state=st)
        st = swdemo.SWState(*(DeviceField.from_field(Field.from_array(a, "f32")) for a in (H, U, V)))
        sim = swdemo.Simulation(swdemo.SWConfig(nx=488, ny=120, dt=0.02, mode=mode), state=st, diagnostics=False)
        sim.advance(1)
        sim.advance(129)
    torch.cuda.synchronize()
    print("sanitize workload done")


if __name__ == "__main__":
    main()
