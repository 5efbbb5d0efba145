#!/usr/bin/env python
"""Benchmark of the shallow-water hot path (BASELINE.json metric:
Gcell-updates/s and HBM GB/s vs roofline).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

A *step* is one Lax-Wendroff update of the whole grid (one launch of the
fused sm_100a step kernel: faces + update + boundary halos).  Workload at
N=1: BASELINE config 3, 16384^2 f32, reflective, fixed dt = 0.3 *
stable_dt(initial state); N>1: weak scaling,
16384^2 cells per GPU, 2-D decomposed with a one-cell halo exchange per
step.  The 6.4 GB working set is ~50x the 126 MB L2, so no L2 flush is
needed between steps.  Prints ONE JSON line on rank 0.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

BYTES_PER_CELL = {"f32": 24, "f64": 48}      # read H,U,V + write oH,oU,oV
FALLBACK_HBM_GBS = 6650.0
FAST_RTOL = 2e-5          # fast-mode tolerance vs the oracle, 256^2 / 1024^2 (tests/test_gpu_parity.py)
FAST_PARITY = ("fast (FMA + approximate reciprocals), at THIS size (16384^2, 20 steps; "
               "profiles/r01/fast_accuracy.json): normwise distance to the bit-exact f32 oracle 7.4e-4 on hu, "
               "6.7e-4 on hv -- the f32 oracle itself is 6.2e-4 from the f64 solution, and fast mode's distance "
               "to f64 is within 1.1x of that (tests/test_gpu_parity.py); rtol 2e-5 vs the f32 oracle at "
               "256^2 / 1024^2. The bit-exact mode is timed beside it (other_mode)")


METRIC = "Gcell-updates/s (shallow-water step)"


def workload(n, world=1, precision="f32"):
    """The workload string both arms report (BASELINE configs 3 / 5)."""
    fp = "fp32" if precision == "f32" else "fp64"
    if world == 1:
        return f"shallow-water {n}x{n} {fp}, reflective, fixed dt=0.3*stable_dt (BASELINE config 3)"
    from paper_1107_2157_b200.decomp import choose_grid
    px, py = choose_grid(world)
    return (f"shallow-water {n}x{n} {fp} per GPU ({px * n}x{py * n} global, 2-D decomposed {px}x{py}), "
            f"reflective, fixed dt=0.3*stable_dt (BASELINE config 5, weak scaling)")


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured"
    return FALLBACK_HBM_GBS, "fallback"


class ClockSampler:
    """NVML sampling of SM clock and throttle reasons during the timed region."""

    def __init__(self, index=0, period=0.004):
        self.samples, self.reasons = [], set()
        self.period, self.index = period, index
        self.ok = False
        self._stop = threading.Event()
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception:
            self.max_mhz = None

    def _loop(self):
        nv = self.nv
        names = {
            "hw_slowdown": getattr(nv, "nvmlClocksEventReasonHwSlowdown", 0x8),
            "sw_thermal_slowdown": getattr(nv, "nvmlClocksEventReasonSwThermalSlowdown", 0x20),
            "hw_thermal_slowdown": getattr(nv, "nvmlClocksEventReasonHwThermalSlowdown", 0x40),
            "sw_power_cap": getattr(nv, "nvmlClocksEventReasonSwPowerCap", 0x4),
        }
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for k, bit in names.items():
                    if r & bit:
                        self.reasons.add(k)
            except Exception:
                pass
            time.sleep(self.period)

    def __enter__(self):
        if self.ok:
            self.t = threading.Thread(target=self._loop, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        if self.ok:
            self._stop.set()
            self.t.join()

    def summary(self):
        if not self.ok or not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["nvml unavailable"]}
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


# ---------------------------------------------------------------------------
# CPU reference (oracle port) -- only used for the cpu_baseline / --impl reference legs
# ---------------------------------------------------------------------------

def cpu_reference_run(n, steps, warmup, threads=None, budget_s=None):
    """The reference CPU path of the step timed on the host cores: the C
    restatement of the reference algorithm (oracle/sw_oracle.c, DSL op
    order, all `threads` host threads) on the FULL n x n workload -- the
    same grid, init and dt as the GPU arm.  `warmup` untimed steps (page
    faults of the fresh buffers, thread start-up), then `steps` timed steps
    (or as many as fit in `budget_s` seconds, at least 2); the per-step
    median is reported.  Both CPU legs (our arm's cpu_baseline and
    --impl reference) use this one function, so they measure the same thing."""
    from oracle import c_oracle
    from oracle import sw_oracle as so
    threads = threads or len(os.sched_getaffinity(0))
    H, U, V = so.init_state(n, n, "f32")
    dt = 0.3 * so.stable_dt(H, U, V, 1.0, 1.0)
    a = (H, U, V)
    b = tuple(np.empty_like(x) for x in a)
    for _ in range(warmup):
        c_oracle.step(*a, 1.0, 1.0, dt, out=b, threads=threads)
        a, b = b, a
    times = []
    t_start = time.perf_counter()
    while len(times) < steps and (budget_s is None or len(times) < 2 or time.perf_counter() - t_start < budget_s):
        t0 = time.perf_counter()
        c_oracle.step(*a, 1.0, 1.0, dt, out=b, threads=threads)
        times.append(time.perf_counter() - t0)
        a, b = b, a
    med = statistics.median(times)
    return {"value": n * n / med / 1e9, "unit": "Gcell-updates/s", "cores": threads, "kind": "port",
            "sample": f"C restatement of the reference step (oracle/sw_oracle.c, DSL op order, -O2, no FMA) "
                      f"on the full {n}x{n} workload, {warmup} warm-up steps, median of {len(times)} timed steps, "
                      f"{threads} host threads", "ms_per_step": med * 1e3, "steps_timed": len(times),
            "warmup": warmup}


def cpu_reference_subprocess(n, steps, warmup, budget_s=None):
    """cpu_reference_run in a fresh interpreter (no CUDA context, no pinned
    buffers, no torch threads): the same conditions as the --impl
    reference arm, which the driver runs as its own process."""
    import subprocess
    code = ("import json, sys; sys.path.insert(0, %r); import bench; "
            "print(json.dumps(bench.cpu_reference_run(%d, %d, %d, budget_s=%r)))" % (ROOT, n, steps, warmup, budget_s))
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=900)
    if r.returncode != 0:
        raise RuntimeError(r.stderr[-500:])
    return json.loads(r.stdout.strip().splitlines()[-1])


def numpy_sample(n, rows):
    """The numpy restatement (single-threaded, like the reference) on a small slab."""
    from oracle import sw_oracle as so
    H, U, V = so.init_state(n, rows, "f32")
    dt = 0.3 * so.stable_dt(H, U, V, 1.0, 1.0)
    t0 = time.perf_counter()
    so.step(H, U, V, 1.0, 1.0, dt)
    t = time.perf_counter() - t0
    return {"value": n * rows / t / 1e9, "cores": 1, "sample": f"numpy oracle, 1 step on {n}x{rows}"}


# ---------------------------------------------------------------------------
# device helpers
# ---------------------------------------------------------------------------

def device_gaussian_state(n_x, n_y, device, x_off=0, y_off=0, n_glob=None, boundary="reflective",
                          precision="f32", amplitude=0.4):
    """Gaussian-hump initial state built on the device (setup only)."""
    import torch
    from paper_1107_2157_b200 import swdemo
    from paper_1107_2157_b200.field import DeviceField
    from paper_1107_2157_b200.region import Extent
    ng_x, ng_y = n_glob if n_glob else (n_x, n_y)
    full = Extent(n_x + 2, n_y + 2)
    H, U, V = (DeviceField(full, precision, device, fill=0.0) for _ in range(3))
    xs = (torch.arange(n_x, dtype=torch.float64, device=device) + x_off + 0.5) - ng_x / 2.0
    ys = (torch.arange(n_y, dtype=torch.float64, device=device) + y_off + 0.5) - ng_y / 2.0
    w = ng_x / 8.0
    for r0 in range(0, n_y, 2048):          # chunk to bound f64 temporaries
        r1 = min(n_y, r0 + 2048)
        h = 1.0 + amplitude * torch.exp(-(xs[None, :] ** 2 + ys[r0:r1, None] ** 2) / (w * w))
        H.data[1 + r0:1 + r1, 1:-1] = h.to(torch.float32 if precision == "f32" else torch.float64)
    st = swdemo.SWState(H, U, V)
    swdemo.apply_boundary(st, boundary)
    return st


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--n", "--grid-n", dest="n", type=int, default=16384, help="cells per side (per GPU)")
    ap.add_argument("--global-n", type=int, default=0,
                    help="N>1 strong scaling: a fixed global grid of this many cells per side "
                         "(BASELINE config 4: 32768) instead of --grid-n per GPU")
    ap.add_argument("--mode", default="fast", choices=["exact", "fast"],
                    help="fast: FMA + approximate reciprocals, as accurate as the f32 oracle (headline); "
                         "exact: bit-identical to the oracle")
    ap.add_argument("--variant", default="auto", choices=["auto", "tma", "generic"])
    ap.add_argument("--precision", default="f32", choices=["f32", "f64"],
                    help="field precision (f64: 48 B/cell; the headline is f32, BASELINE configs)")
    ap.add_argument("--seg", type=int, default=0, help="TMA kernel rows per CTA segment (0 = auto)")
    ap.add_argument("--warps", type=int, default=0, choices=[0, 1, 2, 4], help="warps per TMA CTA (0 = auto)")
    ap.add_argument("--alt", type=int, default=1, choices=[0, 1],
                    help="TMA kernel: odd segments sweep top-down (L2 reuse of shared halo rows)")
    ap.add_argument("--transport", default="auto", choices=["auto", "peer", "nccl"],
                    help="N>1 halo exchange: peer = fused into the step kernel over NVLink peer memory "
                         "(CUDA IPC + mailbox flags); nccl = pack + NCCL send/recv + unpack (baseline); "
                         "auto = peer, falling back to nccl on every rank if the IPC setup fails")
    ap.add_argument("--diag", default="none", choices=["none", "diag", "cfl"],
                    help="fused reductions in the timed steps: none; diag = mass, max|hu|, max|hv|, error word "
                         "(run()'s per-step diagnostics); cfl = diag + the CFL bound, dt recomputed on device "
                         "every step (SPEC.md:529-537 run)")
    ap.add_argument("--amplitude", type=float, default=0.4,
                    help="Gaussian hump amplitude of the synthetic state (0: a lake at rest; profiling only)")
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-other", action="store_true", help="skip the other-mode timing (profiling runs)")
    ap.add_argument("--no-extras", action="store_true",
                    help="skip the BASELINE config 2 (4096^2 x 1000 steps) and grid-sweep (config 5b) lines")
    ap.add_argument("--sweep", default="16,32,64,128,256,512,1024,2048,4096,8192,16384",
                    help="grid sizes of the config-5b sweep reported under extras")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    n = args.n

    if args.impl == "reference":
        if rank != 0:
            return 0
        cores = len(os.sched_getaffinity(0))
        r = cpu_reference_run(n, args.steps, args.warmup, threads=cores)
        line = {"metric": METRIC, "value": r["value"], "unit": "Gcell-updates/s",
                "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
                "ms_per_step": r["ms_per_step"], "higher_is_better": True, "scaling": "weak",
                "vs_baseline": None, "dtype": "f32", "data": "synthetic (Gaussian hump)",
                "config": {"workload": workload(n, 1), "parallelism": f"{cores} host threads",
                           "sample": f"the full {n}x{n} grid every step (same grid, init and dt as the GPU arm); "
                                     "per-step median"},
                "impl": "reference",
                "cpu_baseline": {"value": r["value"], "unit": "Gcell-updates/s", "cores": cores,
                                 "kind": "port", "sample": r["sample"]},
                "e2e": {"value": r["value"], "unit": "Gcell-updates/s", "h2d_bytes_per_step": 0,
                        "d2h_bytes_per_step": 0}}
        print(json.dumps(line))
        return 0

    import torch
    if world > 1:
        return multi_gpu_main(args, rank, world)

    from paper_1107_2157_b200 import _native as N
    from paper_1107_2157_b200 import swdemo

    torch.cuda.set_device(0)
    dev = torch.device("cuda", 0)
    tune = N.Tune(seg=args.seg, warps=args.warps, no_alternate=1 - args.alt)
    st = device_gaussian_state(n, n, dev, precision=args.precision, amplitude=args.amplitude)
    dt0 = swdemo.stable_dt(st, 1.0)
    dt = 0.3 * dt0
    r = time_steps(st, n, dt, args.mode, args.variant, args.steps, args.warmup, sample_clocks=True,
                   precision=args.precision, diag=args.diag, tune=tune)
    total_ms, per_launch, clocks = r["total_ms"], r["per_launch"], r["clocks"]
    ms_step = total_ms / args.steps
    cells = n * n
    value = cells * args.steps / (total_ms / 1e3) / 1e9
    avg_launch_ms = sum(per_launch) / len(per_launch)
    bytes_launch = BYTES_PER_CELL[args.precision] * cells
    achieved = bytes_launch / (avg_launch_ms / 1e3) / 1e9
    peak, peak_src = peaks()
    other_line = None
    if not args.no_other:
        other = "exact" if args.mode == "fast" else "fast"
        st2 = device_gaussian_state(n, n, dev, precision=args.precision)
        r2 = time_steps(st2, n, dt, other, args.variant, min(args.steps, 20), 10, precision=args.precision)
        del st2
        other_line = {"mode": other, "value": round(cells * r2["steps"] / (r2["total_ms"] / 1e3) / 1e9, 3),
                      "ms_per_step": round(r2["total_ms"] / r2["steps"], 5), "steps": r2["steps"],
                      "parity": "bit-exact vs oracle" if other == "exact" else FAST_PARITY}

    traffic = None
    tp = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tp):
        try:
            t = json.load(open(tp))
            key = f"{args.mode}_{n}" + ("" if args.precision == "f32" else "_f64")
            traffic = t.get(key)
        except Exception:
            traffic = None

    line = {
        "metric": METRIC, "value": round(value, 3), "unit": "Gcell-updates/s",
        "n_gpus": 1, "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms_step, 5),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": args.precision,
        "data": "synthetic (Gaussian hump h=1+0.4exp(-r^2/(n/8)^2), hu=hv=0)",
        "config": {"workload": workload(n, 1, args.precision),
                   "precision": args.precision, "diagnostics": args.diag,
                   "mode": args.mode, "parity": "bit-exact vs oracle" if args.mode == "exact" else FAST_PARITY,
                   "variant": args.variant, "schedule": tma_schedule(n, args), "global_batch": cells,
                   "parallelism": "single GPU",
                   "l2": f"working set {BYTES_PER_CELL[args.precision] * (n + 2) * (n + 2) / 1e9:.1f} GB >> "
                         "126 MB L2 (no flush needed)"},
        "hbm_gbs": round(achieved, 1),
        "roofline": {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                     "frac": round(achieved / peak, 4), "peak_source": peak_src, "traffic": traffic,
                     "algorithmic_bytes_per_launch": bytes_launch, "avg_launch_ms": round(avg_launch_ms, 5),
                     "frac_of_nominal_8TBs": round(achieved / 8000.0, 4),
                     **({"note": "achieved exceeds the measured peak: that figure is a torch copy_ "
                                 "(MEASURED_PEAKS.json); this kernel's DRAM traffic (ncu, `traffic`) equals its "
                                 "algorithmic bytes, so it streams HBM faster than that copy -- see "
                                 "frac_of_nominal_8TBs"} if achieved > peak else {})},
        "gpu_launches": args.steps,
        "clocks": clocks.summary(),
        "other_mode": other_line,
    }

    if not args.no_e2e and args.precision == "f32":
        line["e2e"] = e2e_run(n, dt, args, dev)
    if not args.no_extras and args.precision == "f32" and n == 16384:
        line["extras"] = extras_run(args, dev)
    if not args.no_cpu:
        try:
            # same function and policy as --impl reference (warm-up, full grid,
            # per-step median), bounded to ~15 s of CPU work
            cb = cpu_reference_subprocess(n, args.steps, args.warmup, budget_s=15.0)
            cb["numpy_1core"] = numpy_sample(n, 256)
            line["cpu_baseline"] = cb
        except Exception as e:  # pragma: no cover
            line["cpu_baseline"] = {"value": None, "error": str(e)}
    print(json.dumps(line))
    return 0


def tma_schedule(n, args):
    """The TMA kernel's launch schedule for this run (fkc_tma_plan: the
    host-side plan the library uses), or None for the generic kernel."""
    import ctypes
    from paper_1107_2157_b200 import _native as N
    if args.variant == "generic" or (args.variant == "auto" and n * n < (5 << 17)):
        return None
    g = N.Grid(n, n, n + 32, N.F32 if args.precision == "f32" else N.F64, 0)
    out = (ctypes.c_int * 7)()
    red = {"none": 0, "diag": 1, "cfl": 2}[args.diag]
    tune = N.Tune(seg=args.seg, warps=args.warps)
    if N.lib().fkc_tma_plan(ctypes.byref(g), N.MODE_FAST if args.mode == "fast" else N.MODE_EXACT, red,
                            ctypes.byref(tune), out):
        return None
    w, bands, nseg, seg, tail, jt, cps = list(out)
    return {"kernel": "sw_step_tma", "warps_per_cta": w, "ctas": bands * nseg, "ctas_per_sm": cps,
            "segment_rows": seg, "tail_segment_rows": tail, "order": "alternating per step", "pdl": True}


def time_steps(st, n, dt, mode, variant, steps, warmup, sample_clocks=False, precision="f32", diag="none",
               tune=None):
    """K steps of the fused step kernel, CUDA events on the launching stream
    (one event pair per launch: the step kernel is the only launch)."""
    import torch
    from paper_1107_2157_b200 import swdemo
    cfg = swdemo.SWConfig(nx=n, ny=n, steps=steps + warmup, dt=None if diag == "cfl" else dt, mode=mode,
                          variant=variant, precision=precision, cfl_factor=0.3)
    stream = torch.cuda.Stream()
    with torch.cuda.stream(stream):
        sim = swdemo.Simulation(cfg, state=st, diagnostics=diag != "none", stream=stream, tune=tune)
        sim.advance(warmup)
        torch.cuda.synchronize()
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(steps + 1)]
        t_start, t_end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        clocks = ClockSampler(0) if sample_clocks else None
        if clocks:
            clocks.__enter__()
        torch.cuda.synchronize()
        t_start.record(stream)
        for k in range(steps):
            ev[k].record(stream)
            sim.advance(1)
        ev[steps].record(stream)
        t_end.record(stream)
        torch.cuda.synchronize()
        if clocks:
            clocks.__exit__(None, None, None)
    if diag != "none":
        sim.rows()                      # raises NonfiniteValue / NonPositiveDepth from the error words
    fin = sim.state()
    assert bool(torch.isfinite(fin.H.data).all().item()), "non-finite state after the timed run"
    return {"total_ms": t_start.elapsed_time(t_end), "steps": steps,
            "per_launch": [ev[k].elapsed_time(ev[k + 1]) for k in range(steps)], "clocks": clocks}


def extras_run(args, dev):
    """BASELINE config 2 (4096^2, 1000 steps, one native call per mode, after
    10 warm-up steps) and the config-5b grid sweep 16^2 .. 16384^2 -- the
    paper's Table 1 widths 16 .. 4096 and beyond -- (fast
    mode; each size's steps replayed from one CUDA graph: the small end runs
    the resident cluster loop inside it), device-timed with CUDA events.
    Reported beside the headline, not as it."""
    import torch
    from paper_1107_2157_b200 import swdemo
    out = {}
    c2 = {}
    for mode in ("fast", "exact"):
        st = device_gaussian_state(4096, 4096, dev)
        dt = 0.3 * swdemo.stable_dt(st, 1.0)
        cfg = swdemo.SWConfig(nx=4096, ny=4096, steps=1010, dt=dt, mode=mode)
        stream = torch.cuda.Stream()
        with torch.cuda.stream(stream):
            sim = swdemo.Simulation(cfg, state=st, diagnostics=False, stream=stream)
            sim.advance(10)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            sim.advance(1000)
            e1.record(stream)
            torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        assert bool(torch.isfinite(sim.state().H.data).all().item())
        c2[mode] = {"value": round(4096 * 4096 * 1000 / (ms / 1e3) / 1e9, 2), "ms_total": round(ms, 3),
                    "us_per_step": round(ms, 3)}
        del sim, st
    out["config2_4096sq_1000_steps"] = {"unit": "Gcell-updates/s", **c2,
                                        "how": "one fkc_sw_advance_n call of 1000 steps, CUDA events"}
    # BASELINE config 4's one-GPU base: 32768^2 (25.8 GB of state), fast mode
    try:
        n4 = 32768
        st = device_gaussian_state(n4, n4, dev)
        dt = 0.3 * swdemo.stable_dt(st, 1.0)
        cfg = swdemo.SWConfig(nx=n4, ny=n4, steps=25, dt=dt, mode="fast")
        stream = torch.cuda.Stream()
        with torch.cuda.stream(stream):
            sim = swdemo.Simulation(cfg, state=st, diagnostics=False, stream=stream)
            sim.advance(5)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            sim.advance(20)
            e1.record(stream)
            torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        out["config4_32768sq_1gpu"] = {"unit": "Gcell-updates/s", "value": round(n4 * n4 * 20 / (ms / 1e3) / 1e9, 2),
                                       "us_per_step": round(ms / 20 * 1e3, 1),
                                       "how": "20 steps after 5 warm-up, one fkc_sw_advance_n call, CUDA events; "
                                              "the strong-scaling base of BASELINE config 4"}
        del sim, st
        torch.cuda.empty_cache()
    except Exception as e:  # noqa: BLE001 - an extra, reported not fatal
        out["config4_32768sq_1gpu"] = {"unavailable": str(e)[:120]}
    sweep = []
    for n in (int(x) for x in args.sweep.split(",") if x):
        st = device_gaussian_state(n, n, dev)
        dt = 0.3 * swdemo.stable_dt(st, 1.0)
        cfg = swdemo.SWConfig(nx=n, ny=n, dt=dt, mode="fast")
        stream = torch.cuda.Stream()
        with torch.cuda.stream(stream):
            sim = swdemo.Simulation(cfg, state=st, diagnostics=False, stream=stream)
            k = 20 if n >= 8192 else 200
            replay = sim.capture(k)
            replay()
            torch.cuda.synchronize()
            reps = max(2, min(50, int(1e9 / (n * n * k))))
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            for _ in range(reps):
                replay()
            e1.record(stream)
            torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / (reps * k)
        sweep.append({"n": n, "us_per_step": round(ms * 1e3, 3), "value": round(n * n / (ms / 1e3) / 1e9, 2),
                      "hbm_equiv_gbs": round(24 * n * n / (ms / 1e3) / 1e9, 1),
                      "regime": ("resident (whole loop on chip)" if n <= 224 else "launch-bound") if n <= 512
                      else ("L2-resident" if n <= 2048 else "HBM")})
        del sim, st
        torch.cuda.empty_cache()
    out["sweep_fast"] = {"unit": "Gcell-updates/s", "rows": sweep,
                         "how": "Simulation.capture(k) CUDA graph replays, CUDA events, fixed dt"}
    return out


def res_streamed(n, args) -> bool:
    """Whether swdemo.run takes the streamed host path for the e2e call."""
    from paper_1107_2157_b200 import swdemo
    return n * n >= swdemo.STREAM_MIN_CELLS and args.variant in ("auto", "tma") and n % 4 == 0


def e2e_run(n, dt, args, dev):
    """Same metric through the public API with HOST buffers, at the
    commanded --steps: the initial state is copied from pinned host memory,
    ``swdemo.run`` advances it with per-step fused diagnostics (mass,
    max|hu|, max|hv|, error word; each step's row streamed back), and the
    final state comes back to pinned host memory -- all inside the timed
    region.  One untimed run of the same call first (a warm process: CUDA
    context, allocator, tensor maps), then one timed run; a labelled
    200-step run is reported beside it (the copies amortised over more
    steps)."""
    import torch
    from paper_1107_2157_b200 import swdemo
    from paper_1107_2157_b200.field import Field
    from paper_1107_2157_b200.region import Extent
    st = device_gaussian_state(n, n, dev)
    full = Extent(n + 2, n + 2)
    pinned = []
    for f in (st.H, st.U, st.V):
        t = torch.empty((n + 2, n + 2), dtype=torch.float32, pin_memory=True)
        t.copy_(f.data)
        pinned.append(t)
    del st
    torch.cuda.empty_cache()
    host_state = swdemo.SWState(*(Field(full, t.numpy(), "f32") for t in pinned))
    out_pinned = [torch.empty((n + 2, n + 2), dtype=torch.float32, pin_memory=True) for _ in range(3)]
    host_out = swdemo.SWState(*(Field(full, t.numpy(), "f32") for t in out_pinned))

    def timed(steps):
        cfg = swdemo.SWConfig(nx=n, ny=n, steps=steps, dt=dt, mode=args.mode, variant=args.variant)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        res = swdemo.run(cfg, state=host_state, out=host_out)
        el = time.perf_counter() - t0
        return n * n * steps / el / 1e9, el, res

    timed(min(args.steps, 3))                     # warm-up call (untimed)
    value, el, res = timed(args.steps)
    long_value, long_el, _ = timed(200)
    state_bytes = 3 * 4 * (n + 2) * (n + 2)
    return {"value": round(value, 3), "unit": "Gcell-updates/s", "steps": args.steps,
            "seconds": round(el, 4),
            "h2d_bytes_per_step": round(state_bytes / args.steps, 1),
            "d2h_bytes_per_step": round((state_bytes + 40 * (args.steps + 1)) / args.steps, 1),
            "api": "paper_1107_2157_b200.swdemo.run(cfg, state=<host pinned Fields>, out=<host pinned Fields>)",
            "path": "streamed host run (fkc_sw_run_host): 1-D staged band copies (upload, pack and download streams) overlap the "
                    "steps, which run band by band as a wavefront (one multi-band launch per band period) for the "
                    "first / last up to 32 steps" if res_streamed(n, args) else "device loop (fkc_sw_advance_n)",
            "diagnostics": "per-step mass/max|hu|/max|hv|/error word fused in the step kernel; the 40-byte "
                           "rows copied device->host with the run (streamed run: once per wavefront phase)",
            "warm": "one untimed run() of the same call first (CUDA context, allocator, tensor maps)",
            "final_mass": res.rows[-1][3],
            "long_run_200_steps": {"value": round(long_value, 3), "seconds": round(long_el, 4),
                                   "note": "same call with steps=200 (host copies amortised over 10x the steps)"}}


# ---------------------------------------------------------------------------
# N > 1 (torchrun): weak scaling 16384^2 cells per GPU, or strong scaling
# ---------------------------------------------------------------------------

def multi_gpu_main(args, rank: int, world: int) -> int:
    """N > 1 (torchrun, one process per GPU): the decomposed run of
    paper_1107_2157_b200.decomp -- weak scaling (BASELINE config 5) or, with
    --global-n, strong scaling (config 4)."""
    import json
    import time

    import torch
    import torch.distributed as dist

    from paper_1107_2157_b200 import swdemo
    from paper_1107_2157_b200.decomp import CartGrid, DistributedSimulation, choose_grid, gaussian_tile

    local = int(os.environ.get("LOCAL_RANK", rank))
    # FKC_BENCH_ONE_DEVICE=1: every rank on cuda:0 with gloo host collectives
    # -- exercises the N>1 code path (IPC peer memory, mailboxes) on a
    # one-GPU box; its timings are meaningless (time-sliced contexts)
    one_dev = os.environ.get("FKC_BENCH_ONE_DEVICE") == "1"
    if one_dev:
        local = 0
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if one_dev:
        dist.init_process_group("gloo")
    else:
        dist.init_process_group("nccl", device_id=dev)
    px, py = choose_grid(world)
    n = args.n
    strong = bool(getattr(args, "global_n", 0))
    # weak scaling (default): n^2 cells per GPU; strong: a fixed global grid
    grid = CartGrid(px, py, args.global_n, args.global_n, "reflective") if strong else \
        CartGrid(px, py, px * n, py * n, "reflective")
    # fixed dt = 0.3 * stable_dt of the initial global state (h max 1.4, u = v = 0)
    dt = 0.3 * 1.0 / float(np.sqrt(np.float32(9.8) * np.float32(1.4)))
    cfg = swdemo.SWConfig(nx=grid.NX, ny=grid.NY, dt=dt, mode=args.mode, variant=args.variant)
    stream = torch.cuda.Stream(dev)
    with torch.cuda.stream(stream):
        sim = DistributedSimulation(cfg, grid, rank, dev, stream=stream, transport=args.transport)
        sim.advance(args.warmup)
        torch.cuda.synchronize()
        dist.barrier()
        clocks = ClockSampler(local) if rank == 0 else None
        if clocks:
            clocks.__enter__()
        t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0.record(stream)
        sim.advance(args.steps)
        t1.record(stream)
        torch.cuda.synchronize()
        if clocks:
            clocks.__exit__(None, None, None)
        dist.barrier()
    ms = torch.tensor([t0.elapsed_time(t1)], device="cpu" if one_dev else dev)
    dist.all_reduce(ms, op=dist.ReduceOp.MAX)
    total_ms = float(ms.item())
    launches = sim._launches_per_step()
    transport, fallback = sim.transport, sim.fallback_reason
    sim.close()
    del sim
    torch.cuda.empty_cache()
    e2e = None if getattr(args, "no_e2e", False) else multi_gpu_e2e(args, cfg, grid, rank, world, dev, one_dev)
    cells = grid.NX * grid.NY
    value = cells * args.steps / (total_ms / 1e3) / 1e9
    if rank == 0:
        peak, src = peaks()
        per_gpu_gbs = BYTES_PER_CELL["f32"] * (cells / world) * args.steps / (total_ms / 1e3) / 1e9
        line = {"metric": METRIC, "value": round(value, 3),
                "unit": "Gcell-updates/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
                "ms_per_step": round(total_ms / args.steps, 5), "higher_is_better": True,
                "scaling": "strong" if strong else "weak",
                "vs_baseline": None, "dtype": "f32", "data": "synthetic (Gaussian hump)",
                "config": {"workload": (f"shallow-water {grid.NX}x{grid.NY} fp32 2-D decomposed {px}x{py}, "
                                        "reflective, fixed dt=0.3*stable_dt (BASELINE config 4, strong scaling)")
                           if strong else workload(n, world),
                           "exchange": "one-cell halo exchange per step " +
                                       ("fused into the step kernel (NVLink peer stores + mailbox flags)"
                                        if transport == "peer" else "(pack + NCCL send/recv + unpack)"),

                           "global": f"{grid.NX}x{grid.NY}", "mode": args.mode, "parallelism": f"domain{px}x{py}"},
                "roofline": {"bound": "hbm", "achieved": round(per_gpu_gbs, 1), "peak": peak, "unit": "GB/s",
                             "frac": round(per_gpu_gbs / peak, 4), "peak_source": src,
                             "note": "per-GPU HBM rate of the whole step incl. exchange", "traffic": None},
                "gpu_launches": args.steps * launches,
                "clocks": clocks.summary()}
        if e2e is not None:
            line["e2e"] = e2e
        line["config"]["transport"] = transport
        if fallback:
            line["config"]["transport_fallback"] = fallback[:300]
        print(json.dumps(line))
    dist.destroy_process_group()
    return 0


def multi_gpu_e2e(args, cfg, grid, rank: int, world: int, dev, one_dev: bool):
    """End to end through the public API at N GPUs: every rank's tile
    starts in pinned host memory, DistributedSimulation uploads it, sets up
    the exchange, advances `steps` steps and the final tile is copied back;
    wall clock between two barriers, max over ranks."""
    import time

    import torch
    import torch.distributed as dist

    from paper_1107_2157_b200 import swdemo
    from paper_1107_2157_b200.decomp import DistributedSimulation, gaussian_tile
    from paper_1107_2157_b200.field import Field
    from paper_1107_2157_b200.region import Extent
    t = grid.tile(rank)
    full = Extent(t.nx + 2, t.ny + 2)
    steps = args.steps
    pin = [torch.zeros((t.ny + 2, t.nx + 2), dtype=torch.float32, pin_memory=True) for _ in range(6)]
    pin[0][1:-1, 1:-1] = torch.from_numpy(gaussian_tile(grid, rank, "f32", cfg.dx, cfg.dy, cfg.base,
                                                        cfg.amplitude, cfg.center, cfg.width))
    host_in = swdemo.SWState(*(Field(full, p.numpy(), "f32") for p in pin[:3]), cfg.g, cfg.dx, cfg.dy)
    host_out = swdemo.SWState(*(Field(full, p.numpy(), "f32") for p in pin[3:]), cfg.g, cfg.dx, cfg.dy)
    torch.cuda.synchronize()
    dist.barrier()
    t0 = time.perf_counter()
    stream = torch.cuda.Stream(dev)
    with torch.cuda.stream(stream):
        sim = DistributedSimulation(cfg, grid, rank, dev, stream=stream, transport=args.transport, state=host_in)
        sim.advance(steps)
        sim.state().to_host(host_out)
    torch.cuda.synchronize()
    el = time.perf_counter() - t0
    sim.close()
    dist.barrier()
    tt = torch.tensor([el], dtype=torch.float64, device="cpu" if one_dev else dev)
    dist.all_reduce(tt, op=dist.ReduceOp.MAX)
    el = float(tt.item())
    state_bytes = 3 * 4 * (t.nx + 2) * (t.ny + 2) * world
    return {"value": round(grid.NX * grid.NY * steps / el / 1e9, 3), "unit": "Gcell-updates/s",
            "h2d_bytes_per_step": round(state_bytes / steps, 1), "d2h_bytes_per_step": round(state_bytes / steps, 1),
            "steps": steps, "api": "DistributedSimulation(cfg, grid, rank, state=<host pinned tile>) -> "
                                   "advance(steps) -> state().to_host(<host pinned tile>)"}


if __name__ == "__main__":
    sys.exit(main())
