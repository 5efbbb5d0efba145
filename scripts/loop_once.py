"""One persistent-loop call (for ncu): python scripts/loop_once.py N STEPS MODE [SEG] [VARIANT]"""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from bench import device_gaussian_state
from paper_1107_2157_b200 import _native as N
from paper_1107_2157_b200 import swdemo
n, k, mode = int(sys.argv[1]), int(sys.argv[2]), sys.argv[3]
seg = int(sys.argv[4]) if len(sys.argv) > 4 else 0
variant = sys.argv[5] if len(sys.argv) > 5 else "loop"
st = device_gaussian_state(n, n, torch.device("cuda", 0))
dt = 0.3 * swdemo.stable_dt(st, 1.0)
cfg = swdemo.SWConfig(nx=n, ny=n, dt=dt, mode=mode, variant=variant)
sim = swdemo.Simulation(cfg, state=st, diagnostics=False, tune=N.Tune(seg=seg))
sim.advance(k)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
sim.advance(k)
e1.record()
torch.cuda.synchronize()
print(f"n={n} k={k} mode={mode} seg={seg} variant={variant}: {e0.elapsed_time(e1) / k * 1e3:.3f} us/step")
