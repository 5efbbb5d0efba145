"""Wall time of the streamed host run (fkc_sw_run_host) at the e2e shape
(16384^2 f32, pinned host state in and out) for a few step counts and band
heights, beside the plain upload + download.  python scripts/stream_timing.py"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1107_2157_b200 import swdemo  # noqa: E402
from paper_1107_2157_b200.field import Field  # noqa: E402
from paper_1107_2157_b200.region import Extent  # noqa: E402

n = int(os.environ.get("N", 16384))
full = Extent(n + 2, n + 2)
pin = [torch.ones((n + 2, n + 2), dtype=torch.float32, pin_memory=True) for _ in range(6)]
for t in pin[1:3]:
    t.zero_()
st = swdemo.SWState(*(Field(full, t.numpy(), "f32") for t in pin[:3]))
out = swdemo.SWState(*(Field(full, t.numpy(), "f32") for t in pin[3:]))
rows = []
for steps in [int(x) for x in os.environ.get("STEPS", "0,1,20,200").split(",")]:
    for br in [int(b) for b in os.environ.get("BANDS", "0,64,256,1024").split(",")]:
        cfg = swdemo.SWConfig(nx=n, ny=n, steps=steps, dt=0.05, mode="fast")
        swdemo._run_streamed(cfg, st, out, band_rows=br)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        swdemo._run_streamed(cfg, st, out, band_rows=br)
        el = time.perf_counter() - t0
        r = {"steps": steps, "band_rows": br, "seconds": round(el, 4),
             "gcell_s": round(n * n * steps / el / 1e9, 2) if steps else None}
        rows.append(r)
        print(json.dumps(r), flush=True)
