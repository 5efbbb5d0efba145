"""PCIe copy rates on this box: H2D alone, D2H alone, both at once on two
streams (pinned host memory, 1 GiB each way), and 2-D pitched copies of the
e2e field shape.  python scripts/pcie_duplex.py"""
import json
import torch

n = 1 << 28          # 1 GiB of f32
h_in = torch.empty(n, dtype=torch.float32, pin_memory=True)
h_out = torch.empty(n, dtype=torch.float32, pin_memory=True)
d_a = torch.empty(n, dtype=torch.float32, device="cuda")
d_b = torch.empty(n, dtype=torch.float32, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def timed(fn):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / 1e3


def h2d():
    with torch.cuda.stream(s1):
        d_a.copy_(h_in, non_blocking=True)
    torch.cuda.current_stream().wait_stream(s1)


def d2h():
    with torch.cuda.stream(s2):
        h_out.copy_(d_b, non_blocking=True)
    torch.cuda.current_stream().wait_stream(s2)


def both():
    s1.wait_stream(torch.cuda.current_stream())
    s2.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s1):
        d_a.copy_(h_in, non_blocking=True)
    with torch.cuda.stream(s2):
        h_out.copy_(d_b, non_blocking=True)
    torch.cuda.current_stream().wait_stream(s1)
    torch.cuda.current_stream().wait_stream(s2)


for f in (h2d, d2h, both):
    f()
gb = n * 4 / 1e9
r = {"h2d_GBs": round(gb / timed(h2d), 1), "d2h_GBs": round(gb / timed(d2h), 1)}
t = timed(both)
r["both_total_GBs"] = round(2 * gb / t, 1)
r["both_seconds"] = round(t, 4)
print(json.dumps(r))

# 2-D pitched copies of the e2e field shape (16386 x 16386 f32 host rows,
# device pitch 16416), one field each way, in 128-row chunks
import ctypes  # noqa: E402
import os  # noqa: E402
import sys  # noqa: E402
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1107_2157_b200 import _native as N  # noqa: E402
L = N.lib()
w, hrows = 16386, 16386
dp = 16416
hf_in = torch.empty((hrows, w), dtype=torch.float32, pin_memory=True)
hf_out = torch.empty((hrows, w), dtype=torch.float32, pin_memory=True)
df_a = torch.empty((hrows, dp), dtype=torch.float32, device="cuda")
df_b = torch.empty((hrows, dp), dtype=torch.float32, device="cuda")


def chunks2d(up, stream, rows=128):
    for r in range(0, hrows, rows):
        nr = min(rows, hrows - r)
        if up:
            N.check(L.fkc_copy2d(df_a.data_ptr() + r * dp * 4, dp * 4, hf_in.data_ptr() + r * w * 4, w * 4, w * 4, nr,
                                 stream.cuda_stream))
        else:
            N.check(L.fkc_copy2d(hf_out.data_ptr() + r * w * 4, w * 4, df_b.data_ptr() + r * dp * 4, dp * 4, w * 4, nr,
                                 stream.cuda_stream))


def up2d():
    s1.wait_stream(torch.cuda.current_stream())
    chunks2d(True, s1)
    torch.cuda.current_stream().wait_stream(s1)


def down2d():
    s2.wait_stream(torch.cuda.current_stream())
    chunks2d(False, s2)
    torch.cuda.current_stream().wait_stream(s2)


def both2d():
    s1.wait_stream(torch.cuda.current_stream())
    s2.wait_stream(torch.cuda.current_stream())
    chunks2d(True, s1)
    chunks2d(False, s2)
    torch.cuda.current_stream().wait_stream(s1)
    torch.cuda.current_stream().wait_stream(s2)


for f in (up2d, down2d, both2d):
    f()
gb = hrows * w * 4 / 1e9
r = {"h2d_2d_GBs": round(gb / timed(up2d), 1), "d2h_2d_GBs": round(gb / timed(down2d), 1)}
t = timed(both2d)
r["both_2d_total_GBs"] = round(2 * gb / t, 1)
print(json.dumps(r))
