"""Pure PCIe duplex of the e2e shape (3 x 16386^2 f32 each way, pinned) in row chunks
(the copy floor of the streamed host run).  python scripts/pcie_duplex_chunks.py"""
import torch, json, sys
n_rows, w = 16386, 16386
row_b = w * 4
res = {}
hin = [torch.empty(n_rows * w, dtype=torch.float32, pin_memory=True) for _ in range(3)]
hout = [torch.empty(n_rows * w, dtype=torch.float32, pin_memory=True) for _ in range(3)]
dev = [torch.empty(n_rows * w, dtype=torch.float32, device="cuda") for _ in range(6)]
s_up, s_dn = torch.cuda.Stream(), torch.cuda.Stream()
def run(rows, lag):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    s_up.wait_stream(torch.cuda.current_stream()); s_dn.wait_stream(torch.cuda.current_stream())
    nch = (n_rows + rows - 1) // rows
    for c in range(nch + lag):
        if c < nch:
            a, b = c * rows * w, min(n_rows, (c + 1) * rows) * w
            with torch.cuda.stream(s_up):
                for f in range(3): dev[f][a:b].copy_(hin[f][a:b], non_blocking=True)
        d = c - lag
        if 0 <= d < nch:
            a, b = d * rows * w, min(n_rows, (d + 1) * rows) * w
            with torch.cuda.stream(s_dn):
                for f in range(3): hout[f][a:b].copy_(dev[3 + f][a:b], non_blocking=True)
    torch.cuda.current_stream().wait_stream(s_up); torch.cuda.current_stream().wait_stream(s_dn)
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1)
for rows in (256, 1024, 4096):
    run(rows, 0)
    res[rows] = round(run(rows, 0), 2)
print(json.dumps({"ms_for_3.2GB_each_way_by_chunk_rows": res}))
