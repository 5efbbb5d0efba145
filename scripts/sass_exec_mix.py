#!/usr/bin/env python
"""Executed-instruction mix of a kernel from an ncu source page export
(ncu -i X.ncu-rep --page source --csv --print-source sass):
per opcode, warp-level instructions executed and stall samples; per cell
when --cells is given."""
import collections
import csv
import sys

path = sys.argv[1]
cells = float(sys.argv[2]) if len(sys.argv) > 2 else 0.0
rows = list(csv.reader(open(path)))
hdr_i = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
hdr = rows[hdr_i]
ci, si, ei = hdr.index("Source"), hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Instructions Executed")
ops = collections.Counter()
stall = collections.Counter()
tot = 0
top = []
for r in rows[hdr_i + 1:]:
    if len(r) <= ei or not r[ei].strip().isdigit():
        continue
    src = r[ci].strip()
    toks = src.split()
    if not toks:
        continue
    op = toks[1] if toks[0].startswith("@") and len(toks) > 1 else toks[0]
    op = op.split(".")[0]
    n = int(r[ei])
    ops[op] += n
    stall[op] += int(r[si] or 0)
    tot += n
    top.append((int(r[si] or 0), n, r[0], src))
print(f"total warp instructions executed: {tot}" + (f"  ({tot / cells:.3f} per cell)" if cells else ""))
for op, n in ops.most_common(40):
    print(f"{op:10s} {n:14d} {n / tot * 100:6.2f}%" + (f"  {n / cells:.4f}/cell" if cells else "") + f"  stall samples {stall[op]}")
print("\ntop stalled instructions:")
for s, n, a, src in sorted(top, reverse=True)[:25]:
    print(f"{s:8d} {n:12d}  {src}")
