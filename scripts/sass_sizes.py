#!/usr/bin/env python
"""Instruction count per kernel in the built library (cuobjdump -sass)."""
import re
import subprocess
import sys

lib = sys.argv[1] if len(sys.argv) > 1 else "paper_1107_2157_b200/lib/libfkc_sw.so"
out = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
cur, counts = None, {}
for line in out.splitlines():
    m = re.search(r"Function : (\S+)", line)
    if m:
        cur = m.group(1)
        counts[cur] = 0
    elif cur and re.match(r"\s+/\*[0-9a-f]{4,6}\*/", line):
        counts[cur] += 1
for k, v in counts.items():
    if len(sys.argv) < 3 or sys.argv[2] in k:
        print(f"{v:7d} {v * 16 / 1024:7.1f} KB  {k[:90]}")
