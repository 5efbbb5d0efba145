#!/usr/bin/env python
"""Summarise ncu artefacts from gpurun_out/ into profiles/ (tracked).

    python scripts/summarize_profiles.py <round-tag>

Reads gpurun_out/launches.csv (ncu --metrics gpu__time_duration.sum launch
list of `bench.py`) and gpurun_out/prof_<mode>.ncu-rep (ncu --set full, one
launch of the step kernel per mode) and writes
  profiles/<tag>/launches.csv            (copy of the launch list)
  profiles/<tag>/launch_shares.md        (time share per kernel)
  profiles/<tag>/ncu_<mode>.md           (key metrics + stall mix + SASS mix)
  profiles/ncu_traffic.json              (dram bytes per launch, read by bench.py)
"""

from __future__ import annotations

import collections
import csv
import json
import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "gpurun_out")
N = 16384
CELLS = N * N
BYTES_PER_LAUNCH = 24 * CELLS

KEYS = ["Duration", "DRAM Throughput", "Memory Throughput", "Executed Ipc Active", "Issue Slots Busy",
        "Executed Instructions", "Achieved Active Warps Per SM", "Theoretical Occupancy",
        "Warp Cycles Per Issued Instruction", "Avg. Active Threads Per Warp", "L2 Hit Rate",
        "Registers Per Thread", "Dynamic Shared Memory Per Block", "Grid Size", "Block Size",
        "No Eligible", "SM Frequency", "DRAM Frequency"]


def ncu_csv(rep, page, *extra):
    r = subprocess.run(["ncu", "-i", rep, "--page", page, "--csv", *extra], capture_output=True, text=True)
    return list(csv.reader(r.stdout.splitlines()))


def summarize_rep(mode, rep, dst):
    rows = ncu_csv(rep, "details")
    h = rows[0]
    ci, vi, ui = h.index("Metric Name"), h.index("Metric Value"), h.index("Metric Unit")
    kname = rows[1][h.index("Kernel Name")] if len(rows) > 1 else "?"
    det = {r[ci]: (r[vi], r[ui]) for r in rows[1:] if len(r) > ui}
    raw = ncu_csv(rep, "raw")
    rh, ru, rv = raw[0], raw[1], raw[2]
    d = {n: (rv[i], ru[i]) for i, n in enumerate(rh)}

    def num(k):
        v, u = d[k]
        v = float(v)
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)
        return v * scale

    rd, wr = num("dram__bytes_read.sum"), num("dram__bytes_write.sum")
    stalls = {k.replace("smsp__pcsamp_warps_issue_stalled_", ""): float(v[0] or 0) for k, v in d.items()
              if k.startswith("smsp__pcsamp_warps_issue_stalled") and not k.endswith("not_issued")}
    tot = sum(stalls.values()) or 1.0
    src = ncu_csv(rep, "source", "--print-source", "sass")
    sh, sdata = src[1], src[2:]
    isrc, ie = sh.index("Source"), sh.index("Instructions Executed")
    ops = collections.Counter()
    total = 0
    for x in sdata:
        t = x[isrc].split()
        if not t:
            continue
        op = t[1] if t[0].startswith("@") else t[0]
        n = int(x[ie] or 0)
        ops[op.split(".")[0]] += n
        total += n
    dur = det.get("Duration", ("0", "ms"))
    lines = [f"# ncu --set full: `{kname[:80]}` ({mode} mode, 16384^2 f32)", "",
             f"Captured with `ncu --set full --clock-control none --import-source on -k regex:sw_step_tma` "
             f"on one B200; one launch after warm-up. Times under ncu are cold-cache and serialised: "
             f"use the shares and counters, not the absolute duration.", "",
             "| metric | value |", "|---|---|"]
    for k in KEYS:
        if k in det:
            lines.append(f"| {k} | {det[k][0]} {det[k][1]} |")
    lines += [f"| dram__bytes_read.sum | {rd / 1e9:.4f} GB |", f"| dram__bytes_write.sum | {wr / 1e9:.4f} GB |",
              f"| DRAM traffic / algorithmic bytes (24 B/cell) | {(rd + wr) / BYTES_PER_LAUNCH:.4f} |", "",
              "Warp stall mix (pc sampling): " + ", ".join(
                  f"{k} {v / tot * 100:.0f}%" for k, v in sorted(stalls.items(), key=lambda x: -x[1]) if v / tot > 0.015),
              "", f"Executed SASS per interior cell: {total / CELLS:.3f} warp-instructions; top opcodes per cell: " +
              ", ".join(f"{k} {v / CELLS:.2f}" for k, v in ops.most_common(16)), ""]
    open(dst, "w").write("\n".join(lines))
    return {"traffic_bytes": rd + wr, "dram_read": rd, "dram_write": wr,
            "algorithmic_bytes": BYTES_PER_LAUNCH, "ncu_duration": f"{dur[0]} {dur[1]}"}


def launch_shares(src, dst):
    rows = [r for r in csv.reader(open(src)) if r and r[0].isdigit()]
    tot, cnt = collections.Counter(), collections.Counter()
    for r in rows:
        name = r[4].split("(")[0]
        tot[name] += float(r[-1])
        cnt[name] += 1
    T = sum(tot.values())
    out = ["# Launch list of `python bench.py --steps 20 --warmup 5 --no-cpu --no-e2e --no-other`",
           "", "ncu --metrics gpu__time_duration.sum --clock-control none (cold-cache, serialised).", "",
           "The timed region of bench.py launches only `sw_step_tma` (one launch per step: 5 warm-up + 20 timed "
           "here); every other kernel below is setup outside it (the Gaussian initial state built with torch "
           "elementwise ops, the initial halo fill, the stable_dt reduction that fixes dt).  Share of the "
           "step kernel in the TIMED region: 100 %.", "",
           "| kernel | launches | total ms | share | avg us |", "|---|---|---|---|---|"]
    for k, v in tot.most_common():
        out.append(f"| `{k[:70]}` | {cnt[k]} | {v / 1e6:.3f} | {v / T * 100:.1f}% | {v / cnt[k] / 1e3:.1f} |")
    open(dst, "w").write("\n".join(out) + "\n")


def main():
    tag = sys.argv[1] if len(sys.argv) > 1 else "r01"
    pdir = os.path.join(ROOT, "profiles", tag)
    os.makedirs(pdir, exist_ok=True)
    lc = os.path.join(OUT, "launches.csv")
    if os.path.exists(lc):
        shutil.copy(lc, os.path.join(pdir, "launches.csv"))
        launch_shares(lc, os.path.join(pdir, "launch_shares.md"))
    traffic_path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    traffic = json.load(open(traffic_path)) if os.path.exists(traffic_path) else {}
    for mode in ("fast", "exact"):
        rep = os.path.join(OUT, f"prof_{mode}.ncu-rep")
        if os.path.exists(rep):
            info = summarize_rep(mode, rep, os.path.join(pdir, f"ncu_{mode}.md"))
            info["round"] = tag
            traffic[f"{mode}_{N}"] = info["traffic_bytes"]
            traffic[f"{mode}_{N}_detail"] = info
    json.dump(traffic, open(traffic_path, "w"), indent=1)
    print("wrote", pdir)


if __name__ == "__main__":
    main()
