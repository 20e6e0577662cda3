#!/usr/bin/env python3
"""Top stalled SASS instructions from an `ncu --page source --csv --print-source sass` export.

  python tools/sass_hot.py gpurun_out/X.sass.csv [--top 30] [--stalls]
"""
import argparse
import csv
import re

ap = argparse.ArgumentParser()
ap.add_argument("path")
ap.add_argument("--top", type=int, default=30)
ap.add_argument("--stalls", action="store_true", help="print the per-reason stall columns of the top rows")
a = ap.parse_args()
rows = list(csv.reader(open(a.path)))
h = rows[1]
data = [dict(zip(h, r)) for r in rows[2:] if len(r) == len(h)]
tot = sum(int(d["Warp Stall Sampling (All Samples)"] or 0) for d in data)
ex = sum(int(d["Instructions Executed"] or 0) for d in data)
print(f"{len(data)} instructions, {tot} stall samples, {ex} warp instructions executed")
ops = {}
for d in data:
    op = d["Source"].split()[0] if d["Source"].split() else "?"
    if op.startswith("@"):
        op = d["Source"].split()[1]
    op = re.sub(r"\..*", "", op)
    e = ops.setdefault(op, [0, 0])
    e[0] += int(d["Instructions Executed"] or 0)
    e[1] += int(d["Warp Stall Sampling (All Samples)"] or 0)
print("opcode mix (executed, % of instr, % of stall samples):")
for op, (n, s) in sorted(ops.items(), key=lambda x: -x[1][0])[:20]:
    print(f"  {op:10s} {n:12d} {100 * n / max(ex, 1):6.1f}% {100 * s / max(tot, 1):6.1f}%")
stall_cols = [c for c in h if c.startswith("stall_") or "Stall" in c and c not in (
    "Warp Stall Sampling (All Samples)", "Warp Stall Sampling (Not-issued Samples)")]
print("top stalled instructions:")
for d in sorted(data, key=lambda d: -int(d["Warp Stall Sampling (All Samples)"] or 0))[:a.top]:
    s = int(d["Warp Stall Sampling (All Samples)"] or 0)
    line = f"  {100 * s / max(tot, 1):5.1f}% {d['Address'][-5:]} {d['Source'].strip()[:70]:70s} exec {d['Instructions Executed']}"
    if a.stalls:
        reasons = sorted(((int(d[c] or 0), c) for c in stall_cols if (d[c] or "0").isdigit() and int(d[c] or 0) > 0),
                         reverse=True)[:3]
        line += "  " + ", ".join(f"{c}={v}" for v, c in reasons)
    print(line)
