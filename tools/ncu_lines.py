#!/usr/bin/env python
"""Aggregate an ncu source page exported with --print-source cuda,sass by CUDA
source line: instructions executed and warp-stall samples per line.
Usage: ncu -i X.ncu-rep --page source --csv --print-source cuda,sass > s.csv
       python tools/ncu_lines.py s.csv [N]"""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
N = int(sys.argv[2]) if len(sys.argv) > 2 else 30
agg = defaultdict(lambda: [0.0, 0.0, ""])
fname = "?"
cur = None
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] in ("Function Name", "Line No"):
        continue
    # line rows: [line, src, addr, sass, stall_all, stall_notissued, samples, instr_exec, ...]
    try:
        line = int(r[0])
    except ValueError:
        continue
    key = (fname, line)
    try:
        agg[key][0] += float(r[4] or 0)
        agg[key][1] += float(r[7] or 0)
    except (ValueError, IndexError):
        pass
    agg[key][2] = r[1][:90]
tw = sum(v[0] for v in agg.values()) or 1
te = sum(v[1] for v in agg.values()) or 1
for (f, l), (w, e, s) in sorted(agg.items(), key=lambda x: -x[1][0])[:N]:
    print(f"stall={100*w/tw:5.1f}% instr={100*e/te:5.1f}%  {f}:{l}  {s.strip()}")
