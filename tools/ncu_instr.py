#!/usr/bin/env python
"""Top CUDA source lines by executed instructions (per element) from an ncu
source CSV (--print-source cuda,sass).  usage: ncu_instr.py s.csv n_elements [N]"""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
nel = float(sys.argv[2])
N = int(sys.argv[3]) if len(sys.argv) > 3 else 25
agg = defaultdict(lambda: [0.0, ""])
fname = "?"
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    try:
        line = int(r[0])
        agg[(fname, line)][0] += float(r[7] or 0)
        agg[(fname, line)][1] = r[1][:85]
    except (ValueError, IndexError):
        continue
te = sum(v[0] for v in agg.values())
print(f"total {te:.3g} warp-instr = {32*te/nel:.1f} thread-instr per element")
for (f, l), (e, s) in sorted(agg.items(), key=lambda x: -x[1][0])[:N]:
    print(f"{32*e/nel:6.2f}/elem  {f}:{l}  {s.strip()}")
