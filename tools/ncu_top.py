#!/usr/bin/env python
"""Summarise an ncu source-page CSV (SASS view): top instructions by warp-stall
samples.  Usage: ncu -i X.ncu-rep --page source --csv --print-source sass > s.csv;
python tools/ncu_top.py s.csv [N]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
iS = hdr.index("Source")
iW = hdr.index("Warp Stall Sampling (All Samples)")
iE = hdr.index("Instructions Executed")
data = []
for r in rows[2:]:
    try:
        data.append((float(r[iW] or 0), r[0], r[iS], r[iE]))
    except (ValueError, IndexError):
        pass
tot = sum(d[0] for d in data) or 1
N = int(sys.argv[2]) if len(sys.argv) > 2 else 25
for w, addr, src, ex in sorted(data, reverse=True)[:N]:
    print(f"{100*w/tot:5.1f}%  {addr}  {src[:90]:90s} exec={ex}")
