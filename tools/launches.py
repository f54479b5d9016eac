"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list: per-kernel totals and the sequence."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr, seq = None, []
for r in rows:
    if r and r[0] == "ID":
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        if d.get("Metric Name") == "gpu__time_duration.sum":
            v = float(d["Metric Value"].replace(",", ""))
            u = d["Metric Unit"]
            ms = v / 1e6 if u in ("ns", "nsecond") else v / 1e3 if u in ("us", "usecond") else v
            seq.append((d["Kernel Name"].split("(")[0][:60], ms, d.get("Grid Size", "")))
agg = collections.defaultdict(lambda: [0.0, 0])
for n, ms, _ in seq:
    agg[n][0] += ms
    agg[n][1] += 1
tot = sum(v[0] for v in agg.values())
print(f"total {tot:.3f} ms over {len(seq)} launches")
for n, (ms, c) in sorted(agg.items(), key=lambda x: -x[1][0]):
    print(f"{ms:10.3f} ms {100 * ms / tot:5.1f} % {c:5d}  {n}")
if "-v" in sys.argv:
    for n, ms, g in seq:
        print(f"{ms:9.3f} {g:>16} {n}")
