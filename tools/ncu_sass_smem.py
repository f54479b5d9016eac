"""SASS instructions of one kernel ranked by shared-memory wavefronts:
ncu -i R --page source --csv --launch-skip S --launch-count 1 --print-source sass > f.csv
python tools/ncu_sass_smem.py f.csv [top]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
h = rows[1]
iw, ii, isrc, ie = h.index("L1 Wavefronts Shared"), h.index("L1 Wavefronts Shared Ideal"), h.index("Source"), \
    h.index("Instructions Executed")
data = []
for r in rows[2:]:
    try:
        data.append((float(r[iw]), float(r[ii]), float(r[ie]), r[0][-5:], r[isrc].strip()))
    except (ValueError, IndexError):
        pass
tot = sum(d[0] for d in data)
print(f"total smem wavefronts {tot/1e6:.1f}M")
for w, ideal, ex, a, s in sorted(data, key=lambda d: -d[0])[:top]:
    print(f"{w/1e6:9.2f}M ideal {ideal/1e6:8.2f}M  instr {ex/1e6:8.2f}M  {w/max(ex,1):5.2f}/instr  {a} {s}")

agg = {}
for w, ideal, ex, a, s in data:
    s2 = s.replace("@!P", "@P")
    op = s2.split()[1] if s2.startswith("@") else s2.split()[0]
    t = agg.setdefault(op, [0.0, 0.0])
    t[0] += w
    t[1] += ex
print("by opcode (wavefronts, instr):")
for op, (w, ex) in sorted(agg.items(), key=lambda x: -x[1][0])[:15]:
    if w:
        print(f"  {op:28s} {w/1e6:9.1f}M  {ex/1e6:8.1f}M instr  {w/max(ex,1):5.2f}/instr")
