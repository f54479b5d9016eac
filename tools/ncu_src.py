"""Per-source-line hot spots of one kernel in an ncu report:
python tools/ncu_src.py REPORT [launch_skip] [top]  (needs --import-source on, -lineinfo)."""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
skip = sys.argv[2] if len(sys.argv) > 2 else "0"
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--launch-skip", skip, "--launch-count", "1",
                      "--print-source", "cuda,sass"], capture_output=True, text=True).stdout
cur, hdr, out = None, None, []
for r in csv.reader(io.StringIO(txt)):
    if not r:
        continue
    if r[0] == "File Path":
        cur = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr and r[0].isdigit() and len(r) == len(hdr):
        g = lambda k: int(float(r[hdr.index(k)] or 0)) if r[hdr.index(k)] not in ("-", "") else 0
        out.append((g("Warp Stall Sampling (All Samples)"), g("Instructions Executed"), g("L1 Wavefronts Shared"),
                    cur, r[0], r[1][:80]))
out.sort(reverse=True)
tot = sum(o[0] for o in out) or 1
print("total samples", tot, "warp-instr", sum(o[1] for o in out), "smem wavefronts", sum(o[2] for o in out))
for o in out[:top]:
    print(f"{o[0]:7d} {100*o[0]/tot:5.1f}% ins {o[1]/1e6:8.2f}M wf {o[2]/1e6:7.2f}M {o[3]}:{o[4]} {o[5]}")
