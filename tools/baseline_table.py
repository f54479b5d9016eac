#!/usr/bin/env python
"""BASELINE.md section 3 rows from committed bench lines:
python tools/baseline_table.py profiles/r06a_bench.json profiles/r06b_bench_c1.json ..."""
import json
import sys

print("| Config | Oracle (1 core), measured on its sample | Measured GPU time | GPU elements/s | GPU eff. GB/s | % of 8 TB/s | % of measured copy | Host CPU / cores | Source |")
print("|---|---|---|---|---|---|---|---|---|")
for f in sys.argv[1:]:
    d = json.loads(open(f).read().strip().splitlines()[-1])
    w = d["config"]["workload"].split(":")[0].upper()
    cb = d.get("cpu_baseline") or {}
    orc = f"{cb['value'] / 1e6:.1f} M elem/s ({cb['sample'].split(';')[-1].strip()})" if cb else "-"
    host = f"{cb.get('cpu_model', '?')} / {cb.get('host_cpus', '?')}" if cb else "-"
    print(f"| {w} | {orc} | {d['ms_per_step']:.3f} ms | {d['value']:.3g} | {d['eff_GBps']:.0f} | "
          f"{100 * d['frac_of_8TBps']:.1f} | {100 * d['frac_of_measured_copy']:.1f} | {host} | `{f}` |")
