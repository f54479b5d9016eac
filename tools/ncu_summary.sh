#!/bin/bash
# Summarise an ncu report: key metrics, stall mix, top CUDA source lines.
# usage: tools/ncu_summary.sh report.ncu-rep [Nlines]
R=$1; N=${2:-15}
ncu -i $R --page details --csv 2>/dev/null | grep -E '"(Duration|DRAM Throughput|Memory Throughput|Achieved Occupancy|Registers Per Thread|Issue Slots Busy|L2 Hit Rate|Theoretical Occupancy|Executed Ipc Active|Block Limit Registers|Block Limit Shared Mem|Dynamic Shared Memory Per Block)"' | awk -F'","' '{gsub(/"/,"",$NF); printf "%s %s %s; ", $(NF-2), $(NF-1), $NF} END {print ""}'
ncu -i $R --page raw --csv 2>/dev/null | python3 -c "
import csv,sys
r=list(csv.reader(sys.stdin)); h=r[0]; v=r[2]; d={}
for i,name in enumerate(h):
    if 'smsp__pcsamp_warps_issue_stalled' in name and not name.endswith('not_issued'):
        try: d[name.replace('smsp__pcsamp_warps_issue_stalled_','')]=float(v[i])
        except: pass
    if name in ('dram__bytes_read.sum','dram__bytes_write.sum','smsp__inst_executed.sum','sm__cycles_elapsed.avg'):
        print(name, v[i], end='; ')
print()
t=sum(d.values()) or 1
print('stalls:', ' '.join(f'{k}={100*x/t:.0f}%' for k,x in sorted(d.items(),key=lambda x:-x[1])[:8]))
"
ncu -i $R --page source --csv --print-source cuda,sass 2>/dev/null > /tmp/_src.csv
python3 $(dirname $0)/ncu_lines.py /tmp/_src.csv $N
