"""Key metrics + stall reasons of every kernel in an ncu report:
python tools/ncu_brief.py REPORT"""
import csv
import io
import subprocess
import sys

txt = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
hdr, data = rows[0], rows[2:]
KEYS = [("gpu__time_duration.sum", "time"), ("dram__bytes_read.sum", "dram_rd"), ("dram__bytes_write.sum", "dram_wr"),
        ("smsp__inst_executed.sum", "warp_instr"), ("sm__warps_active.avg.pct_of_peak_sustained_active", "occ%"),
        ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue%"),
        ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "smem_wf"),
        ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smem_conf"),
        ("lts__t_sector_hit_rate.pct", "L2hit%"), ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "dram%"),
        ("l1tex__t_requests_pipe_lsu_mem_global_op_st.sum", "st_req"),
        ("l1tex__t_sectors_pipe_lsu_mem_global_op_st.sum", "st_sect"),
        ("launch__registers_per_thread", "regs"), ("launch__occupancy_limit_shared_mem", "occ_smem")]
for r in data:
    name = r[hdr.index("Kernel Name")][:60]
    out = []
    for k, lab in KEYS:
        if k in hdr:
            out.append(f"{lab}={r[hdr.index(k)]}")
    print(name)
    print("   " + "  ".join(out))
    st = [(float(r[i] or 0), h.replace("smsp__average_warps_issue_stalled_", "").replace("_per_issue_active.ratio", ""))
          for i, h in enumerate(hdr) if h.startswith("smsp__average_warps_issue_stalled_") and
          h.endswith("_per_issue_active.ratio") and r[i].replace(".", "", 1).isdigit()]
    st.sort(reverse=True)
    print("   stalls: " + ", ".join(f"{n} {v:.2f}" for v, n in st[:8]))
