"""Warp-stall breakdown and a few headline counters of the first kernel in an
ncu report (--page raw).  usage: python scripts/ncu_stalls.py <report.ncu-rep>"""
import csv, subprocess, sys
raw = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(raw.splitlines()))
h, v = rows[0], rows[2] if len(rows) > 2 else rows[1]
d = dict(zip(h, v))
num = lambda x: float(x.replace(",", "")) if x and x.replace(",", "").replace(".", "").isdigit() else 0.0
st = {k: num(x) for k, x in d.items() if "smsp__pcsamp_warps_issue_stalled" in k and not k.endswith("not_issued")}
tot = sum(st.values()) or 1
for k, x in sorted(st.items(), key=lambda kv: -kv[1])[:10]:
    print(f"{x / tot * 100:5.1f}% {k.replace('smsp__pcsamp_warps_issue_stalled_', 'stall_')}")
for k in ["gpu__time_duration.sum", "smsp__inst_executed.sum", "sm__warps_active.avg.pct_of_peak_sustained_active",
          "smsp__issue_active.avg.pct_of_peak_sustained_active", "lts__t_sector_hit_rate.pct",
          "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
          "dram__bytes_read.sum", "dram__bytes_write.sum", "launch__occupancy_limit_shared_mem",
          "launch__shared_mem_per_block_dynamic", "launch__registers_per_thread"]:
    print(f"  {k} {d.get(k)}")
