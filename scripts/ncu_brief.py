"""Key metrics + derived views of one ncu --set full report (any kernel):
    python scripts/ncu_brief.py REPORT "title line" > summary.txt"""
import csv
import subprocess
import sys

rep, title = sys.argv[1], sys.argv[2]
txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(txt.splitlines()))
d = dict(zip(r[0], zip(r[1], r[2])))
keys = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "l1tex__throughput.avg.pct_of_peak_sustained_elapsed",
        "lts__throughput.avg.pct_of_peak_sustained_elapsed", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "l1tex__t_sector_hit_rate.pct", "lts__t_sector_hit_rate.pct", "sm__warps_active.avg.per_cycle_active",
        "smsp__thread_inst_executed_per_inst_executed.ratio", "launch__registers_per_thread", "launch__grid_size",
        "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_lg_throttle_per_issue_active.ratio", "dram__bytes.sum.per_second"]
print(f"# {title}")
print(f"# report: {rep}")
for k in keys:
    if k in d:
        print(f"{k:82s} {d[k][1]:>18s} {d[k][0]}")
