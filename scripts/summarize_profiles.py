"""Copy a gpu_round.sh evidence run from gpurun_out/ into profiles/ with text summaries.

    python scripts/summarize_profiles.py TAG   (TAG as passed to gpu_round.sh, e.g. r1d)
"""
import collections
import csv
import json
import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
G = os.path.join(ROOT, "gpurun_out")
P = os.path.join(ROOT, "profiles")
tag = sys.argv[1]
round_tag = tag[:2]

shutil.copy(os.path.join(G, "bench.json"), os.path.join(P, f"{round_tag}_bench.json"))
shutil.copy(os.path.join(G, "bench_ref.json"), os.path.join(P, f"{round_tag}_bench_reference.json"))
shutil.copy(os.path.join(G, "gpu_tests.log"), os.path.join(P, f"{round_tag}_gpu_tests.log"))
for extra in ("bench_relight.json", "bench_bake.json", "smoke.log"):
    if os.path.exists(os.path.join(G, extra)):
        shutil.copy(os.path.join(G, extra), os.path.join(P, f"{round_tag}_{extra}"))
shutil.copy(os.path.join(G, "launches.csv"), os.path.join(P, f"{round_tag}_launches.csv"))
rep = os.path.join(P, f"{round_tag}_march_kernel_full.ncu-rep")
shutil.copy(os.path.join(G, f"prof_march_{tag}.ncu-rep"), rep)

# ---- launch list summary
rows = list(csv.reader(open(os.path.join(P, f"{round_tag}_launches.csv"))))
hi = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
hdr = rows[hi]
ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
agg = collections.OrderedDict()
scale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}
for r in rows[hi + 1:]:
    if len(r) <= vi:
        continue
    name = r[ki].split("(")[0].replace("void ", "")
    agg.setdefault(name, []).append(float(r[vi].replace(",", "")) * scale.get(r[ui], 1.0))
tot = sum(sum(v) for v in agg.values())
out = [f"# ncu launch list of `python bench.py --steps 3 --warmup 1 --no-e2e --no-cpu-baseline --no-sampler-ceiling` (B200, {tag})",
       "# gpu__time_duration.sum with --clock-control none: cold-cache, serialised; compare SHARES, not absolutes.",
       "# march_kernel<layout, proj, 2, tv> is the one instrumented (counted) launch; at::FillFunctor<uchar> is the L2 flush.", ""]
step = 0.0
for k, v in agg.items():
    out.append(f"{len(v):3d} launches  mean {sum(v) / len(v):9.2f} us  share-of-all {100 * sum(v) / tot:5.1f}%  {k}")
    counted = "march_kernel" in k and k.split("<")[-1].split(",")[2].strip() == "2"
    if k.startswith("nsl") and not counted:
        step += sum(v) / len(v)
mk = [sum(v) / len(v) for k, v in agg.items()
      if "march_kernel" in k and k.split("<")[-1].split(",")[2].strip() == "0"]
out += ["", f"one bench step (volume build + finalize + frame_setup + cull + march means): {step:.1f} us; "
            f"march_kernel share of the step: {100 * mk[0] / step:.1f}%" if mk else ""]
open(os.path.join(P, f"{round_tag}_launches_summary.txt"), "w").write("\n".join(out) + "\n")
print("\n".join(out))

# ---- ncu full metrics summary + traffic json
txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(txt.splitlines()))
d = dict(zip(r[0], zip(r[1], r[2])))
keys = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed.avg.per_cycle_active", "smsp__inst_executed.sum", "smsp__thread_inst_executed.sum",
        "l1tex__throughput.avg.pct_of_peak_sustained_elapsed",
        "l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed",
        "lts__throughput.avg.pct_of_peak_sustained_elapsed", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "l1tex__t_sector_hit_rate.pct", "lts__t_sector_hit_rate.pct", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__thread_inst_executed_per_inst_executed.ratio", "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__occupancy_limit_registers", "launch__grid_size", "launch__block_size",
        "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_not_selected_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio", "sm__warps_active.avg.per_cycle_active",
        "dram__bytes.sum.per_second", "lts__t_sectors.sum"]
lines = ["# ncu --set full of march_kernel<OCT_F32, ORTHO, FAST> on C2 (60 frames 512^2 over 128^3, guide lights)",
         "# command: ncu --set full --clock-control none --import-source on -k regex:march_kernel -s 2 -c 1 "
         "python scripts/profile_march.py", f"# report: {os.path.relpath(rep, ROOT)}", ""]
for k in keys:
    if k in d:
        lines.append(f"{k:82s} {d[k][1]:>18s} {d[k][0]}")
# derived views against the chip's peaks (north star: "achieved L1/TEX and L2 throughput, HBM GB/s,
# and warp execution efficiency against the chip's peaks")
def val(k, scale=1.0):
    return float(d[k][1].replace(",", "")) * scale if k in d else float("nan")


t_s = val("gpu__time_duration.sum") * ({"usecond": 1e-6, "us": 1e-6, "msecond": 1e-3, "ms": 1e-3}.get(
    d.get("gpu__time_duration.sum", ("us",))[0], 1e-6))
peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))) if os.path.exists(
    os.path.join(ROOT, "MEASURED_PEAKS.json")) else {"hbm_gbs": 6541.1}
lines += ["", "# derived",
          f"warp execution efficiency (active threads per issued instruction / 32): "
          f"{val('smsp__thread_inst_executed_per_inst_executed.ratio') / 32:.3f}",
          f"warps active per SM: {val('sm__warps_active.avg.per_cycle_active'):.1f} of 64",
          f"HBM: {val('dram__bytes.sum.per_second'):.0f} GB/s achieved vs {peaks['hbm_gbs']:.0f} GB/s measured copy peak "
          f"({val('gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed'):.1f} % of DRAM peak per ncu)",
          f"L2: {val('lts__t_sectors.sum') * 32 / t_s / 1e9:.0f} GB/s of sector traffic "
          f"({val('lts__throughput.avg.pct_of_peak_sustained_elapsed'):.1f} % of L2 peak per ncu), "
          f"hit rate {val('lts__t_sector_hit_rate.pct'):.1f} %",
          f"L1/TEX: {val('l1tex__throughput.avg.pct_of_peak_sustained_elapsed'):.1f} % of peak (data-pipe wavefronts), "
          f"hit rate {val('l1tex__t_sector_hit_rate.pct'):.1f} %",
          f"issue slots: {val('smsp__issue_active.avg.pct_of_peak_sustained_active'):.1f} % active "
          f"(the binding limit; long-scoreboard stalls {val('smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio'):.2f} per issue)"]
open(os.path.join(P, f"{round_tag}_ncu_march_summary.txt"), "w").write("\n".join(lines) + "\n")
mult = {"Mbyte": 1e6, "Gbyte": 1e9, "Kbyte": 1e3, "byte": 1}
traffic = (float(d["dram__bytes_read.sum"][1]) * mult[d["dram__bytes_read.sum"][0]]
           + float(d["dram__bytes_write.sum"][1]) * mult[d["dram__bytes_write.sum"][0]])
json.dump({"config": "C2", "layout": "oct_f32", "frames": 60, "dram_bytes_per_launch": traffic,
           "source": f"{os.path.relpath(rep, ROOT)} (dram__bytes_read.sum + dram__bytes_write.sum)"},
          open(os.path.join(P, "ncu_march_traffic.json"), "w"), indent=1)
print("\n".join(lines))
