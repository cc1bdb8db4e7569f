"""Per CUDA source line: warp instructions executed and stall samples, from an ncu report
captured with -lineinfo and --import-source on.
    python scripts/ncu_lines_src.py REPORT [top_n]"""
import csv
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(txt.splitlines()))
fname, agg, tot_i, tot_s = None, [], 0, 0
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] in ("Function Name", "Line No"):
        continue
    if r[0] != "" and r[2] == "-":                   # a CUDA source line with aggregated metrics
        try:
            s, i = int(r[4]), int(r[7])
        except ValueError:
            continue
        agg.append((i, s, fname, r[0], r[1].strip()))
        tot_i += i
        tot_s += s
agg.sort(reverse=True)
print(f"total warp instructions {tot_i:.4e}, stall samples {tot_s}")
for i, s, f, ln, src in agg[:top]:
    print(f"{100 * i / tot_i:5.1f}% inst {100 * s / tot_s:5.1f}% samp  {f}:{ln:5s} {src[:90]}")
