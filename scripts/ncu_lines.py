"""Summarise an ncu source page (cuda,sass CSV) per CUDA source line:
warp-stall samples and warp instructions executed, top N lines."""
import csv, sys, collections
rows = list(csv.reader(open(sys.argv[1])))
hdr_i = next(i for i, r in enumerate(rows) if r and r[0] == "Line No")
hdr = rows[hdr_i]
col = {h: i for i, h in enumerate(hdr)}
i_st = hdr.index("Warp Stall Sampling (All Samples)")
i_ex = hdr.index("Instructions Executed")
line_src = {}
stall = collections.Counter(); inst = collections.Counter()
cur = None
for r in rows[hdr_i + 1:]:
    if not r: continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]; continue
    if r[0] in ("Function Name", "Line No"):
        continue
    if r[0].strip():
        cur = (fname if "fname" in dir() else "?", int(r[0])); line_src[cur] = r[1]
    if len(r) > i_ex and r[2]:
        try:
            stall[cur] += float(r[i_st] or 0); inst[cur] += float(r[i_ex] or 0)
        except ValueError:
            pass
ts, ti = sum(stall.values()), sum(inst.values())
print(f"total stall samples {ts:.0f}, warp instructions {ti:.3e}")
for ln, s in stall.most_common(int(sys.argv[2]) if len(sys.argv) > 2 else 25):
    print(f"{ln[0][:10]}:{ln[1]:4d} stall {100*s/ts:5.1f}%  inst {100*inst[ln]/ti:5.1f}%  {line_src.get(ln,'')[:90]}")
