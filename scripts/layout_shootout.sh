# Layout shoot-out: march + build per step for every fp32 layout on C2, C3 and
# C5 (64 frames), same box, interleaved.  Usage: bash scripts/layout_shootout.sh OUTFILE
out=${1:-gpurun_out/layouts.jsonl}
: > $out
for rep in 1 2; do
  for cfg in "C2" "C3" "C5 --frames 64"; do
    for lay in oct_f32 brick_oct_f32 morton_oct_f32 tex3d_f32 quad_f32; do
      r=$(timeout 300 python bench.py --config $cfg --layout $lay --steps 10 --warmup 3 --no-e2e --no-cpu-baseline \
          --no-sampler-ceiling 2>/dev/null | tail -1)
      python - "$cfg" "$lay" "$r" >> $out <<'PY'
import json, sys
try:
    d = json.loads(sys.argv[3])
    print(json.dumps({"config": sys.argv[1], "layout": sys.argv[2], "march_ms": d["march_ms_per_step"],
                      "build_ms": d["layout_ms_per_step"], "step_ms": d["ms_per_step"],
                      "l1_frac": d["roofline"]["frac"], "clk": d["clocks"]["sm_mhz"]}))
except Exception as e:
    print(json.dumps({"config": sys.argv[1], "layout": sys.argv[2], "error": sys.argv[3][-300:]}))
PY
    done
  done
done
