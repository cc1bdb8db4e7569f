# quick perf sweep of layouts and occupancy block sizes (no e2e / cpu baseline)
for layout in quad_f32 linear_f32 corner_f16; do
  for sh in 1 2 3; do
    r=$(NSL_OCC_SHIFT=$sh timeout 300 python bench.py --steps 50 --warmup 3 --no-e2e --no-cpu-baseline --layout $layout 2>&1 | tail -1)
    python - "$layout" "$sh" "$r" <<'PY'
import json, sys
try:
    d = json.loads(sys.argv[3])
    c = d["counts_per_rank_step"]
    print(f"{sys.argv[1]:11s} shift={sys.argv[2]} rays/s={d['value']:.3e} ms/step={d['ms_per_step']:.3f} march_ms={d['march_ms_per_step']:.3f} "
          f"gathers={c['gathers']:.3e} canon={c['canonical_samples']:.3e} frac={d['roofline']['frac']:.3f} clk={d['clocks']['sm_mhz']}")
except Exception as e:
    print(sys.argv[1], sys.argv[2], "FAILED", sys.argv[3][-300:])
PY
  done
done
