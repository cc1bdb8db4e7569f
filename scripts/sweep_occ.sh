# occupancy block size sweep on the default build: NSL_OCC_SHIFT = 1 (2^3 cells), 2, 3
cd "$(dirname "$0")/.."
for rep in 1 2; do for sh in ${SHIFTS:-1 2 3}; do
  r=$(NSL_OCC_SHIFT=$sh timeout 300 python bench.py --steps ${STEPS:-60} --warmup 3 --no-e2e --no-cpu-baseline 2>&1 | tail -1)
  python - "shift=$sh" "$r" <<'PY'
import json, sys
d = json.loads(sys.argv[2]); c = d["counts_per_rank_step"]
print(f"{sys.argv[1]:10s} ms/step={d['ms_per_step']:.4f} march_ms={d['march_ms_per_step']:.4f} gath={c['gathers']:.4e} "
      f"tp={c['tested_primary']:.4e} tl={c['tested_light']:.4e}")
PY
done; done
