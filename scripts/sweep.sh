# quick perf sweep (no e2e / cpu baseline): register caps x occupancy block sizes
run() {
  r=$(env "$@" timeout 300 python bench.py --steps 50 --warmup 3 --no-e2e --no-cpu-baseline 2>&1 | tail -1)
  python - "$*" "$r" <<'PY'
import json, sys
try:
    d = json.loads(sys.argv[2]); c = d["counts_per_rank_step"]
    print(f"{sys.argv[1]:45s} rays/s={d['value']:.3e} ms/step={d['ms_per_step']:.3f} march_ms={d['march_ms_per_step']:.3f} "
          f"gath={c['gathers']:.3e} canon={c['canonical_samples']:.3e} tp={c['tested_primary']:.3e} tl={c['tested_light']:.3e} clk={d['clocks']['sm_mhz']}")
except Exception as e:
    print(sys.argv[1], "FAILED", sys.argv[2][-400:])
PY
}
bash scripts/build_variants.sh
for mb in ${MBS:-5}; do for st in 0 1; do for sh in ${SHIFTS:-2}; do
  run NSL_LIB=/tmp/libnsl_mb${mb}_t8_s${st}.so NSL_OCC_SHIFT=$sh
done; done; done
