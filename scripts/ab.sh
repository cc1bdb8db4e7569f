# A/B of compile-time variants: VARIANTS="name1:-DFOO=1 -DBAR=2;name2:..." bash scripts/ab.sh
# builds /tmp/libnsl_<name>.so for each, then runs the bench REPS times per variant (interleaved).
set -e
cd "$(dirname "$0")/.."
IFS=';' read -ra VS <<< "${VARIANTS}"
for v in "${VS[@]}"; do
  name="${v%%:*}"; flags="${v#*:}"
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -shared -cudart static \
       $flags -o /tmp/libnsl_${name}.so paper_2604_03748_b200/csrc/*.cu &
done
wait
for rep in $(seq ${REPS:-2}); do
  for v in "${VS[@]}"; do
    name="${v%%:*}"
    r=$(NSL_LIB=/tmp/libnsl_${name}.so timeout 300 python bench.py --steps ${STEPS:-100} --warmup 3 --no-e2e --no-cpu-baseline ${BENCH_ARGS} 2>&1 | tail -1)
    python - "$name" "$r" <<'PY'
import json, sys
try:
    d = json.loads(sys.argv[2]); c = d["counts_per_rank_step"]
    print(f"{sys.argv[1]:20s} ms/step={d['ms_per_step']:.4f} march_ms={d['march_ms_per_step']:.4f} gath={c['gathers']:.4e} clk={d['clocks']['sm_mhz']}")
except Exception as e:
    print(sys.argv[1], "FAILED", sys.argv[2][-400:])
PY
  done
done
