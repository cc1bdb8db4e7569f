# A/B of bake build variants: VARIANTS="name:-DFLAGS;..." bash scripts/ab_bake.sh
set -e
cd "$(dirname "$0")/.."
IFS=';' read -ra VS <<< "${VARIANTS}"
for v in "${VS[@]}"; do
  name="${v%%:*}"; flags="${v#*:}"
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -shared -cudart static \
       $flags -o /tmp/libnsl_${name}.so paper_2604_03748_b200/csrc/*.cu &
done
wait
for rep in 1 2; do for v in "${VS[@]}"; do
  name="${v%%:*}"
  echo "$name $(NSL_LIB=/tmp/libnsl_${name}.so python scripts/bench_bake.py --no-oracle --frames 2 --steps 3 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["ms_per_frame"])')"
done; done
