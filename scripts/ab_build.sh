# A/B of volume-build variants on C4 (60 distinct 256^3 volumes per step): layout ms per step
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
  echo "$name $(NSL_LIB=/tmp/libnsl_${name}.so python bench.py --config ${CFG:-C4} --frames ${FRAMES:-60} --steps 10 --no-e2e --no-cpu-baseline | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["layout_ms_per_step"], d["march_ms_per_step"])')"
done; done
