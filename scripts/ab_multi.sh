# A/B of several (source tree, nvcc flags) variants of the library on one bench config.
# VARIANTS="name:tree:flags;..."  tree = . (working tree) or a copy such as ab_old
# prints step / layout / march ms per run, REPS rounds interleaved.
set -e
cd "$(dirname "$0")/.."
IFS=';' read -ra VS <<< "${VARIANTS}"
for v in "${VS[@]}"; do
  IFS=':' read -r name tree flags <<< "$v"
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -Xcompiler -fPIC -shared -cudart static \
       $flags -o /tmp/libnsl_${name}.so $tree/paper_2604_03748_b200/csrc/*.cu &
done
wait
for rep in $(seq ${REPS:-3}); do for v in "${VS[@]}"; do
  IFS=':' read -r name tree flags <<< "$v"
  echo "$name $(NSL_LIB=/tmp/libnsl_${name}.so python bench.py --config ${CFG:-C2} ${FRAMES:+--frames $FRAMES} --steps ${STEPS:-50} --no-e2e --no-cpu-baseline ${EXTRA} | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["ms_per_step"], d["layout_ms_per_step"], d["march_ms_per_step"])')"
done; done
