# A/B of two source trees: the working tree vs $OLD (a copy of paper_2604_03748_b200/csrc + include)
# bench config: CFG (default C2), FRAMES, extra env per run; prints step / layout / march ms.
set -e
cd "$(dirname "$0")/.."
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -Xcompiler -fPIC -shared -cudart static \
     -o /tmp/libnsl_new.so paper_2604_03748_b200/csrc/*.cu &
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -Xcompiler -fPIC -shared -cudart static \
     -o /tmp/libnsl_old.so $OLD/paper_2604_03748_b200/csrc/*.cu &
wait
for rep in 1 2 3; do for v in old new; do
  echo "$v $(NSL_LIB=/tmp/libnsl_${v}.so python bench.py --config ${CFG:-C2} ${FRAMES:+--frames $FRAMES} --steps ${STEPS:-50} --no-e2e --no-cpu-baseline | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["ms_per_step"], d["layout_ms_per_step"], d["march_ms_per_step"])')"
done; done
