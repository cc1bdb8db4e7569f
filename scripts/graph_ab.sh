# eager vs CUDA-graph replay of the bench step, interleaved: bash scripts/graph_ab.sh [bench args]
for rep in 1 2; do for g in "" "--graph"; do
  timeout 300 python bench.py --steps 200 --warmup 5 --no-e2e --no-cpu-baseline --no-sampler-ceiling $g "$@" | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('${g:-eager}', '$*', round(d['ms_per_step'],5), 'ms/step', round(d['value']/1e9,3), 'G rays/s')"
done; done
