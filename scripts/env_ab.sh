# bench.py under environment variants, interleaved: bash scripts/env_ab.sh "VAR=val" ["VAR2=val" ...] -- [bench args]
vars=(); while [ $# -gt 0 ] && [ "$1" != "--" ]; do vars+=("$1"); shift; done; shift
for rep in 1 2 3; do for v in "" "${vars[@]}"; do
  env $v timeout 300 python bench.py --steps 100 --warmup 3 --no-e2e --no-cpu-baseline --no-sampler-ceiling "$@" | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('${v:-default}', '$*', 'step', round(d['ms_per_step'],4), 'march', round(d['march_ms_per_step'],4), 'build', round(d['layout_ms_per_step'],4))"
done; done
