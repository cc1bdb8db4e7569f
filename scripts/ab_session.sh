set -u
o=gpurun_out/ab7; mkdir -p $o
b() { r=$(env $1 timeout 300 python bench.py $2 --warmup 5 --no-e2e --no-cpu-baseline --no-sampler-ceiling 2>/dev/null | tail -1)
      python -c "import json,sys; d=json.loads(sys.argv[1]); print('$1', '$2', 'step', round(d['ms_per_step'],4), 'march', round(d['march_ms_per_step'],4), 'build', round(d['layout_ms_per_step'],4), 'frac', round(d['roofline']['frac'],4))" "$r" >> $o/ab.txt; }
for rep in 1 2; do
  b "NSL_SPLIT=0" "--config C1 --steps 200"
  b "NSL_SPLIT=1" "--config C1 --steps 200"
  b "NSL_CULL_EARLY_TILES=2048" "--config P482 --steps 50"
  b "NSL_CULL_EARLY_TILES=512" "--config P482 --steps 50"
  b "NSL_CULL_EARLY_TILES=2048" "--config P482 --steps 50 --layout brick_oct_f32"
  b "NSL_CULL_EARLY_TILES=512" "--config P482 --steps 50 --layout brick_oct_f32"
  b "NSL_CULL_EARLY_TILES=512" "--config C1 --steps 200"
done
