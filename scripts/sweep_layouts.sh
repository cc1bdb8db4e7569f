for layout in quad_f32 corner_f16 linear_f32; do
  r=$(timeout 300 python bench.py --steps 50 --warmup 3 --no-e2e --no-cpu-baseline --layout $layout 2>&1 | tail -1)
  python -c "
import json,sys
d=json.loads(sys.argv[1]); c=d['counts_per_rank_step']
print('$layout', 'march_ms=%.3f'%d['march_ms_per_step'], 'rays/s=%.3e'%d['value'])" "$r"
done
