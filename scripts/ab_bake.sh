# A/B of bake variants built by scripts/ab_local.sh: bash scripts/ab_bake.sh NAME [NAME ...]
for rep in 1 2; do for v in "$@"; do
  NSL_LIB=abl/libnsl_$v.so timeout 300 python scripts/bench_bake.py --no-oracle --steps 5 | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$v', round(d['ms_per_frame'],3), 'frac', round(d['roofline']['frac'],3), 'peak', round(d['roofline']['peak']))"
done; done
