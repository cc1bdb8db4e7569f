# Per-config bench lines: C2 (the headline), C1, C3, C4 (60 distinct volumes, and
# the whole 240-frame batch via --scaling strong), C5 (all 1024 frames; OCT and BRICK_OCT), each
# with roofline + cpu_baseline.  Usage (on a GPU box): bash scripts/per_config.sh OUTDIR
set -u
out=${1:-gpurun_out}
mkdir -p $out
timeout 300 python bench.py --steps 50 --warmup 5 > $out/bench_C2.json 2> $out/bench_C2.err
timeout 300 python bench.py --config C1 --steps 200 --warmup 5 > $out/bench_C1.json 2> $out/bench_C1.err
timeout 300 python bench.py --config C1 --frames 256 --steps 100 --warmup 5 --no-e2e > $out/bench_C1x256.json 2> $out/bench_C1x256.err
timeout 400 python bench.py --config C3 --steps 20 --warmup 3 > $out/bench_C3.json 2> $out/bench_C3.err
timeout 600 python bench.py --config C4 --frames 60 --steps 5 --warmup 3 > $out/bench_C4x60.json 2> $out/bench_C4x60.err
timeout 900 python bench.py --config C4 --scaling strong --steps 3 --warmup 2 > $out/bench_C4_strong240.json 2> $out/bench_C4_strong240.err
timeout 600 python bench.py --config C5 --steps 3 --warmup 3 --no-e2e --cpu-seconds 20 > $out/bench_C5.json 2> $out/bench_C5.err
timeout 600 python bench.py --config C5 --layout brick_oct_f32 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > $out/bench_C5_brick.json 2> $out/bench_C5_brick.err
timeout 300 python bench.py --config P482 --steps 50 --warmup 5 > $out/bench_P482.json 2> $out/bench_P482.err
