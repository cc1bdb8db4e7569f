# Round-2 evidence run (one GPU): the GPU test suite, smoke(), the default bench and the reference
# arm, the ncu launch list of the bench command, per-config lines.  Usage: bash scripts/evidence_r2.sh
set -u
o=gpurun_out/r2ev
mkdir -p $o
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $o/smi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q > $o/gpu_tests.log 2>&1; echo "rc=$?" >> $o/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $o/smoke.log 2>&1; echo "rc=$?" >> $o/smoke.log
timeout 300 python bench.py > $o/bench.json 2> $o/bench.err
timeout 300 python bench.py --impl reference --steps 20 --warmup 5 > $o/bench_reference.json 2> $o/bench_reference.err
timeout 300 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --no-sampler-ceiling > $o/plain.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $o/launches.csv \
      python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --no-sampler-ceiling > $o/ncu.log 2>&1
bash scripts/per_config.sh $o
