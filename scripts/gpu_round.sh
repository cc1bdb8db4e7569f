# full round-1 evidence run: tests, smoke, bench (+reference arm), ncu launch list, ncu full profile
set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/smi.txt; nproc >> gpurun_out/smi.txt
timeout 1200 python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
timeout 300 python scripts/bench_relight.py > gpurun_out/bench_relight.json 2>&1; echo "relight rc=$?"
timeout 300 python scripts/bench_bake.py > gpurun_out/bench_bake.json 2>&1; echo "bake rc=$?"
timeout 600 python bench.py --impl reference --steps 10 --warmup 3 > gpurun_out/bench_ref.json 2>&1; echo "ref rc=$?"
CMD="python bench.py --steps 3 --warmup 1 --no-e2e --no-cpu-baseline --no-sampler-ceiling"
timeout 300 $CMD > gpurun_out/launch_plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/launch_ncu.log 2>&1; echo "launch-list rc=$?"
timeout 300 python scripts/profile_march.py > gpurun_out/prof_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:march_kernel -s 2 -c 1 -o gpurun_out/prof_march_${TAG:-r1} -f python scripts/profile_march.py > gpurun_out/ncu_full.log 2>&1; echo "ncu rc=$?"
