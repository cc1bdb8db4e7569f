set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 1200 python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?"
tail -40 gpurun_out/gpu_tests.log
timeout 600 python bench.py > gpurun_out/bench.log 2>&1; echo "bench rc=$?"; tail -c 2500 gpurun_out/bench.log
timeout 300 python scripts/profile_march.py > gpurun_out/prof_plain.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:march_kernel -s 2 -c 1 -o gpurun_out/prof_march_r1 -f python scripts/profile_march.py > gpurun_out/ncu_full.log 2>&1; echo "ncu rc=$?"; tail -5 gpurun_out/ncu_full.log
