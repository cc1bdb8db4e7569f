python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
if [ -z "$NOTEST" ]; then timeout 1200 python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?"; tail -5 gpurun_out/gpu_tests.log; fi
bash scripts/sweep.sh 2>&1 | tee gpurun_out/sweep.log
