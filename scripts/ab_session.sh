set -u
o=gpurun_out/v20; mkdir -p $o
timeout 1200 python -m pytest tests -m gpu -q -x > $o/tests.log 2>&1; echo rc=$? >> $o/tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $o/smoke.log 2>&1; echo rc=$? >> $o/smoke.log
timeout 300 python bench.py > $o/bench.json 2> $o/bench.err
