set -u
o=gpurun_out/ab4; mkdir -p $o
bash scripts/ab_bake.sh bk0 bk1 > $o/bake.txt 2>&1
python scripts/ab_run.py bk0 bk1 --reps 2 --steps 100 --bench-args "--config C2" > $o/c2.txt 2>&1
timeout 900 python -m pytest tests -m gpu -q -x > $o/tests.log 2>&1; echo rc=$? >> $o/tests.log
