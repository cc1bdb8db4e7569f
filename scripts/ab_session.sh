set -u
o=gpurun_out/ab12; mkdir -p $o
python scripts/ab_run.py pl0 pl1 --reps 3 --steps 20 --bench-args "--config C3 --frames 16" > $o/c3.txt 2>&1
python scripts/ab_run.py pl0 pl1 --reps 2 --steps 100 --bench-args "--config C2" > $o/c2.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -q -x > $o/tests.log 2>&1; echo rc=$? >> $o/tests.log
