set -u
o=gpurun_out/ab2; mkdir -p $o
python scripts/ab_run.py base occ32 --reps 3 --steps 100 --bench-args "--config C2" > $o/c2.txt 2>&1
python scripts/ab_run.py base occ32 --reps 2 --steps 20 --bench-args "--config C3 --frames 16" > $o/c3.txt 2>&1
python scripts/ab_run.py base occ32 --reps 2 --steps 3 --bench-args "--config C5 --frames 32" > $o/c5.txt 2>&1
timeout 900 python -m pytest tests -m gpu -q -x > $o/tests.log 2>&1; echo rc=$? >> $o/tests.log
