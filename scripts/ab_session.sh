set -u
o=gpurun_out/ab21; mkdir -p $o
python scripts/ab_run.py base mel --reps 3 --steps 100 --bench-args "--config C2" > $o/c2.txt 2>&1
python scripts/ab_run.py base mel --reps 2 --steps 3 --bench-args "--config C5 --frames 32" > $o/c5.txt 2>&1
python scripts/ab_run.py base mel --reps 2 --steps 20 --bench-args "--config C3 --frames 16" > $o/c3.txt 2>&1
