set -u
o=gpurun_out/ab5; mkdir -p $o
python scripts/ab_run.py cf0 cf1 --reps 3 --steps 100 --bench-args "--config C2" > $o/c2.txt 2>&1
python scripts/ab_run.py cf0 cf1 --reps 2 --steps 20 --bench-args "--config C3 --frames 16" > $o/c3.txt 2>&1
python scripts/ab_run.py cf0 cf1 --reps 2 --steps 3 --bench-args "--config C5 --frames 32" > $o/c5.txt 2>&1
python scripts/ab_run.py cf0 cf1 --reps 2 --steps 50 --bench-args "--config C1" > $o/c1.txt 2>&1
