set -u
o=gpurun_out/ab9; mkdir -p $o
python scripts/ab_run.py pn1 pk --reps 3 --steps 100 --bench-args "--config C2" > $o/c2.txt 2>&1
python scripts/ab_run.py pn1 pk --reps 2 --steps 3 --bench-args "--config C5 --frames 32" > $o/c5.txt 2>&1
python scripts/ab_run.py pn1 pk --reps 2 --steps 5 --bench-args "--config C4 --frames 16" > $o/c4.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x > $o/tests.log 2>&1; echo rc=$? >> $o/tests.log
