set -u
o=gpurun_out/ab1; mkdir -p $o
python scripts/ab_run.py base ftz pf pf48 --reps 3 --steps 100 --bench-args "--config C2" > $o/c2.txt 2>&1
python scripts/ab_run.py base ftz pf pf48 --reps 2 --steps 20 --bench-args "--config C3 --frames 16" > $o/c3.txt 2>&1
python scripts/ab_run.py base ftz pf pf48 --reps 2 --steps 3 --bench-args "--config C5 --frames 32" > $o/c5.txt 2>&1
NSL_LIB=$PWD/abl/libnsl_pf.so timeout 900 python -m pytest tests -m gpu -q -x > $o/tests_pf.log 2>&1; echo rc=$? >> $o/tests_pf.log
