# Final round-2 evidence on one GPU: scripts/evidence_r2.sh (tests, smoke, bench, reference arm,
# launch list, per-config lines) plus one ncu --set full capture of the C2 march.
set -u
bash scripts/evidence_r2.sh
timeout 300 python scripts/profile_march.py > gpurun_out/r2ev/prof_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:march_kernel -s 2 -c 1 \
    -o gpurun_out/r2ev/march_C2_full -f python scripts/profile_march.py > gpurun_out/r2ev/ncu_full.log 2>&1
echo "ncu rc=$?" >> gpurun_out/r2ev/ncu_full.log
