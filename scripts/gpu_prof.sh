export NSL_OCC_SHIFT=${NSL_OCC_SHIFT:-2}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 300 python scripts/profile_march.py > gpurun_out/prof_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:march_kernel -s 2 -c 1 -o gpurun_out/prof_march_${TAG:-x} -f python scripts/profile_march.py > gpurun_out/ncu_full.log 2>&1; echo "ncu rc=$?"; tail -3 gpurun_out/ncu_full.log
