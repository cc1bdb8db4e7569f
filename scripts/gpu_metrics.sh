# quick ncu metric comparison of library variants on the C2 march kernel
bash scripts/build_variants.sh
M=gpu__time_duration.sum,smsp__inst_executed.sum,smsp__thread_inst_executed.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__warps_active.avg.pct_of_peak_sustained_active,smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio,smsp__average_warps_issue_stalled_wait_per_issue_active.ratio,smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio,smsp__average_warps_issue_stalled_no_instruction_per_issue_active.ratio,smsp__average_warps_issue_stalled_branch_resolving_per_issue_active.ratio,l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed
for lib in ${LIBS}; do
  NSL_LIB=$lib timeout 300 python scripts/profile_march.py > /dev/null 2>&1 && \
  NSL_LIB=$lib timeout 600 ncu --metrics $M --clock-control none -k regex:march_kernel -s 2 -c 1 --csv python scripts/profile_march.py 2>/dev/null | grep -E '"march_kernel|gpu__|smsp__|sm__|l1tex' | awk -F'","' -v L=$lib '{print L" "$(NF-2)" "$(NF)}' | sed 's/"//g'
done
