M=""
for s in no_instruction branch_resolving long_scoreboard short_scoreboard wait barrier membar sleeping dispatch_stall misc mio_throttle lg_throttle math_pipe_throttle drain selected not_selected tex_throttle imc_miss; do M="$M,smsp__average_warps_issue_stalled_${s}_per_issue_active.ratio"; done
M="gpu__time_duration.sum,smsp__inst_executed.sum,sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active$M"
for v in codec3 codec4; do
ncu --metrics $M --kernel-name regex:gemm_tc_kernel --launch-skip 0 --launch-count 1 --csv python tools/profile_kernels.py --mu 64 --only "expert gate" --once --$v > gpurun_out/stalls_$v.csv 2>/dev/null
done
