cd ${GRAFT_REPO_ROOT:-.}
for v in ${TCV:-0 8}; do
DSMOE_B200_GATHER=explicit DSMOE_B200_GEMM_FLAGS=$v STEPS=1 timeout 300 ncu --metrics gpu__time_duration.sum,sm__cycles_elapsed.max,sm__pipe_tc_cycles_active.sum,sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_tc.sum,sm__pipe_tensor_op_hmma_cycles_active.sum --clock-control none --profile-from-start off -k regex:gemm_tc_kernel --launch-skip ${SKIP:-1} --launch-count 1 python tools/profile_step.py 2>&1 | grep -E "gpu__|sm__" ; echo "-- flags $v"; done
