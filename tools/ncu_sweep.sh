#!/bin/bash
# Per-kernel cycles (clock-independent) and durations of one C2 forward at
# 0 / 25 / 50 % 2T drop (ncu, serialised, --clock-control none), plus one
# `ncu --set full` capture of every kernel at 25 % (traffic, tensor-pipe,
# DRAM throughput).  Usage: bash tools/ncu_sweep.sh TAG [CFG]
cd ${GRAFT_REPO_ROOT:-.}
TAG=${1:-r2}
CFG=${2:-c2}
mkdir -p gpurun_out
M=gpu__time_duration.sum,sm__cycles_elapsed.max,sm__cycles_active.avg,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_active
for D in 0.0 0.25 0.5; do
  CFG=$CFG DROP=$D STEPS=1 timeout 600 ncu --metrics $M --clock-control none --profile-from-start off --csv \
     --log-file gpurun_out/sweep_${TAG}_${CFG}_$D.csv python tools/profile_step.py > gpurun_out/sweep_${TAG}_${CFG}_$D.log 2>&1
  echo "drop $D rc=$?"
done
CFG=$CFG DROP=0.25 STEPS=1 timeout 1200 ncu --set full --clock-control none --import-source on --profile-from-start off \
   -o gpurun_out/prof_all_${TAG}_${CFG} -f python tools/profile_step.py > gpurun_out/ncu_all_${TAG}_${CFG}.log 2>&1; echo "ncu-all rc=$?"
python tools/ncu_summary.py gpurun_out/prof_all_${TAG}_${CFG}.ncu-rep gpurun_out/${TAG}_${CFG}_ncu_all_kernels.json > /dev/null 2>&1; echo "summary rc=$?"
