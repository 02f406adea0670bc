#!/bin/bash
# A/B of the gate K split at T = 16384 (C2, 25% drop): per-kernel ncu times for S = 1 and S = 2.
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
for S in 1 2; do
  DSMOE_B200_GATE_SPLIT=$S DROP=0.25 STEPS=3 timeout 600 ncu --metrics gpu__time_duration.sum,sm__cycles_elapsed.max --clock-control none \
    --profile-from-start off --csv --log-file gpurun_out/gate_split_$S.csv python tools/profile_step.py > gpurun_out/gate_split_$S.log 2>&1
  echo "split $S rc=$?"
done
