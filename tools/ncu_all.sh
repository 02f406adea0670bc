#!/bin/bash
# Full ncu capture of every kernel of one C2 forward step (25% drop) + launch list.
cd ${GRAFT_REPO_ROOT:-.}
TAG=${1:-r08}
mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv \
   --log-file gpurun_out/launches_$TAG.csv python tools/profile_step.py > gpurun_out/ncu_launch_$TAG.log 2>&1; echo "ncu-list rc=$?"
STEPS=1 timeout 1200 ncu --set full --clock-control none --import-source on --profile-from-start off \
   -o gpurun_out/prof_all_$TAG -f python tools/profile_step.py > gpurun_out/ncu_all_$TAG.log 2>&1; echo "ncu-all rc=$?"
