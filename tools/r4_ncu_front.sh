#!/bin/bash
# ncu --set full of the front-end kernels (gate_route, permute) of one C2 step, with source
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
TAG=${1:-front}
STEPS=1 timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off \
   -k "regex:gate_route|permute" -o gpurun_out/prof_$TAG -f python tools/profile_step.py > gpurun_out/ncu_$TAG.log 2>&1; echo "ncu rc=$?"
