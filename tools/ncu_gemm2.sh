#!/bin/bash
# ncu --set full of GEMM2 (third gemm_tc launch of a step) at C2 25% drop.
cd ${GRAFT_REPO_ROOT:-.}
TAG=${1:-g2}
mkdir -p gpurun_out
STEPS=1 timeout 600 ncu --set full --clock-control none --import-source on --profile-from-start off \
   -k regex:gemm_tc_kernel --launch-skip 2 --launch-count 1 -o gpurun_out/${TAG} -f python tools/profile_step.py > gpurun_out/${TAG}.log 2>&1; echo "rc=$?"
