#!/bin/bash
# ncu --set full of GEMM1 (gemm_tc_kernel<1>) at C2 25% drop: fused-gather vs explicit X_perm.
cd ${GRAFT_REPO_ROOT:-.}
TAG=${1:-g1}
mkdir -p gpurun_out
STEPS=1 timeout 600 ncu --set full --clock-control none --import-source on --profile-from-start off \
   -k regex:gemm_tc_kernel --launch-skip 1 --launch-count 1 -o gpurun_out/${TAG}_fused -f python tools/profile_step.py > gpurun_out/${TAG}_fused.log 2>&1; echo "fused rc=$?"
DSMOE_B200_GATHER=explicit STEPS=1 timeout 600 ncu --set full --clock-control none --import-source on --profile-from-start off \
   -k regex:gemm_tc_kernel --launch-skip 1 --launch-count 1 -o gpurun_out/${TAG}_explicit -f python tools/profile_step.py > gpurun_out/${TAG}_explicit.log 2>&1; echo "explicit rc=$?"
