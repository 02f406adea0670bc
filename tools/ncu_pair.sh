#!/bin/bash
# ncu --set full of the CTA-pair GEMM2 (third gemm launch of a step).
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
DSMOE_B200_CTA_PAIR=12 STEPS=1 timeout 600 ncu --set full --clock-control none --import-source on --profile-from-start off \
   -k regex:gemm_tc_kernel --launch-skip 2 --launch-count 1 -o gpurun_out/pair_g2 -f python tools/profile_step.py > gpurun_out/pair_g2.log 2>&1; echo "rc=$?"
