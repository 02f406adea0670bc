#!/bin/bash
# Router / permutation evidence: ncu --set full with source of the router and
# permutation kernels, router lanes-per-token A/B, permutation phase times.
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
STEPS=1 timeout 600 ncu --set full --clock-control none --import-source on --profile-from-start off \
  -k "regex:router_quad|permute_fused|gemm_tc_kernel<0" -o gpurun_out/prof_router -f python tools/profile_step.py > gpurun_out/ncu_router.log 2>&1; echo "ncu rc=$?"
bash tools/router_lpt_ab.sh
