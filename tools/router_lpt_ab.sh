#!/bin/bash
# A/B: router lanes per token (4 vs 8) — ncu times of gate / router / permute at C2 25%; permutation phases.
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
for L in 4 8; do
  DSMOE_B200_ROUTER_LPT=$L DROP=0.25 STEPS=3 timeout 600 ncu --metrics gpu__time_duration.sum,sm__cycles_elapsed.max --clock-control none \
    --profile-from-start off --csv --log-file gpurun_out/router_lpt_$L.csv python tools/profile_step.py > gpurun_out/router_lpt_$L.log 2>&1
  echo "lpt $L rc=$?"
done
DSMOE_B200_LIB=build/variants/perm_phases/libdsmoe_b200.so timeout 300 python tools/permute_phases.py > gpurun_out/permute_phases.txt 2>&1; echo "phases rc=$?"; tail -6 gpurun_out/permute_phases.txt
DSMOE_B200_ROUTER_LPT=8 timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_permute.py -m gpu -q -x > gpurun_out/pytest_lpt8.log 2>&1; echo "lpt8 tests rc=$?"; tail -3 gpurun_out/pytest_lpt8.log
