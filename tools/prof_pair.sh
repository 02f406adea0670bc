#!/bin/bash
cd ${GRAFT_REPO_ROOT:-.}
timeout 300 python -m pytest tests/test_gpu_parity.py -m gpu -q -x 2>&1 | tail -2
timeout 120 python tools/probe_c2.py 2>&1 | tail -2 | cut -c1-400
STEPS=1 timeout 600 ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:gemm_tc2 -c 2 -o gpurun_out/prof_pair -f python tools/profile_step.py > gpurun_out/ncu_pair.log 2>&1; echo ncu=$?
