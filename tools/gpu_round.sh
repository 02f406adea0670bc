#!/bin/bash
# One GPU session: tests, smoke, bench, ncu launch list + full capture.
# Usage (from the repo root on the GPU box): bash tools/gpu_round.sh [tag] [ncu kernel regex]
TAG=${1:-r01}
KRE=${2:-"gemm_tc_kernel|router_kernel|scan_codes|seg_plan"}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/gpu_$TAG.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; echo "smoke rc=$?"
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?"; tail -15 gpurun_out/pytest_gpu_$TAG.log
timeout 900 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; echo "bench rc=$?"; tail -c 2500 gpurun_out/bench_$TAG.json; tail -3 gpurun_out/bench_$TAG.err
if [ "${NCU:-1}" = "1" ]; then
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv \
     --log-file gpurun_out/launches_$TAG.csv python tools/profile_step.py > gpurun_out/ncu_launch_$TAG.log 2>&1; echo "ncu-list rc=$?"
  STEPS=1 timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off \
     -k "regex:$KRE" -o gpurun_out/prof_$TAG -f python tools/profile_step.py > gpurun_out/ncu_full_$TAG.log 2>&1; echo "ncu-full rc=$?"
fi
