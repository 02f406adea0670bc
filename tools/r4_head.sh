#!/bin/bash
# Validation at HEAD after a session restart: smoke, GPU suite, bench, reference arm, launch list.
cd ${GRAFT_REPO_ROOT:-.}
TAG=${1:-r4}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw,power.limit --format=csv > gpurun_out/gpu_$TAG.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; echo "smoke rc=$?"; tail -3 gpurun_out/smoke_$TAG.log
timeout 900 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; echo "bench rc=$?"; tail -c 1500 gpurun_out/bench_$TAG.json; tail -3 gpurun_out/bench_$TAG.err
timeout 600 ncu --metrics gpu__time_duration.sum,sm__cycles_elapsed.max,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --profile-from-start off --csv \
   --log-file gpurun_out/launches_$TAG.csv python tools/profile_step.py > gpurun_out/ncu_launch_$TAG.log 2>&1; echo "ncu-list rc=$?"
timeout 1800 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_all_$TAG.log 2>&1; echo "pytest rc=$?"; tail -8 gpurun_out/pytest_all_$TAG.log
