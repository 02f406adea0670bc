#!/bin/bash
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_gate_route.py tests/test_gpu_parity.py tests/test_gpu_benched.py tests/test_gpu_rate.py tests/test_gpu_ep.py -m gpu -q -x > gpurun_out/pytest_gr2.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gr2.log
DROP=0.25 STEPS=3 timeout 600 ncu --metrics gpu__time_duration.sum,sm__cycles_elapsed.max,dram__bytes_read.sum --clock-control none \
    --profile-from-start off --csv --log-file gpurun_out/gr2_list.csv python tools/profile_step.py > gpurun_out/gr2_list.log 2>&1; echo "list rc=$?"
timeout 600 python bench.py --steps 20 --warmup 5 --extra "" --no-ep > gpurun_out/bench_gr2.json 2> gpurun_out/bench_gr2.err; echo "bench rc=$?"; tail -c 1500 gpurun_out/bench_gr2.json
