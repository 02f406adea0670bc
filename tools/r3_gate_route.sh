#!/bin/bash
# Fused gate + router: parity tests, the routing-heavy GPU suites, launch list A/B (fused vs two kernels), bench.
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_gate_route.py tests/test_gpu_parity.py tests/test_gpu_benched.py tests/test_gpu_fullsize.py tests/test_gpu_rate.py tests/test_gpu_ep.py -m gpu -q -x > gpurun_out/pytest_gr.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/pytest_gr.log
for M in 1 0; do
  DSMOE_B200_GATE_ROUTE=$M DROP=0.25 STEPS=3 timeout 600 ncu --metrics gpu__time_duration.sum,sm__cycles_elapsed.max,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    --profile-from-start off --csv --log-file gpurun_out/gr_list_$M.csv python tools/profile_step.py > gpurun_out/gr_list_$M.log 2>&1
  echo "list $M rc=$?"
done
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_gr.json 2> gpurun_out/bench_gr.err; echo "bench rc=$?"; tail -c 1800 gpurun_out/bench_gr.json
STEPS=1 timeout 600 ncu --set full --clock-control none --import-source on --profile-from-start off \
  -k "regex:gate_route" -o gpurun_out/prof_gr -f python tools/profile_step.py > gpurun_out/ncu_gr.log 2>&1; echo "ncu rc=$?"
