#!/bin/bash
# Round-2 (session r4) evidence at HEAD: superchunk tests, driver-style bench + reference arm,
# EP lines (1-rank NCCL, 2-rank gloo), ncu launch list, ncu --set full of every kernel of one step.
cd ${GRAFT_REPO_ROOT:-.}
TAG=${1:-r4}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw,power.limit --format=csv > gpurun_out/gpu_$TAG.txt
timeout 600 python -m pytest tests/test_gpu_superchunk.py -q -x > gpurun_out/pytest_sc_$TAG.log 2>&1; echo "sc tests rc=$?"; tail -2 gpurun_out/pytest_sc_$TAG.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; echo "bench rc=$?"; tail -c 600 gpurun_out/bench_$TAG.json
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/bench_ref_$TAG.json 2> gpurun_out/bench_ref_$TAG.err; echo "ref rc=$?"; tail -c 400 gpurun_out/bench_ref_$TAG.json
timeout 900 python bench.py --ep --steps 10 --warmup 3 > gpurun_out/bench_ep1_$TAG.json 2> gpurun_out/bench_ep1_$TAG.err; echo "ep1 rc=$?"; tail -c 400 gpurun_out/bench_ep1_$TAG.json
DSMOE_B200_EP_BACKEND=gloo timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 5 --warmup 3 > gpurun_out/bench_ep2_$TAG.json 2> gpurun_out/bench_ep2_$TAG.err; echo "ep2 rc=$?"; tail -c 400 gpurun_out/bench_ep2_$TAG.json
bash tools/ncu_all.sh $TAG
