#!/bin/bash
# EP checks on one GPU: tests, the 1-rank NCCL bench line, a 2-rank gloo bench line.
TAG=${1:-r2d}
SEL=${2:-"tests/test_gpu_ep_multirank.py tests/test_gpu_ep_mixtral.py tests/test_gpu_ep.py"}
mkdir -p gpurun_out
timeout 1500 python -m pytest $SEL -m gpu -x -q > gpurun_out/pytest_$TAG.log 2>&1; echo "pytest rc=$?"; tail -25 gpurun_out/pytest_$TAG.log
timeout 900 python bench.py --ep --steps 10 --warmup 3 > gpurun_out/bench_ep1_$TAG.json 2> gpurun_out/bench_ep1_$TAG.err; echo "ep1 rc=$?"; tail -c 2500 gpurun_out/bench_ep1_$TAG.json; tail -5 gpurun_out/bench_ep1_$TAG.err
DSMOE_B200_EP_BACKEND=gloo timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 5 --warmup 3 > gpurun_out/bench_ep2_$TAG.json 2> gpurun_out/bench_ep2_$TAG.err; echo "ep2 rc=$?"; tail -c 2500 gpurun_out/bench_ep2_$TAG.json; tail -5 gpurun_out/bench_ep2_$TAG.err
