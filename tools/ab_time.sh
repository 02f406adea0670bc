#!/bin/bash
# Interleaved A/B of library variants by wall-clock device time (CUDA events,
# back-to-back forwards: PDL overlap and power-capped clocks included).
# Usage: VARIANTS="X=0 DSMOE_B200_LIB=build/variants/nopdl/libdsmoe_b200.so" bash tools/ab_time.sh
cd ${GRAFT_REPO_ROOT:-.}
for rep in 1 2 3; do
for v in ${VARIANTS:-X=0}; do
  printf "%-60s " "$v"
  env ${v//,/ } timeout 300 python - <<'PY'
import os, sys, torch
sys.path.insert(0, ".")
import bench, paper_2508_18376_b200 as D
torch.cuda.set_device(0)
ctx = D.Context()
layer, _ = bench.build_layer("c2", ctx)
x = torch.randn(16384, 2048, device="cuda", generator=torch.Generator(device="cuda").manual_seed(3)).bfloat16()
out = torch.empty_like(x)
res = []
for tg in (0.0, 0.25):
    pol, _ = bench.calibrate(ctx, layer, x, tg)
    ms = bench.time_steps(lambda: D.forward(ctx, layer, x, pol, out=out), 100, 10) / 100
    res.append(ms)
print(" ".join(f"{m:.4f}" for m in res), f"speedup {res[0]/res[1]:.3f}")
PY
done; done
