"""Diagnostic: phase durations of the fused permutation kernel (variant build
with -DDSB_PERMUTE_PHASES=1) on the C2 bench step."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
import paper_2508_18376_b200 as D
torch.cuda.set_device(0)
ctx = D.Context()
layer, _ = bench.build_layer("c2", ctx)
x = bench.bench_tokens("c2", 16384).cuda()
pol, _ = bench.calibrate(ctx, layer, x, 0.25)
for _ in range(3):
    D.forward(ctx, layer, x, pol)
torch.cuda.synchronize()
print("---")
for _ in range(2):
    D.forward(ctx, layer, x, pol)
torch.cuda.synchronize()
