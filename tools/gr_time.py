"""ncu target: C2 forwards at a fixed 2T threshold (no calibration), for A/B
of gate_route variants (diagnostic builds may route wrongly)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
import paper_2508_18376_b200 as D
torch.cuda.set_device(0)
ctx = D.Context()
layer, _ = bench.build_layer("c2", ctx)
x = bench.bench_tokens("c2", int(os.environ.get("T", "16384"))).cuda()
pol = D.DropPolicy.two_t_from(0.085)
for _ in range(3):
    D.forward(ctx, layer, x, pol)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()
for _ in range(int(os.environ.get("STEPS", "3"))):
    D.forward(ctx, layer, x, pol)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
