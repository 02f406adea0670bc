"""Host-side cost of one D.forward call (no sync): must stay well below the
device step time so the GPU never waits on the launcher."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
import paper_2508_18376_b200 as D
torch.cuda.set_device(0)
ctx = D.Context()
layer, _ = bench.build_layer("c2", ctx)
x = torch.randn(16384, 2048, device="cuda").bfloat16()
out = torch.empty_like(x)
pol, _ = bench.calibrate(ctx, layer, x, 0.25)
for _ in range(5):
    D.forward(ctx, layer, x, pol, out=out)
torch.cuda.synchronize()
n = 50
t0 = time.perf_counter()
for _ in range(n):
    D.forward(ctx, layer, x, pol, out=out)
t1 = time.perf_counter()
torch.cuda.synchronize()
t2 = time.perf_counter()
print(f"host enqueue per forward {1e3 * (t1 - t0) / n:.3f} ms, device per forward {1e3 * (t2 - t0) / n:.3f} ms")
