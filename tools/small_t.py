"""Per-forward device time and host enqueue time at small token counts (C2
layer): the launch-latency regime of decode-style serving."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
import paper_2508_18376_b200 as D
torch.cuda.set_device(0)
ctx = D.Context()
layer, _ = bench.build_layer(os.environ.get("CFG", "c2"), ctx)
d = bench.CONFIGS[os.environ.get("CFG", "c2")][0]
pol = D.DropPolicy.two_t_from(0.08)
for T in (1, 8, 64, 512, 4096):
    x = torch.randn(T, d, device="cuda").bfloat16()
    out = torch.empty_like(x)
    for _ in range(10):
        D.forward(ctx, layer, x, pol, out=out)
    torch.cuda.synchronize()
    n = 200
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    e0.record()
    for _ in range(n):
        D.forward(ctx, layer, x, pol, out=out)
    e1.record()
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    print(f"T={T:5d}  device {1e3 * e0.elapsed_time(e1) / n:8.1f} us/forward   host enqueue {1e6 * (t1 - t0) / n:8.1f} us/forward")
