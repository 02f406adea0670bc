"""CUDA-graph capture of the forward (serving): capture D.forward on the
context's stream once per token count, replay, compare with eager and time
both at small T."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
import paper_2508_18376_b200 as D
torch.cuda.set_device(0)
s = torch.cuda.Stream()
ctx = D.Context(stream=s)
layer, _ = bench.build_layer("c2", ctx)
pol = D.DropPolicy.two_t_from(0.08)
for T in (1, 8, 64, 512):
    x = torch.randn(T, 2048, device="cuda").bfloat16()
    out = torch.empty_like(x)
    with torch.cuda.stream(s):
        for _ in range(3):
            D.forward(ctx, layer, x, pol, out=out)
        s.synchronize()
        ref = out.clone()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            D.forward(ctx, layer, x, pol, out=out)
        out.zero_()
        g.replay()
        s.synchronize()
        same = torch.equal(out, ref)
        n = 200
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        for _ in range(n):
            g.replay()
        e1.record(s)
        s.synchronize()
        tg = e0.elapsed_time(e1) / n * 1e3
        e0.record(s)
        for _ in range(n):
            D.forward(ctx, layer, x, pol, out=out)
        e1.record(s)
        s.synchronize()
        te = e0.elapsed_time(e1) / n * 1e3
    print(f"T={T:4d} graph==eager {same}  graph {tg:7.1f} us  eager {te:7.1f} us")
