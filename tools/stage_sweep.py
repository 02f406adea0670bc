"""Per-stage device time (CUDA events, back-to-back forwards) at 0/25/50% 2T
drop on the bench layer: which stages shrink with the drop rate."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
import paper_2508_18376_b200 as D
torch.cuda.set_device(0)
ctx = D.Context()
cfg = os.environ.get("CFG", "c2")
layer, _ = bench.build_layer(cfg, ctx)
x = torch.randn(16384, bench.CONFIGS[cfg][0], device="cuda").bfloat16()
out = torch.empty_like(x)
res = {}
for tg in (0.0, 0.25, 0.5):
    pol, rate = bench.calibrate(ctx, layer, x, tg)
    for _ in range(20):
        D.forward(ctx, layer, x, pol, out=out)
    ctx.set_profiling(True)
    for _ in range(60):
        D.forward(ctx, layer, x, pol, out=out)
    p = ctx.profile()
    ctx.set_profiling(False)
    res[tg] = {k: 1e3 * p[k] / p["calls"] for k in ctx.STAGES}
    print(f"drop {rate:.3f}: " + "  ".join(f"{k} {v:6.1f}" for k, v in res[tg].items()) + f"  total {sum(res[tg].values()):7.1f} us")
for k in ctx.STAGES:
    if res[0.0][k] > 0:
        print(f"{k:13s} 25%: {res[0.25][k] / res[0.0][k]:.3f}  50%: {res[0.5][k] / res[0.0][k]:.3f}")
