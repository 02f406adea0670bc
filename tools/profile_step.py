"""Build the bench layer, calibrate, warm up, then run N forward steps inside
cudaProfilerStart/Stop so ncu (--profile-from-start off) sees only them."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2508_18376_b200 as D  # noqa: E402

cfg = os.environ.get("CFG", "c2")
drop = float(os.environ.get("DROP", "0.25"))
steps = int(os.environ.get("STEPS", "2"))
T = int(os.environ.get("T", "16384"))
torch.cuda.set_device(0)
ctx = D.Context()
layer, _ = bench.build_layer(cfg, ctx)
x = bench.bench_tokens(bench.base_cfg(cfg), T).cuda()
pol, rate = bench.calibrate(ctx, layer, x, drop)
for _ in range(3):
    D.forward(ctx, layer, x, pol)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()
for _ in range(steps):
    D.forward(ctx, layer, x, pol)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
print("drop_rate", rate, "launches/step", D.last_launch_count())
