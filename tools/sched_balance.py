"""Per-pair work of the grouped GEMMs under the static round-robin tile
schedule (tile i -> CTA pair i mod 74), from the C2 bench routing at 0/25/50%:
max / mean pair cost = the tail the persistent kernels wait for.  Tile costs in
MMA cycles of one SM (M = 256 pair tile: 1; half-M tail: 0.5) x K blocks x N/256."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import bench
import paper_2508_18376_b200 as D

cfg = os.environ.get("CFG", "c2")
torch.cuda.set_device(0)
ctx = D.Context()
layer, _ = bench.build_layer(cfg, ctx)
d = bench.CONFIGS[cfg][0]
x = bench.bench_tokens(bench.base_cfg(cfg), 16384).cuda()
P = 74
cd = lambda a, b: -(-a // b)
out = {}
for tg in (0.0, 0.25, 0.5):
    pol, rate = bench.calibrate(ctx, layer, x, tg)
    seg, R, _ = D.dispatch(ctx, layer, x, pol)
    np.save(f"gpurun_out/seg_{cfg}_{int(tg*100)}.npy", seg)
    c1, c2 = [], []
    for u in range(seg.shape[0]):
        nf, nt = int(seg[u, 1]), int(seg[u, 2])
        wpad = [512, 512]  # C2: two sub-blocks of 512 neurons, 128-neuron N chunks
        mt_all, mt_full = cd(nt, 256), cd(nf, 256)
        for mt in range(mt_all):
            for p, w in enumerate(wpad):
                if p == 1 and mt >= mt_full:
                    continue
                for c in range(cd(w, 128)):
                    mv = min(256, (nt - mt * 256))
                    c1.append((0.5 if mv <= 128 else 1.0) * (d // 64))
        for mt in range(cd(nt, 256)):
            full = mt * 256 < nf
            mv = min(256, nt - mt * 256)
            for nt_ in range(cd(d, 256)):
                c2.append((0.5 if mv <= 128 else 1.0) * (16 if full else 8))
    res = {"drop": rate}
    for name, c in (("gemm1", c1), ("gemm2", c2)):
        c = np.array(c)
        load = np.zeros(P)
        for i, v in enumerate(c):
            load[i % P] += v
        # greedy longest-first (ideal static balance) for comparison
        g = np.zeros(P)
        for v in sorted(c, reverse=True):
            g[g.argmin()] += v
        res[name] = {"tiles": len(c), "rr_max_over_mean": round(load.max() / load.mean(), 4),
                     "greedy_max_over_mean": round(g.max() / g.mean(), 4)}
    out[str(tg)] = res
    print(tg, res, flush=True)
json.dump(out, open("gpurun_out/sched_balance.json", "w"), indent=1)
