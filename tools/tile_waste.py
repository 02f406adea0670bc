"""Tile-quantisation waste of the grouped GEMMs at 0/25/50% drop on the bench
layer (C2): MMA rows issued vs rows that carry work."""
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
x = torch.randn(16384, bench.CONFIGS[cfg][0], device="cuda").to(torch.bfloat16)
for tg in (0.0, 0.25, 0.5):
    pol, rate = bench.calibrate(ctx, layer, x, tg)
    seg, R, _ = D.dispatch(ctx, layer, x, pol)
    nf, nt = seg[:, 1].astype(np.int64), seg[:, 2].astype(np.int64)
    c = lambda n: (n + 127) // 128
    # GEMM1: 4 chunks of major (all rows) + 4 of minor (full rows); GEMM2: K major or full per m-tile
    g1_issued = (c(nt) * 4 + c(nf) * 4) * 128
    g1_useful = nt * 4 + nf * 4
    g2_issued = sum((c(nt[u]) * 512 + min(c(nf[u]), c(nt[u])) * 512) * 128 for u in range(len(nt)))
    g2_useful = int((nt * 512 + nf * 512).sum())
    print(json.dumps({"target": tg, "drop": rate, "rows": int(R), "full_rows": int(nf.sum()),
                      "g1_waste": 1 - g1_useful.sum() / g1_issued.sum(), "g2_waste": 1 - g2_useful / g2_issued,
                      "min_tot": int(nt.min()), "max_tot": int(nt.max()), "min_full": int(nf.min()), "max_full": int(nf.max())}))
