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
    nm = nt - nf  # major-only rows
    out = {"target": tg, "drop": rate, "rows": int(R), "full_rows": int(nf.sum())}
    for M in (128, 256):  # single-CTA tiles / CTA-pair tiles
        c = lambda n: (n + M - 1) // M
        # GEMM1: 4 chunks over all rows (major half) + 4 over the full rows (minor half)
        g1_issued = ((c(nt) + c(nf)) * 4 * M).sum()
        g1_useful = ((nt + nf) * 4).sum()
        # GEMM2: full-row tiles run K = 1024, major-only tiles K = 512 (separate tiles)
        g2_issued = ((c(nf) * 1024 + c(nm) * 512) * M).sum()
        g2_useful = (nf * 1024 + nm * 512).sum()
        out[f"g1_waste_m{M}"] = float(1 - g1_useful / g1_issued)
        out[f"g2_waste_m{M}"] = float(1 - g2_useful / g2_issued)
    print(json.dumps(out))
