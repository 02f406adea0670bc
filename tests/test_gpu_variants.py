"""Every grouped-GEMM variant the library can select stays at parity with the
oracle: CTA pairs for GEMM1 / GEMM2 / both / neither (DSMOE_B200_CTA_PAIR),
the explicit X_perm gather instead of the fused one (DSMOE_B200_GATHER) and
the split permutation (DSMOE_B200_PERMUTE), plain stream-ordered launches
(DSMOE_B200_PDL=0) and the unsplit gate (DSMOE_B200_GATE_SPLIT=1).  The switches are read once per
process, so each case runs in a fresh interpreter."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CASE = r"""
import sys, json
import numpy as np, torch
sys.path.insert(0, %(root)r)
import oracle as O
import paper_2508_18376_b200 as D
torch.cuda.set_device(0)
ctx = D.Context()
res = []
for (d, ffn, E, K, S, T, t) in [(512, 384, 16, 4, 1, 700, 0.3), (256, 256, 8, 2, 0, 333, 0.0)]:
    L = O.partial_transform(O.generate_layer(d, ffn, E, K, S=S, seed=d + T), 2)
    dl = D.MoeLayer(L.d, L.ffn, L.E, L.K, L.gate, L.blocks, L.shared, replay_factor=2, dtype="bf16")
    x = O.bf16_round(O.generate_tokens(T, d, seed=T))
    xd = torch.from_numpy(x).cuda().bfloat16()
    pol = D.DropPolicy.two_t_from(t) if t > 0 else D.DropPolicy()
    _, lg = D.route_and_drop(ctx, dl, xd, pol, return_logits=True)
    ro = O.route_from_logits(lg.cpu().numpy(), K, 2, "2t" if t > 0 else "none", t)
    y = D.forward(ctx, dl, xd, pol).float().cpu().numpy().astype(np.float64)
    yo = O.moe_forward(L, x, ro.idx, ro.raw, ro.frac).astype(np.float64)
    den = max(np.abs(y).max(), np.abs(yo).max())
    res.append(float(np.abs(y - yo).max() / den))
print("RESULT", json.dumps(res))
"""


@pytest.mark.parametrize("env", [
    {"DSMOE_B200_CTA_PAIR": "0"},
    {"DSMOE_B200_CTA_PAIR": "1"},
    {"DSMOE_B200_CTA_PAIR": "2"},
    {"DSMOE_B200_CTA_PAIR": "12", "DSMOE_B200_GATHER": "explicit"},
    {"DSMOE_B200_CTA_PAIR": "0", "DSMOE_B200_GATHER": "explicit", "DSMOE_B200_PERMUTE": "split"},
    {"DSMOE_B200_PDL": "0", "DSMOE_B200_GATE_SPLIT": "1"},
], ids=lambda e: ",".join(f"{k[11:]}={v}" for k, v in e.items()))
def test_gemm_variant_parity(env):
    r = subprocess.run([sys.executable, "-c", CASE % {"root": ROOT}], env={**os.environ, **env},
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    line = [l for l in r.stdout.splitlines() if l.startswith("RESULT")][-1]
    for resid in json.loads(line.split(" ", 1)[1]):
        assert resid < 1e-2
