"""Segment tails of every size class through the grouped GEMMs: a caller-
supplied routing (moe_forward, moe.hpp:239) gives each expert an exact count
of full rows and major-only rows, so tiles end at 1, 63, 64, 65, 127, 128,
129, 255, 256 and 257 rows — the M = 128 CTA-pair tails (<= 128 rows, one or
both CTAs holding rows), M = 256 tiles, and the single-CTA path for widths
whose N is not a multiple of 128."""
import os
import subprocess
import sys

import numpy as np
import pytest

import oracle as O

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

# (full rows, major-only rows) per expert
COUNTS = [(1, 0), (63, 1), (64, 64), (65, 63), (127, 128), (128, 129), (129, 0), (255, 2), (256, 1), (257, 65),
          (0, 0), (0, 7)]


def scaled_residual(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    den = max(np.abs(a).max(), np.abs(b).max())
    return 0.0 if den == 0 else float(np.abs(a - b).max() / den)


def _case(ffn, seed):
    import paper_2508_18376_b200 as D
    E, K, d = len(COUNTS), 1, 256
    L = O.partial_transform(O.generate_layer(d, ffn, E, K, seed=seed), 2)
    dl = D.MoeLayer(L.d, L.ffn, L.E, L.K, L.gate, L.blocks, L.shared, replay_factor=2, dtype="bf16")
    rows = [(e, 1.0) for e, (nf, nm) in enumerate(COUNTS) for _ in range(nf)] + \
           [(e, 0.0) for e, (nf, nm) in enumerate(COUNTS) for _ in range(nm)]
    rng = np.random.default_rng(seed)
    rng.shuffle(rows)
    T = len(rows)
    idx = np.array([[2 * e, 2 * e + 1] for e, _ in rows], np.int32)
    raw = rng.uniform(0.2, 1.0, size=(T, 1)).repeat(2, axis=1)
    frac = np.array([[1.0, f] for _, f in rows])
    x = O.bf16_round(O.generate_tokens(T, d, seed=seed + 1))
    ctx = D.Context()
    y = D.moe_forward(ctx, dl, torch.from_numpy(x).cuda().bfloat16(),
                      (torch.from_numpy(idx), torch.from_numpy(raw), torch.from_numpy(frac)))
    yo = O.moe_forward(L, x, idx, raw, frac)
    return scaled_residual(y.float().cpu().numpy(), yo)


@pytest.mark.parametrize("ffn", [256, 128, 384])
def test_tail_sizes(ffn):
    torch.cuda.set_device(0)
    assert _case(ffn, 71 + ffn) < 1e-2


@pytest.mark.parametrize("pair", ["0", "1", "2", "12"])
def test_tail_sizes_cta_variants(pair):
    """Same cases with single-CTA tiles ("0"), pairs on one GEMM ("1": GEMM2
    tiles nest in GEMM1 tiles -> unified GEMM2 tiles; "2": they do not ->
    full / major-only GEMM2 tiles) and pairs on both."""
    code = (f"import sys; sys.path.insert(0, {os.path.dirname(os.path.dirname(os.path.abspath(__file__)))!r}); "
            "sys.path.insert(0, %r); import torch; torch.cuda.set_device(0); import test_gpu_tails as t; "
            "print('RES', max(t._case(f, 71 + f) for f in (256, 128)))" % os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-c", code], env={**os.environ, "DSMOE_B200_CTA_PAIR": pair},
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    assert float([l for l in r.stdout.splitlines() if l.startswith("RES")][-1].split()[1]) < 1e-2
