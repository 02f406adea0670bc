"""Fused gate + router kernel (K0 + K1 in one launch, gate_route_kernel in
csrc/router.cu): the tensor-core gate GEMM of a 128-token tile and the
routing of that tile in the same CTA.

Bars: routing (indices, raw, normalized, fractions) and DropStats bit-exact
with the oracle's route_from_logits (dropping.hpp:248-258) on the logits the
kernel reports; those logits within 1e-5 of the exact fp32 matmul; and the
fused launch bit-identical (logits, routing, stats) to the two-kernel chain
(gate GEMM + router_quad_kernel, DSMOE_B200_GATE_ROUTE=0, run in a
subprocess because the switch is read once per process).  Cases cover
Epad 32 / 64 with E < Epad, K = 6 / 8 / 16, P = 1 / 2, batches from one
token to several tiles per CTA (T > 128 x 148), and T not a multiple of the
tile or of the 32-token chunk.
"""
import json
import os
import subprocess
import sys

import numpy as np
import pytest

import oracle as O

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "tests"))

# (d, E, K, P, T, kind, t)
CASES = [
    (256, 64, 8, 2, 40000, "2t", 0.10),  # 313 tiles: several tiles per CTA, both accumulator stages
    (512, 32, 8, 2, 300, "2t", 0.10),    # Epad 32, partial last tile
    (256, 40, 6, 1, 1, "1t", 0.20),      # E < Epad = 64, one token
    (256, 64, 16, 2, 777, "2t", 0.05),   # K = 16
    (256, 64, 8, 1, 2000, "1t", 0.08),   # P = 1
    (2048, 64, 8, 2, 4133, "2t", 0.085),  # C2 width
    (256, 24, 4, 2, 129, "none", 0.0),   # E < Epad = 32, no drop
]


def _layer(d, E, K, P, seed):
    from test_gpu_parity import rand_layer
    return rand_layer(d, 64, E, K, seed=seed, P=P)


def _tokens(T, d, seed):
    return O.bf16_round(np.random.default_rng(seed).standard_normal((T, d), dtype=np.float32))


def _run(case, i):
    """Route one case on the device; returns host arrays (logits, idx, raw, norm, frac) and stats."""
    import paper_2508_18376_b200 as pkg
    d, E, K, P, T, kind, t = case
    L = _layer(d, E, K, P, 100 + i)
    x = _tokens(T, d, 200 + i)
    ctx = pkg.Context()
    layer = pkg.MoeLayer(L.d, L.ffn, L.E, L.K, L.gate, L.blocks, L.shared, replay_factor=L.P, dtype="bf16",
                         gate_prenormalized=L.prenorm)
    pol = {"none": pkg.DropPolicy(), "1t": pkg.DropPolicy.one_t(t), "2t": pkg.DropPolicy.two_t_from(t)}[kind]
    r, lg = pkg.route_and_drop(ctx, layer, torch.from_numpy(x).cuda().bfloat16(), pol,
                               logits_mode=pkg.LOGITS_TENSOR, return_logits=True)
    idx, raw, norm, frac = r.host()
    return L, x, lg.cpu().numpy(), (idx, raw, norm, frac), r.stats


def _dump(path):
    """Subprocess body: every case through the current library setting -> npz."""
    torch.cuda.set_device(0)
    out = {}
    for i, case in enumerate(CASES):
        _, _, lg, rt, st = _run(case, i)
        out[f"lg{i}"] = lg
        for n, a in zip(("idx", "raw", "norm", "frac"), rt):
            out[f"{n}{i}"] = np.asarray(a)
        out[f"st{i}"] = np.array(json.dumps(st))
    np.savez(path, **out)


@pytest.mark.parametrize("i", range(len(CASES)))
def test_fused_routing_matches_oracle(i):
    torch.cuda.set_device(0)
    case = CASES[i]
    d, E, K, P, T, kind, t = case
    L, x, lg, (idx, raw, norm, frac), st = _run(case, i)
    # tensor-core logits vs the exact fp32 matmul of the bf16 operands
    lo = O.gate_logits(x, L.gate)
    den = max(np.abs(lg).max(), np.abs(lo).max())
    assert np.abs(lg - lo).max() / den < 1e-5
    ro = O.route_from_logits(lg, K, P, kind, t, normalize=not L.prenorm)
    sh = ro.idx.shape
    assert np.array_equal(idx.reshape(sh), ro.idx)
    assert np.array_equal(raw.reshape(sh), ro.raw)
    assert np.array_equal(norm.reshape(sh), ro.norm)
    assert np.array_equal(frac.reshape(sh), ro.frac)
    so = O.drop_stats(np.ones_like(ro.frac), ro.frac, P, 0, T, d, L.ffn)
    for k, v in so.items():
        assert st[k] == v, k


def test_fused_equals_two_kernel_chain(tmp_path):
    """Same logits bits, same routing, same stats as gate GEMM + router."""
    paths = {}
    for mode in ("1", "0"):
        p = tmp_path / f"gr{mode}.npz"
        env = dict(os.environ, DSMOE_B200_GATE_ROUTE=mode)
        code = (f"import sys; sys.path.insert(0, {ROOT!r}); sys.path.insert(0, {os.path.join(ROOT, 'tests')!r}); "
                f"import test_gpu_gate_route as m; m._dump({str(p)!r})")
        r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=600)
        assert r.returncode == 0, r.stderr[-3000:]
        paths[mode] = p
    a, b = np.load(paths["1"]), np.load(paths["0"])
    assert sorted(a.files) == sorted(b.files)
    for k in a.files:
        assert np.array_equal(a[k], b[k]), k
