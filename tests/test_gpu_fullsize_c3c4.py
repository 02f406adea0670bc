"""GPU parity at the other BASELINE shapes, where the
oracle can only check a token subsample:

* C4, DeepSeek-V2-Lite layer: 64 routed experts (ffn 1408, split P=2 into
  704-wide halves) + 2 shared experts, top-6, d=2048, T=16384 — routing, masks
  and drop_stats bit-exact on identical logits over every token; forward on a
  strided subsample within the bf16 scaled residual (shared experts weigh 1,
  moe.hpp:267-268);
* C3, Mixtral-8x7B after complete_transform(P=4): 32 experts of width 3584
  split P=2 into 1792-wide halves, top-8, d=4096 — forward subsample parity.
"""
import numpy as np
import pytest

import oracle as O

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

TOL_BF16 = 1e-2


def D():
    import paper_2508_18376_b200 as pkg
    return pkg


def scaled_residual(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    den = max(np.abs(a).max(), np.abs(b).max())
    return 0.0 if den == 0 else float(np.abs(a - b).max() / den)


def _layer(d, ffn, E, K, S, seed):
    rng = np.random.default_rng(seed)
    sd = 1.0 / np.sqrt(d)
    r = lambda *s: O.bf16_round(rng.standard_normal(s, dtype=np.float32) * sd)
    gate = r(d, E)
    blocks = [(r(d, ffn), r(d, ffn), r(ffn, d)) for _ in range(E)]
    shared = [(r(d, ffn), r(d, ffn), r(ffn, d)) for _ in range(S)]
    return O.partial_transform(O.Layer(d, ffn, E, K, gate, blocks, shared), 2)


@pytest.fixture(scope="module")
def ctx():
    torch.cuda.set_device(0)
    return D().Context()


def _dev(L):
    return D().MoeLayer(L.d, L.ffn, L.E, L.K, L.gate, L.blocks, L.shared, replay_factor=2, dtype="bf16")


def test_c4_fullsize_routing_stats_and_subsample(ctx):
    pkg = D()
    L = _layer(2048, 1408, 64, 6, 2, seed=41)
    layer = _dev(L)
    T = 16384
    x = O.bf16_round(np.random.default_rng(42).standard_normal((T, 2048), dtype=np.float32))
    xd = torch.from_numpy(x).cuda().bfloat16()
    t = 0.12
    pol = pkg.DropPolicy.two_t_from(t)
    r, lg = pkg.route_and_drop(ctx, layer, xd, pol, return_logits=True)
    ro = O.route_from_logits(lg.cpu().numpy(), 6, 2, "2t", t)
    idx, raw, norm, frac = r.host()
    sh = ro.idx.shape
    assert np.array_equal(idx.reshape(sh), ro.idx)
    assert np.array_equal(frac.reshape(sh), ro.frac)
    assert np.array_equal(norm.reshape(sh), ro.norm)
    st = O.drop_stats(np.ones_like(ro.frac), ro.frac, 2, 2, T, L.d, L.ffn)
    for k, v in st.items():
        assert r.stats[k] == v, k
    y = pkg.forward(ctx, layer, xd, pol).float().cpu().numpy()
    sel = np.arange(11, T, 1021)
    yo = O.moe_forward(L, x[sel], ro.idx[sel], ro.raw[sel], ro.frac[sel])
    assert scaled_residual(y[sel], yo) < TOL_BF16


def test_c3_shape_subsample(ctx):
    pkg = D()
    L = _layer(4096, 3584, 32, 8, 0, seed=43)
    layer = _dev(L)
    T = 4096
    x = O.bf16_round(np.random.default_rng(44).standard_normal((T, 4096), dtype=np.float32))
    xd = torch.from_numpy(x).cuda().bfloat16()
    for kind, t in (("none", 0.0), ("2t", 0.05)):
        pol = pkg.DropPolicy() if kind == "none" else pkg.DropPolicy.two_t_from(t)
        _, lg = pkg.route_and_drop(ctx, layer, xd, pol, return_logits=True)
        ro = O.route_from_logits(lg.cpu().numpy(), 8, 2, kind, t)
        y = pkg.forward(ctx, layer, xd, pol).float().cpu().numpy()
        sel = np.arange(5, T, 683)
        yo = O.moe_forward(L, x[sel], ro.idx[sel], ro.raw[sel], ro.frac[sel])
        assert scaled_residual(y[sel], yo) < TOL_BF16, kind
