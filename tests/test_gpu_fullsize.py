"""GPU parity at the benchmark size (C2: OLMoE layer shape, T = 16384 bf16
tokens, partial P=2 split so the 2T policy applies), where the oracle cannot
run the whole forward in seconds.  Checked through what does not depend on
size:

* routing, drop masks and drop_stats on identical fp32 logits: bit-exact over
  all 16384 tokens (route_from_logits / drop_stats, dropping.hpp:171-195);
* the forward on a strided token subsample against the oracle (the path is
  per-token separable, moe.hpp:253-269), within the bf16 scaled residual;
* determinism: two forwards are bit-identical (no atomics on the data path);
* token-permutation equivariance: forward(x[perm]) == forward(x)[perm] bit for
  bit (a row's arithmetic does not depend on where the permutation put it);
* a token count that is not a multiple of any tile (16389).
"""
import numpy as np
import pytest

import oracle as O

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

TOL_BF16 = 1e-2
T_FULL = 16384


def D():
    import paper_2508_18376_b200 as pkg
    return pkg


def scaled_residual(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    den = max(np.abs(a).max(), np.abs(b).max())
    return 0.0 if den == 0 else float(np.abs(a - b).max() / den)


@pytest.fixture(scope="module")
def ctx():
    torch.cuda.set_device(0)
    return D().Context()


@pytest.fixture(scope="module")
def c2full():
    rng = np.random.default_rng(2024)
    d, ffn, E, K = 2048, 1024, 64, 8
    sd = 1.0 / np.sqrt(d)
    gate = O.bf16_round(rng.standard_normal((d, E), dtype=np.float32) * sd)
    blocks = [tuple(O.bf16_round(rng.standard_normal(s, dtype=np.float32) * sd) for s in ((d, ffn), (d, ffn), (ffn, d)))
              for _ in range(E)]
    L = O.partial_transform(O.Layer(d, ffn, E, K, gate, blocks, []), 2)
    x = O.bf16_round(rng.standard_normal((T_FULL + 5, d), dtype=np.float32))
    layer = D().MoeLayer(L.d, L.ffn, L.E, L.K, L.gate, L.blocks, L.shared, replay_factor=2, dtype="bf16")
    return L, layer, x


@pytest.mark.parametrize("t", [0.0, 0.08, 0.11])
def test_fullsize_routing_and_stats_exact(ctx, c2full, t):
    L, layer, x = c2full
    pkg = D()
    xd = torch.from_numpy(x[:T_FULL]).cuda().bfloat16()
    pol = pkg.DropPolicy() if t == 0 else pkg.DropPolicy.two_t_from(t)
    r, lg = pkg.route_and_drop(ctx, layer, xd, pol, return_logits=True)
    ro = O.route_from_logits(lg.cpu().numpy(), 8, 2, "none" if t == 0 else "2t", t)
    idx, raw, norm, frac = r.host()
    sh = ro.idx.shape
    assert np.array_equal(idx.reshape(sh), ro.idx)
    assert np.array_equal(raw.reshape(sh), ro.raw)
    assert np.array_equal(norm.reshape(sh), ro.norm)
    assert np.array_equal(frac.reshape(sh), ro.frac)
    st = O.drop_stats(np.ones_like(ro.frac), ro.frac, 2, 0, T_FULL, L.d, L.ffn)
    for k, v in st.items():
        assert r.stats[k] == v, k


def _forward(pkg, ctx, layer, x, pol):
    return pkg.forward(ctx, layer, torch.from_numpy(x).cuda().bfloat16(), pol)


def test_fullsize_forward_subsample_and_determinism(ctx, c2full):
    L, layer, x = c2full
    pkg = D()
    pol = pkg.DropPolicy.two_t_from(0.085)
    xs = x[:T_FULL]
    y1 = _forward(pkg, ctx, layer, xs, pol)
    y2 = _forward(pkg, ctx, layer, xs, pol)
    assert torch.equal(y1, y2), "forward is not deterministic"
    _, lg = pkg.route_and_drop(ctx, layer, torch.from_numpy(xs).cuda().bfloat16(), pol, return_logits=True)
    ro = O.route_from_logits(lg.cpu().numpy(), 8, 2, "2t", 0.085)
    sel = np.arange(3, T_FULL, 257)
    yo = O.moe_forward(L, xs[sel], ro.idx[sel], ro.raw[sel], ro.frac[sel])
    assert scaled_residual(y1.float().cpu().numpy()[sel], yo) < TOL_BF16


def test_fullsize_token_permutation_equivariance(ctx, c2full):
    _, layer, x = c2full
    pkg = D()
    pol = pkg.DropPolicy.two_t_from(0.085)
    xs = x[:T_FULL]
    perm = np.random.default_rng(5).permutation(T_FULL)
    y = _forward(pkg, ctx, layer, xs, pol)
    yp = _forward(pkg, ctx, layer, np.ascontiguousarray(xs[perm]), pol)
    assert torch.equal(yp, y[torch.from_numpy(perm).cuda()])


def test_ragged_token_count(ctx, c2full):
    L, layer, x = c2full
    pkg = D()
    pol = pkg.DropPolicy.two_t_from(0.1)
    T = T_FULL + 5
    y = _forward(pkg, ctx, layer, x, pol)
    assert y.shape == (T, L.d)
    _, lg = pkg.route_and_drop(ctx, layer, torch.from_numpy(x).cuda().bfloat16(), pol, return_logits=True)
    ro = O.route_from_logits(lg.cpu().numpy(), 8, 2, "2t", 0.1)
    sel = np.array([0, 1, 127, 128, 8191, T - 6, T - 5, T - 2, T - 1])
    yo = O.moe_forward(L, x[sel], ro.idx[sel], ro.raw[sel], ro.frac[sel])
    assert scaled_residual(y.float().cpu().numpy()[sel], yo) < TOL_BF16
