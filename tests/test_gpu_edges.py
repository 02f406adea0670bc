"""Edge cases of the device path against the oracle: the largest expert count
and top-K the device supports (E = 256, K = 16, warp-per-token router), a
drop threshold that removes every selection but the keep-top-1 guard
(dropping.hpp:117-119), the guard off (rows can vanish entirely), one token,
and token counts around the 32-token router chunk / 128-row tile sizes."""
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


@pytest.fixture(scope="module")
def ctx():
    torch.cuda.set_device(0)
    return D().Context()


def _layer(d, ffn, E, K, seed, P=2):
    rng = np.random.default_rng(seed)
    sd = 1.0 / np.sqrt(d)
    r = lambda *s: O.bf16_round(rng.standard_normal(s, dtype=np.float32) * sd)
    L = O.Layer(d, ffn, E, K, r(d, E), [(r(d, ffn), r(d, ffn), r(ffn, d)) for _ in range(E)], [])
    return O.partial_transform(L, P) if P > 1 else L


def _dev(L):
    return D().MoeLayer(L.d, L.ffn, L.E, L.K, L.gate, L.blocks, L.shared, replay_factor=L.P, dtype="bf16")


def _check(ctx, L, x, kind, t, keep_top1=True, sel=None):
    pkg = D()
    layer = _dev(L)
    xd = torch.from_numpy(x).cuda().bfloat16()
    if kind == "none":
        pol = pkg.DropPolicy()
    elif kind == "1t":
        pol = pkg.DropPolicy.one_t(t, keep_top1)
    else:
        pol = pkg.DropPolicy.two_t_from(t, keep_top1)
    r, lg = pkg.route_and_drop(ctx, layer, xd, pol, return_logits=True)
    ro = O.route_from_logits(lg.cpu().numpy(), L.K, L.P, kind, t, keep_top1=keep_top1)
    idx, raw, norm, frac = r.host()
    sh = ro.idx.shape
    assert np.array_equal(idx.reshape(sh), ro.idx)
    assert np.array_equal(frac.reshape(sh), ro.frac)
    assert np.array_equal(norm.reshape(sh), ro.norm)
    y = pkg.forward(ctx, layer, xd, pol).float().cpu().numpy()
    sel = np.arange(x.shape[0]) if sel is None else sel
    yo = O.moe_forward(L, x[sel], ro.idx[sel], ro.raw[sel], ro.frac[sel])
    if np.abs(yo).max() == 0:
        assert np.abs(y[sel]).max() == 0
    else:
        assert scaled_residual(y[sel], yo) < TOL_BF16
    return ro


def test_max_experts_and_topk(ctx):
    L = _layer(256, 128, 256, 16, seed=51)
    x = O.bf16_round(np.random.default_rng(52).standard_normal((300, 256), dtype=np.float32))
    _check(ctx, L, x, "2t", 0.06)


def test_drop_everything_but_top1(ctx):
    L = _layer(512, 256, 16, 4, seed=53)
    x = O.bf16_round(np.random.default_rng(54).standard_normal((257, 512), dtype=np.float32))
    ro = _check(ctx, L, x, "2t", 0.995)
    # exactly one full selection per token survives (the guard restores all its copies)
    assert np.all((ro.frac[:, :L.K] > 0).sum(axis=1) == 1)


def test_keep_top1_off_rows_vanish(ctx):
    L = _layer(512, 256, 16, 4, seed=55)
    x = O.bf16_round(np.random.default_rng(56).standard_normal((200, 512), dtype=np.float32))
    ro = _check(ctx, L, x, "1t", 0.999, keep_top1=False)
    assert np.all(ro.frac == 0)  # nothing kept: the output must be exactly zero


@pytest.mark.parametrize("T", [1, 31, 32, 33, 127, 129, 4097])
def test_token_counts(ctx, T):
    L = _layer(256, 256, 8, 2, seed=57)
    x = O.bf16_round(np.random.default_rng(58 + T).standard_normal((T, 256), dtype=np.float32))
    _check(ctx, L, x, "2t", 0.3, sel=np.unique(np.linspace(0, T - 1, min(T, 40)).astype(int)))
