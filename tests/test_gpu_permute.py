"""GPU: the token permutation (K2) is bit-equal to the CPU counting sort
(oracle.permutation), for the router's own routing and for imported ones;
drop-rate sweeps; boundary thresholds; error paths."""
import numpy as np
import pytest

import oracle as O

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


def D():
    import paper_2508_18376_b200 as pkg
    return pkg


@pytest.fixture(scope="module")
def ctx():
    return D().Context()


def small_layer(E=16, K=4, d=128, ffn=192, P=2, seed=0, S=0):
    L = O.generate_layer(d, ffn, E, K, S=S, seed=seed)
    return O.partial_transform(L, P) if P > 1 else L


@pytest.mark.parametrize("T", [1, 127, 128, 300, 2000])
@pytest.mark.parametrize("t", [0.0, 0.15, 0.24])
def test_permutation_matches_counting_sort(ctx, T, t):
    L = small_layer()
    x = O.generate_tokens(T, 128, seed=T)
    pkg = D()
    layer = pkg.MoeLayer(L.d, L.ffn, L.E, L.K, L.gate, L.blocks, replay_factor=2, dtype="f32")
    pol = pkg.DropPolicy.two_t_from(t) if t > 0 else pkg.DropPolicy()
    pkg.forward(ctx, layer, torch.from_numpy(x).cuda(), pol, logits_mode=pkg.LOGITS_EXACT)
    rt, sp, sg = ctx.permutation(T, L.K, L.E)
    ro = O.route(L, x, "2t" if t > 0 else "none", t)
    wrt, wsp, wsg = O.permutation(ro.idx, ro.frac, L.K, 2, L.E)
    assert np.array_equal(sg, wsg)
    assert np.array_equal(rt, wrt)
    assert np.array_equal(sp, wsp)


def test_permutation_imported_half_fractions(ctx):
    L = small_layer(P=1)
    T = 500
    x = O.generate_tokens(T, 128, seed=1)
    ro = O.route(L, x)
    rng = np.random.default_rng(0)
    frac = rng.choice([0.0, 0.5, 1.0], size=ro.frac.shape)
    pkg = D()
    layer = pkg.MoeLayer(L.d, L.ffn, L.E, L.K, L.gate, L.blocks, dtype="f32")
    y = pkg.moe_forward(ctx, layer, torch.from_numpy(x).cuda(),
                        (torch.from_numpy(ro.idx).cuda(), torch.from_numpy(ro.raw).cuda(),
                         torch.from_numpy(frac).cuda()))
    rt, sp, sg = ctx.permutation(T, L.K, L.E)
    wrt, wsp, wsg = O.permutation(ro.idx, frac, L.K, 1, L.E)
    assert np.array_equal(rt, wrt) and np.array_equal(sp, wsp) and np.array_equal(sg, wsg)
    yo = O.moe_forward(L, x, ro.idx, ro.raw, frac)
    den = max(np.abs(yo).max(), 1e-30)
    assert np.abs(y.cpu().numpy() - yo).max() / den < 1e-5


def test_noncanonical_routing_accepted(ctx):
    """A kept copy 1 whose copy 0 is dropped is outside the canonical replayed
    layout, but moe_forward (moe.hpp:253-266) evaluates it slot by slot: the
    device takes the block-view path and matches the oracle."""
    L = small_layer(P=2)
    T = 8
    x = O.generate_tokens(T, 128, seed=2)
    ro = O.route(L, x)
    frac = ro.frac.copy()
    frac[0, 0] = 0.0  # copy 0 dropped but copy 1 kept
    pkg = D()
    layer = pkg.MoeLayer(L.d, L.ffn, L.E, L.K, L.gate, L.blocks, replay_factor=2, dtype="f32")
    y = pkg.moe_forward(ctx, layer, torch.from_numpy(x).cuda(),
                        (torch.from_numpy(ro.idx).cuda(), torch.from_numpy(ro.raw).cuda(),
                         torch.from_numpy(frac).cuda()))
    yo = O.moe_forward(L, x, ro.idx, ro.raw, frac)
    assert np.abs(y.cpu().numpy() - yo).max() / max(np.abs(yo).max(), 1e-30) < 1e-5


def test_threshold_boundaries_inclusive(ctx):
    """Thresholds equal to an observed normalized score keep that selection
    (lower band edges are inclusive, dropping.hpp:97-100)."""
    L = small_layer()
    x = O.generate_tokens(256, 128, seed=3)
    pkg = D()
    layer = pkg.MoeLayer(L.d, L.ffn, L.E, L.K, L.gate, L.blocks, replay_factor=2, dtype="f32")
    xd = torch.from_numpy(x).cuda()
    r0 = O.route(L, x)
    for tv in (r0.norm[5, 2], r0.norm[17, 1], r0.norm[100, 3]):
        hi = max(tv, r0.norm[5, 1])
        for kind, mk, kw in (("1t", lambda: pkg.DropPolicy.one_t(tv, keep_top1=False), {}),
                             ("2t", lambda: pkg.DropPolicy.two_t(tv, tv, hi, keep_top1=False),
                              {"t_major": tv, "t_minor": hi})):
            r = pkg.route_and_drop(ctx, layer, xd, mk(), logits_mode=pkg.LOGITS_EXACT)
            ro = O.route(L, x, kind, tv, keep_top1=False, **kw)
            assert np.array_equal(r.host()[3].reshape(ro.frac.shape), ro.frac)


def test_prenormalized_gate_and_keep_top1_off(ctx):
    L = small_layer()
    x = O.generate_tokens(300, 128, seed=4)
    pkg = D()
    layer = pkg.MoeLayer(L.d, L.ffn, L.E, L.K, L.gate, L.blocks, replay_factor=2, dtype="f32",
                         gate_prenormalized=True)
    r = pkg.route_and_drop(ctx, layer, torch.from_numpy(x).cuda(), pkg.DropPolicy.one_t(0.08, keep_top1=False),
                           logits_mode=pkg.LOGITS_EXACT)
    ro = O.route_from_logits(O.gate_logits(x, L.gate), L.K, 2, "1t", 0.08, keep_top1=False, normalize=False)
    idx, raw, norm, frac = r.host()
    assert np.array_equal(norm.reshape(ro.norm.shape), ro.norm)
    assert np.array_equal(frac.reshape(ro.frac.shape), ro.frac)


def test_2t_requires_p2(ctx):
    L = small_layer(P=1)
    pkg = D()
    layer = pkg.MoeLayer(L.d, L.ffn, L.E, L.K, L.gate, L.blocks, dtype="f32")
    with pytest.raises(pkg.DsmoeError) as e:
        pkg.route_and_drop(ctx, layer, torch.zeros((4, 128), device="cuda"), pkg.DropPolicy.two_t_from(0.1))
    assert e.value.code == 3


def test_partial_p4_one_threshold(ctx):
    """partial_transform P=4 (transform.hpp:100) + 1T: all four sub-blocks per kept selection."""
    L = small_layer(P=4, ffn=256)
    x = O.generate_tokens(333, 128, seed=5)
    pkg = D()
    layer = pkg.MoeLayer(L.d, L.ffn, L.E, L.K, L.gate, L.blocks, replay_factor=4, dtype="f32")
    y = pkg.forward(ctx, layer, torch.from_numpy(x).cuda(), pkg.DropPolicy.one_t(0.2), logits_mode=pkg.LOGITS_EXACT)
    ro = O.route(L, x, "1t", 0.2)
    yo = O.moe_forward(L, x, ro.idx, ro.raw, ro.frac)
    assert np.abs(y.cpu().numpy() - yo).max() / np.abs(yo).max() < 1e-5


def test_complete_transform_routes_top_kp(ctx):
    """complete_transform P=4 (transform.hpp:66): E*P experts, top-K*P, W2 x P."""
    L = O.complete_transform(O.generate_layer(128, 256, 8, 2, seed=6), 4)
    x = O.generate_tokens(200, 128, seed=7)
    pkg = D()
    layer = pkg.MoeLayer(L.d, L.ffn, L.E, L.K, L.gate, L.blocks, dtype="f32")
    r = pkg.route_and_drop(ctx, layer, torch.from_numpy(x).cuda(), logits_mode=pkg.LOGITS_EXACT)
    ro = O.route(L, x)
    assert np.array_equal(r.host()[0].reshape(ro.idx.shape), ro.idx)
    y = pkg.forward(ctx, layer, torch.from_numpy(x).cuda(), logits_mode=pkg.LOGITS_EXACT)
    yo = O.moe_forward(L, x, ro.idx, ro.raw, ro.frac)
    assert np.abs(y.cpu().numpy() - yo).max() / np.abs(yo).max() < 1e-5
