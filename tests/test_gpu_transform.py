"""GPU: the partition API on the device (transform.hpp) and moe_forward on
any valid RoutingDecision (moe.hpp:239-271).

* complete_transform / partial_transform / reverse_partial of a device layer
  (dsmoe_b200_transform) read back (dsmoe_b200_layer_get_*) bit-equal to the
  oracle's restatement and to the reference itself (oracle/_ref, where built);
  fp32 and bf16 layers; the error codes of transform.hpp:70-76 / :104-110;
* the transformed layers' forwards equal the oracle's;
* moe_forward with non-canonical routings (copies with different raw scores,
  fraction 0.5 on a split layer, kept minor without major, duplicate
  blocks, P = 3) equals the oracle's moe_forward;
* a 96-expert layer (permutation shared memory > 48 KB with its
  static part) routes and forwards.
"""
import numpy as np
import pytest

import oracle as O

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


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


def dev_layer(L, dtype="f32"):
    return D().MoeLayer(L.d, L.ffn, L.E, L.K, L.gate, L.blocks, L.shared, replay_factor=L.P, dtype=dtype,
                        gate_prenormalized=L.prenorm)


def read_back(ctx, layer):
    g, blocks, shared = D().layer_weights(ctx, layer, device=False)
    f = lambda t: t.float().numpy()
    return f(g), [tuple(f(w) for w in b) for b in blocks], [tuple(f(w) for w in s) for s in shared]


def assert_weights_equal(got, L):
    g, blocks, shared = got
    assert np.array_equal(g, L.gate)
    assert len(blocks) == len(L.blocks) and len(shared) == len(L.shared)
    for a, b in zip(blocks + shared, L.blocks + L.shared):
        for x, y in zip(a, b):
            assert x.shape == y.shape and np.array_equal(x, y)


@pytest.fixture(scope="module")
def base():
    return O.generate_layer(128, 192, 6, 2, S=1, seed=77)


def test_readback_roundtrip(ctx, base):
    assert_weights_equal(read_back(ctx, dev_layer(base)), base)
    Lb = base.round_bf16()
    assert_weights_equal(read_back(ctx, dev_layer(base, "bf16")), Lb)


@pytest.mark.parametrize("p", [2, 4])
@pytest.mark.parametrize("dtype", ["f32", "bf16"])
def test_complete_transform_bit_exact(ctx, base, p, dtype):
    pkg = D()
    src = base if dtype == "f32" else base.round_bf16()
    t = pkg.complete_transform(ctx, dev_layer(src, dtype), p)
    assert (t.E, t.K, t.ffn, t.P) == (6 * p, 2 * p, 192 // p, 1)
    want = O.complete_transform(src, p)  # W2 x p: exact in bf16 for p a power of two
    assert_weights_equal(read_back(ctx, t), want)
    if dtype == "f32" and O.ref_available():
        got = O.RefLayer.from_layer(base).transform(True, p).to_layer()
        assert_weights_equal(read_back(ctx, t), got)


@pytest.mark.parametrize("p", [2, 3])
def test_partial_and_reverse_bit_exact(ctx, base, p):
    pkg = D()
    L = dev_layer(base)
    t = pkg.partial_transform(ctx, L, p)
    assert (t.E, t.K, t.ffn, t.P) == (6, 2, 192, p)
    want = O.partial_transform(base, p)
    assert_weights_equal(read_back(ctx, t), want)
    if O.ref_available():
        assert_weights_equal(read_back(ctx, t), O.RefLayer.from_layer(base).transform(False, p).to_layer())
    back = pkg.transform(ctx, t, "reverse")
    assert back.P == 1
    assert_weights_equal(read_back(ctx, back), base)  # bit-exact round trip (transform.hpp:133-135)


def test_transform_errors(ctx, base):
    pkg = D()
    L = dev_layer(base)
    with pytest.raises(pkg.DsmoeError) as e:
        pkg.complete_transform(ctx, L, 1)
    assert e.value.code == 1
    with pytest.raises(pkg.DsmoeError) as e:
        pkg.complete_transform(ctx, L, 5)  # 192 % 5
    assert e.value.code == 1
    t = pkg.partial_transform(ctx, L, 2)
    with pytest.raises(pkg.DsmoeError) as e:
        pkg.complete_transform(ctx, t, 2)
    assert e.value.code == 3
    with pytest.raises(pkg.DsmoeError) as e:
        pkg.transform(ctx, L, "reverse")
    assert e.value.code == 3


def test_transformed_forwards(ctx, base):
    """The device-transformed layers run the forward like any other layer."""
    pkg = D()
    x = O.generate_tokens(200, 128, seed=5)
    xd = torch.from_numpy(x).cuda()
    L = dev_layer(base)
    for layer, ol in ((pkg.complete_transform(ctx, L, 4), O.complete_transform(base, 4)),
                      (pkg.partial_transform(ctx, L, 2), O.partial_transform(base, 2))):
        kind = "2t" if ol.P == 2 else "1t"
        pol = pkg.DropPolicy.two_t_from(0.3) if kind == "2t" else pkg.DropPolicy.one_t(0.1)
        r = pkg.route_and_drop(ctx, layer, xd, pol, logits_mode=pkg.LOGITS_EXACT)
        ro = O.route(ol, x, kind, pol.t_drop)
        idx, raw, norm, frac = r.host()
        assert np.array_equal(idx.reshape(ro.idx.shape), ro.idx)
        assert np.array_equal(frac.reshape(ro.frac.shape), ro.frac)
        y = pkg.forward(ctx, layer, xd, pol, logits_mode=pkg.LOGITS_EXACT).cpu().numpy()
        assert scaled_residual(y, O.moe_forward(ol, x, ro.idx, ro.raw, ro.frac)) < 1e-5


def _noncanonical(rng, T, E, K, P):
    """Routing that replay_routing + apply_bands never produce but moe_forward
    accepts: per slot any physical block, any fraction in {0, .5, 1}, any raw."""
    n = K * P
    idx = rng.integers(0, E * P, size=(T, n)).astype(np.int32)
    frac = rng.choice([0.0, 0.5, 1.0], size=(T, n))
    raw = rng.uniform(0.01, 0.6, size=(T, n))
    return idx, raw, frac


@pytest.mark.parametrize("P,dtype", [(2, "f32"), (3, "f32"), (2, "bf16")])
def test_moe_forward_noncanonical_routing(ctx, base, P, dtype):
    pkg = D()
    src = base if dtype == "f32" else base.round_bf16()
    ol = O.partial_transform(src, P)
    layer = dev_layer(ol, dtype)
    rng = np.random.default_rng(10 + P)
    T = 150
    x = O.generate_tokens(T, 128, seed=6)
    if dtype == "bf16":
        x = O.bf16_round(x)
    idx, raw, frac = _noncanonical(rng, T, ol.E, ol.K, P)
    idx[0, 1] = idx[0, 0]  # a duplicate block within one token
    xd = torch.from_numpy(x).cuda()
    if dtype == "bf16":
        xd = xd.bfloat16()
    y = pkg.moe_forward(ctx, layer, xd, (torch.from_numpy(idx), torch.from_numpy(raw), torch.from_numpy(frac)))
    yo = O.moe_forward(ol, x, idx, raw, frac)
    tol = 1e-5 if dtype == "f32" else 1e-2
    assert scaled_residual(y.float().cpu().numpy(), yo) < tol
    # the canonical routing still takes the fused path and agrees too
    ro = O.route(ol, x, "1t", 0.2)
    y2 = pkg.moe_forward(ctx, layer, xd, (torch.from_numpy(ro.idx), torch.from_numpy(ro.raw),
                                          torch.from_numpy(ro.frac)))
    assert scaled_residual(y2.float().cpu().numpy(), O.moe_forward(ol, x, ro.idx, ro.raw, ro.frac)) < tol


def test_moe_forward_invalid_routing(ctx, base):
    pkg = D()
    ol = O.partial_transform(base, 2)
    layer = dev_layer(ol)
    x = torch.from_numpy(O.generate_tokens(8, 128, seed=7)).cuda()
    idx = np.zeros((8, 4), np.int32)
    idx[3, 2] = 12  # E*P = 12: out of range (moe.hpp:258-260)
    raw = np.full((8, 4), 0.25)
    frac = np.ones((8, 4))
    with pytest.raises(pkg.DsmoeError) as e:
        pkg.moe_forward(ctx, layer, x, (torch.from_numpy(idx), torch.from_numpy(raw), torch.from_numpy(frac)))
    assert e.value.code == 3
    idx[3, 2] = 0
    frac[1, 1] = 0.25  # routing.validate: fractions in {0, 0.5, 1} (moe.hpp:163-165)
    with pytest.raises(pkg.DsmoeError) as e:
        pkg.moe_forward(ctx, layer, x, (torch.from_numpy(idx), torch.from_numpy(raw), torch.from_numpy(frac)))
    assert e.value.code == 3
    ctx.check()  # the context is usable again after reporting


def test_96_experts(ctx):
    """E = 96 puts the permutation kernel's dynamic + static shared
    memory over the 48 KB default; the launch must opt in."""
    pkg = D()
    L = O.generate_layer(64, 64, 96, 4, seed=96)
    layer = dev_layer(L)
    x = O.generate_tokens(300, 64, seed=8)
    xd = torch.from_numpy(x).cuda()
    pol = pkg.DropPolicy.one_t(0.1)
    y = pkg.forward(ctx, layer, xd, pol, logits_mode=pkg.LOGITS_EXACT).cpu().numpy()
    ro = O.route(L, x, "1t", 0.1)
    assert scaled_residual(y, O.moe_forward(L, x, ro.idx, ro.raw, ro.frac)) < 1e-5


def test_sticky_error_flag(ctx):
    """a forward launched without stats on scores whose Top-K sum
    is not positive (NaN tokens) reports normalize_topk's error
    (dropping.hpp:67) at the next synchronising call, once."""
    pkg = D()
    L = O.generate_layer(64, 64, 4, 2, seed=9)
    layer = dev_layer(L)
    x = torch.from_numpy(O.generate_tokens(40, 64, seed=10)).cuda()
    x[7] = float("nan")
    pkg.forward(ctx, layer, x, pkg.DropPolicy(), logits_mode=pkg.LOGITS_EXACT)  # no stats: no sync
    with pytest.raises(pkg.DsmoeError) as e:
        ctx.check()
    assert e.value.code == 1
    ctx.check()  # reported once, then clear
    x[7] = 0.0
    _, st = pkg.forward(ctx, layer, x, pkg.DropPolicy(), logits_mode=pkg.LOGITS_EXACT, with_stats=True)
    assert st["drop_rate"] == 0.0
