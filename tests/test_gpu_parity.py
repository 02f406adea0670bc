"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle.

Bars (BASELINE.json north_star): routing indices, drop masks, raw and
normalized scores bit-exact on identical fp32 logits; MoE outputs within the
scaled residual max|a-b| / max(max|a|, max|b|) (transform.hpp:190-198) of
1e-5 for fp32 layers and 1e-2 for bf16 layers.
"""
import numpy as np
import pytest

import oracle as O

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

TOL_F32 = 1e-5
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


@pytest.fixture(scope="module")
def c1():
    """BASELINE config C1: E=8, K=2, d=512, ffn=1024, fp32, reconstructed P=2."""
    base = O.generate_layer(512, 1024, 8, 2, seed=1234)
    x = O.generate_tokens(256, 512, seed=99)
    r0 = O.route(base, x)
    rec = O.reconstruct(base, O.profile_importance(base, x, r0.idx, "abs_gate"))
    return base, rec, x


def rand_layer(d, ffn, E, K, S=0, seed=0, bf16=True, P=1, scale=1.0):
    """numpy N(0, scale^2/d) weights (fast generator for the big shapes), bf16-rounded."""
    rng = np.random.default_rng(seed)
    sd = scale / np.sqrt(d)
    r = O.bf16_round if bf16 else (lambda a: a)
    gate = r((rng.standard_normal((d, E), dtype=np.float32) * sd))
    blocks = []
    for _ in range(E):
        blocks.append(tuple(r(rng.standard_normal(s, dtype=np.float32) * sd) for s in ((d, ffn), (d, ffn), (ffn, d))))
    shared = []
    for _ in range(S):
        shared.append(tuple(r(rng.standard_normal(s, dtype=np.float32) * sd) for s in ((d, ffn), (d, ffn), (ffn, d))))
    L = O.Layer(d, ffn, E, K, gate, blocks, shared)
    return L if P == 1 else O.partial_transform(L, P)


def dev_layer(L, dtype):
    return D().MoeLayer(L.d, L.ffn, L.E, L.K, L.gate, L.blocks, L.shared, replay_factor=L.P, dtype=dtype,
                        gate_prenormalized=L.prenorm)


def check_routing(r, ro):
    idx, raw, norm, frac = r.host()
    sh = ro.idx.shape
    assert np.array_equal(idx.reshape(sh), ro.idx)
    assert np.array_equal(raw.reshape(sh), ro.raw)
    assert np.array_equal(norm.reshape(sh), ro.norm)
    assert np.array_equal(frac.reshape(sh), ro.frac)


# ------------------------------------------------------------------ C1 fp32
@pytest.mark.parametrize("kind,t", [("none", 0.0), ("1t", 0.40), ("2t", 0.40), ("2t", 0.30)])
def test_c1_routing_exact_from_tokens(ctx, c1, kind, t):
    _, rec, x = c1
    pkg = D()
    layer = dev_layer(rec, "f32")
    pol = {"none": pkg.DropPolicy(), "1t": pkg.DropPolicy.one_t(t), "2t": pkg.DropPolicy.two_t_from(t)}[kind]
    r, lg = pkg.route_and_drop(ctx, layer, torch.from_numpy(x).cuda(), pol, logits_mode=pkg.LOGITS_EXACT,
                               return_logits=True)
    # exact-order logits are the reference matmul bit for bit
    assert np.array_equal(lg.cpu().numpy(), O.gate_logits(x, rec.gate))
    ro = O.route(rec, x, kind, t)
    check_routing(r, ro)
    st = O.drop_stats(ro.pre_frac, ro.frac, 2, 0, 256, 512, 1024)
    for k, v in st.items():
        assert r.stats[k] == v, k


def test_c1_pinned_drop_rate_and_forward(ctx, c1):
    _, rec, x = c1
    pkg = D()
    layer = dev_layer(rec, "f32")
    xd = torch.from_numpy(x).cuda()
    pol = pkg.DropPolicy.two_t_from(0.40)
    y, st = pkg.forward(ctx, layer, xd, pol, logits_mode=pkg.LOGITS_EXACT, with_stats=True)
    ro = O.route(rec, x, "2t", 0.40)
    yo = O.moe_forward(rec, x, ro.idx, ro.raw, ro.frac)
    assert scaled_residual(y.cpu().numpy(), yo) < TOL_F32
    assert st["drop_rate"] == O.drop_stats(ro.pre_frac, ro.frac, 2, 0, 256, 512, 1024)["drop_rate"]


def test_c1_base_layer_forward_fp32(ctx, c1):
    base, _, x = c1
    pkg = D()
    layer = dev_layer(base, "f32")
    xd = torch.from_numpy(x).cuda()
    y = pkg.forward(ctx, layer, xd, pkg.DropPolicy.one_t(0.3), logits_mode=pkg.LOGITS_EXACT)
    ro = O.route(base, x, "1t", 0.3)
    yo = O.moe_forward(base, x, ro.idx, ro.raw, ro.frac)
    assert scaled_residual(y.cpu().numpy(), yo) < TOL_F32


def test_fraction_half_on_unsplit_block(ctx, c1):
    """moe.hpp:264 — fraction 0.5 evaluates the first ceil(w/2) neurons
    (test_moe_model.cpp:132-159), through an explicit routing."""
    base, _, x = c1
    pkg = D()
    layer = dev_layer(base, "f32")
    xs = x[:64]
    ro = O.route(base, xs)
    frac = np.where((np.arange(ro.frac.size).reshape(ro.frac.shape) % 3) == 0, 0.5, 1.0)
    frac[5, :] = 0.0
    yo = O.moe_forward(base, xs, ro.idx, ro.raw, frac)
    y = pkg.moe_forward(ctx, layer, torch.from_numpy(xs).cuda(),
                        (torch.from_numpy(ro.idx).cuda(), torch.from_numpy(ro.raw).cuda(),
                         torch.from_numpy(frac).cuda()))
    assert scaled_residual(y.cpu().numpy(), yo) < TOL_F32
    assert np.all(y.cpu().numpy()[5] == 0)


# --------------------------------------------------------- bf16, C2 shape
@pytest.fixture(scope="module")
def c2():
    L = rand_layer(2048, 1024, 64, 8, seed=7)
    x = O.bf16_round(np.random.default_rng(99).standard_normal((1000, 2048), dtype=np.float32))
    r0 = O.route(L, x[:256])
    rec = O.reconstruct(L, O.profile_importance(L, x[:256], r0.idx, "abs_gate"))
    return L, rec, x


@pytest.mark.parametrize("kind,t", [("none", 0.0), ("2t", 0.08), ("2t", 0.13)])
def test_c2_routing_exact_on_identical_logits(ctx, c2, kind, t):
    _, rec, x = c2
    pkg = D()
    layer = dev_layer(rec, "bf16")
    xd = torch.from_numpy(x).cuda().bfloat16()
    pol = {"none": pkg.DropPolicy(), "2t": pkg.DropPolicy.two_t_from(t)}[kind]
    r, lg = pkg.route_and_drop(ctx, layer, xd, pol, logits_mode=pkg.LOGITS_TENSOR, return_logits=True)
    lgh = lg.cpu().numpy()
    # tensor-core logits vs the exact fp32 matmul: close, not bit-equal
    lo = O.gate_logits(x, rec.gate)
    assert scaled_residual(lgh, lo) < 1e-5
    ro = O.route_from_logits(lgh, 8, 2, kind, t)
    check_routing(r, ro)


def test_c2_exact_logits_mode_bitexact(ctx, c2):
    _, rec, x = c2
    pkg = D()
    layer = dev_layer(rec, "bf16")
    xd = torch.from_numpy(x).cuda().bfloat16()
    r, lg = pkg.route_and_drop(ctx, layer, xd, pkg.DropPolicy.two_t_from(0.1), logits_mode=pkg.LOGITS_EXACT,
                               return_logits=True)
    assert np.array_equal(lg.cpu().numpy(), O.gate_logits(x, rec.gate))
    check_routing(r, O.route(rec, x, "2t", 0.1))


@pytest.mark.parametrize("kind,t", [("none", 0.0), ("2t", 0.10)])
def test_c2_forward_bf16(ctx, c2, kind, t):
    _, rec, x = c2
    pkg = D()
    layer = dev_layer(rec, "bf16")
    xd = torch.from_numpy(x).cuda().bfloat16()
    pol = {"none": pkg.DropPolicy(), "2t": pkg.DropPolicy.two_t_from(t)}[kind]
    y = pkg.forward(ctx, layer, xd, pol, logits_mode=pkg.LOGITS_EXACT).float().cpu().numpy()
    ro = O.route(rec, x, kind, t)
    sel = np.arange(0, x.shape[0], 37)  # per-token separable: strided subsample
    yo = O.moe_forward(rec, x[sel], ro.idx[sel], ro.raw[sel], ro.frac[sel])
    assert scaled_residual(y[sel], yo) < TOL_BF16


def test_shared_experts_bf16(ctx):
    """C4-like: routed + shared experts (moe.hpp:267-268), T not a multiple of 128."""
    L = rand_layer(256, 192, 16, 3, S=2, seed=3)
    x = O.bf16_round(np.random.default_rng(5).standard_normal((300, 256), dtype=np.float32))
    pkg = D()
    layer = dev_layer(L, "bf16")
    y = pkg.forward(ctx, layer, torch.from_numpy(x).cuda().bfloat16(), pkg.DropPolicy.one_t(0.3),
                    logits_mode=pkg.LOGITS_EXACT).float().cpu().numpy()
    ro = O.route(L, x, "1t", 0.3)
    yo = O.moe_forward(L, x, ro.idx, ro.raw, ro.frac)
    assert scaled_residual(y, yo) < TOL_BF16


def test_empty_and_tiny_batches(ctx, c1):
    _, rec, x = c1
    pkg = D()
    layer = dev_layer(rec, "f32")
    for T in (1, 3, 129):
        xs = x[:T]
        y = pkg.forward(ctx, layer, torch.from_numpy(xs).cuda(), pkg.DropPolicy.two_t_from(0.4),
                        logits_mode=pkg.LOGITS_EXACT)
        ro = O.route(rec, xs, "2t", 0.4)
        yo = O.moe_forward(rec, xs, ro.idx, ro.raw, ro.frac)
        assert scaled_residual(y.cpu().numpy(), yo) < TOL_F32
    y0 = pkg.forward(ctx, layer, torch.empty((0, 512), device="cuda"), pkg.DropPolicy())
    assert y0.shape == (0, 512)


def test_model_forward_dropped_two_layers(ctx):
    """model_forward_dropped (dropping.hpp:263-274): x_{l+1} = x_l + moe_l(x_l),
    the residual fused into the combine, per-layer routing and DropStats."""
    pkg = D()
    Ls = [O.partial_transform(O.generate_layer(128, 128, 8, 2, seed=s), 2) for s in (81, 82)]
    layers = [dev_layer(L, "f32") for L in Ls]
    x = O.generate_tokens(96, 128, seed=83)
    y, stats = pkg.model_forward_dropped(ctx, layers, torch.from_numpy(x).cuda(), pkg.DropPolicy.two_t_from(0.3),
                                         logits_mode=pkg.LOGITS_EXACT)
    cur = x.astype(np.float32)
    for L, st in zip(Ls, stats):
        ro = O.route(L, cur, "2t", 0.3)
        cur = (cur + O.moe_forward(L, cur, ro.idx, ro.raw, ro.frac)).astype(np.float32)
        so = O.drop_stats(np.ones_like(ro.frac), ro.frac, 2, 0, cur.shape[0], L.d, L.ffn)
        assert st["drop_rate"] == so["drop_rate"]
    assert scaled_residual(y.cpu().numpy(), cur) < TOL_F32


def test_model_forward_dropped_per_layer_policies(ctx):
    """A policy per layer: layer l routes under its own
    threshold; per-layer calibration reaches the target on every layer."""
    pkg = D()
    from paper_2508_18376_b200 import analysis as A
    Ls = [O.partial_transform(O.generate_layer(128, 128, 8, 2, seed=s), 2) for s in (84, 85, 86)]
    layers = [dev_layer(L, "f32") for L in Ls]
    x = O.generate_tokens(200, 128, seed=87)
    pols = [pkg.DropPolicy.two_t_from(0.25), pkg.DropPolicy.one_t(0.1), pkg.DropPolicy()]
    y, stats = pkg.model_forward_dropped(ctx, layers, torch.from_numpy(x).cuda(), pols, logits_mode=pkg.LOGITS_EXACT)
    cur = x.astype(np.float32)
    for L, st, (kind, t) in zip(Ls, stats, (("2t", 0.25), ("1t", 0.1), ("none", 0.0))):
        ro = O.route(L, cur, kind, t)
        cur = (cur + O.moe_forward(L, cur, ro.idx, ro.raw, ro.frac)).astype(np.float32)
        so = O.drop_stats(np.ones_like(ro.frac), ro.frac, 2, 0, cur.shape[0], L.d, L.ffn)
        assert st["drop_rate"] == so["drop_rate"]
    assert scaled_residual(y.cpu().numpy(), cur) < TOL_F32
    with pytest.raises(pkg.DsmoeError):
        pkg.model_forward_dropped(ctx, layers, torch.from_numpy(x).cuda(), pols[:2])
    cal, rates = A.calibrate_per_layer(ctx, layers, torch.from_numpy(x).cuda(), 0.25)
    assert all(abs(r - 0.25) < 0.03 for r in rates)
    _, st2 = pkg.model_forward_dropped(ctx, layers, torch.from_numpy(x).cuda(), cal, logits_mode=pkg.LOGITS_EXACT)
    assert [s["drop_rate"] for s in st2] == rates
