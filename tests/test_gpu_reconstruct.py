"""GPU parity for the offline partition (north-star item 1): device
profile_importance is bit-equal to the reference's (reconstruct.hpp:99-149),
the device importance order is the reference's stable sort (:151-168), and the
device-reconstructed layer computes the reference's reconstructed forward."""
import numpy as np
import pytest

import oracle as O

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


def D():
    import paper_2508_18376_b200 as pkg
    return pkg


def scaled_residual(a, b):
    den = max(np.abs(a).max(), np.abs(b).max())
    return float(np.abs(np.asarray(a, np.float64) - b).max() / den)


@pytest.fixture(scope="module")
def ctx():
    return D().Context()


@pytest.mark.parametrize("metric", ["gate", "abs_gate", "gate_up", "abs_gate_up"])
def test_importance_bitexact_c1_fp32(ctx, metric):
    L = O.generate_layer(512, 1024, 8, 2, seed=1234)
    x = O.generate_tokens(256, 512, seed=99)
    r = O.route(L, x)
    pkg = D()
    layer = pkg.MoeLayer(512, 1024, 8, 2, L.gate, L.blocks, dtype="f32")
    vals = pkg.profile_importance(ctx, layer, torch.from_numpy(x).cuda(), torch.from_numpy(r.idx).cuda(), metric)
    assert np.array_equal(vals.cpu().numpy(), O.profile_importance(L, x, r.idx, metric))


def test_golden_reference_order_and_forward(ctx):
    """Against the reference's own outputs (tests/golden/c1_reference.npz)."""
    g = np.load(__file__.replace("test_gpu_reconstruct.py", "golden/c1_reference.npz"))
    L = O.generate_layer(512, 1024, 8, 2, seed=1234)
    x = g["x"]
    pkg = D()
    layer = pkg.MoeLayer(512, 1024, 8, 2, L.gate, L.blocks, dtype="f32")
    xd = torch.from_numpy(x).cuda()
    r0 = pkg.route_and_drop(ctx, layer, xd, logits_mode=pkg.LOGITS_EXACT)
    vals = pkg.profile_importance(ctx, layer, xd, r0.indices, "abs_gate")
    assert np.array_equal(vals.cpu().numpy(), g["importance"])
    rec, order = pkg.reconstruct_experts(ctx, layer, vals)
    assert np.array_equal(order.cpu().numpy(), g["order"])
    r = pkg.route_and_drop(ctx, rec, xd, pkg.DropPolicy.two_t_from(0.40), logits_mode=pkg.LOGITS_EXACT)
    idx, raw, norm, frac = r.host()
    for a, k in ((idx, "idx"), (raw, "raw"), (norm, "norm"), (frac, "frac")):
        assert np.array_equal(a, g[k]), k
    assert r.stats["drop_rate"] == float(g["drop_rate"])
    y = pkg.forward(ctx, rec, xd, pkg.DropPolicy.two_t_from(0.40), logits_mode=pkg.LOGITS_EXACT).cpu().numpy()
    assert scaled_residual(y[g["fwd_rows"]], g["y"]) < 1e-5


def test_bf16_reconstruction_with_shared(ctx):
    rng = np.random.default_rng(4)
    d, ffn, E, K, S = 256, 320, 16, 4, 1
    r16 = O.bf16_round
    mk = lambda *s: r16(rng.standard_normal(s, dtype=np.float32) / np.sqrt(d))
    L = O.Layer(d, ffn, E, K, mk(d, E), [(mk(d, ffn), mk(d, ffn), mk(ffn, d)) for _ in range(E)],
                [(mk(d, ffn), mk(d, ffn), mk(ffn, d)) for _ in range(S)])
    x = r16(rng.standard_normal((200, d), dtype=np.float32))
    r = O.route(L, x)
    want = O.profile_importance(L, x, r.idx, "abs_gate_up")
    pkg = D()
    layer = pkg.MoeLayer(d, ffn, E, K, L.gate, L.blocks, L.shared, dtype="bf16")
    xd = torch.from_numpy(x).cuda().bfloat16()
    vals = pkg.profile_importance(ctx, layer, xd, torch.from_numpy(r.idx).cuda(), "abs_gate_up")
    assert np.array_equal(vals.cpu().numpy(), want)
    rec, order = pkg.reconstruct_experts(ctx, layer, vals)
    orec = O.reconstruct(L, want)
    assert np.array_equal(order.cpu().numpy(), orec.neuron_order)
    y = pkg.forward(ctx, rec, xd, pkg.DropPolicy.two_t_from(0.2), logits_mode=pkg.LOGITS_EXACT).float().cpu().numpy()
    ro = O.route(orec, x, "2t", 0.2)
    assert ro.frac.min() == 0.0
    assert scaled_residual(y, O.moe_forward(orec, x, ro.idx, ro.raw, ro.frac)) < 1e-2


def test_reconstruct_rejects_partitioned_layer(ctx):
    L = O.partial_transform(O.generate_layer(64, 48, 4, 2, seed=1), 2)
    pkg = D()
    layer = pkg.MoeLayer(64, 48, 4, 2, L.gate, L.blocks, replay_factor=2, dtype="f32")
    with pytest.raises(pkg.DsmoeError) as e:
        pkg.reconstruct_experts(ctx, layer, torch.zeros((4, 48), dtype=torch.float64, device="cuda"))
    assert e.value.code == 3
