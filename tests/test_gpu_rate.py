"""GPU: rate-targeted drop on the device (north star item 2).  The device
bisection (dsmoe_b200_calibrate_rate / _forward_rate) must pick the same
threshold, bit for bit, as the host loop over route_and_drop's drop_stats
(the acceptance.cpp:342-352 method, analysis.calibrate_rate), and the
forward under it must equal the forward with that threshold as a policy."""
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
    torch.cuda.set_device(0)
    return D().Context()


def dev_layer(L, dtype="f32", prenorm=False):
    return D().MoeLayer(L.d, L.ffn, L.E, L.K, L.gate, L.blocks, L.shared, replay_factor=L.P, dtype=dtype,
                        gate_prenormalized=prenorm)


CASES = [  # (P, kind, target, keep_top1, S, normalize)
    (2, "2t", 0.25, True, 0, None), (2, "2t", 0.5, True, 1, None), (2, "1t", 0.3, False, 0, None),
    (1, "1t", 0.25, True, 0, None), (2, "2t", 0.2, True, 0, False), (4, "1t", 0.35, True, 0, None),
]


@pytest.mark.parametrize("P,kind,target,keep,S,normalize", CASES)
def test_device_bisection_equals_host(ctx, P, kind, target, keep, S, normalize):
    pkg = D()
    from paper_2508_18376_b200 import analysis as A
    L = O.generate_layer(128, 256, 16, 4, S=S, seed=31 + P)
    L = O.partial_transform(L, P) if P > 1 else L
    layer = dev_layer(L)
    x = torch.from_numpy(O.generate_tokens(600, 128, seed=32)).cuda()
    hp, hr = A.calibrate_rate(ctx, layer, x, target, kind=kind, keep_top1=keep, logits_mode=pkg.LOGITS_EXACT) \
        if normalize is None else _host_cal(ctx, layer, x, target, kind, keep, normalize)
    dp, dr = pkg.calibrate_rate(ctx, layer, x, target, kind=kind, keep_top1=keep, normalize=normalize,
                                logits_mode=pkg.LOGITS_EXACT)
    assert dp.t_drop == hp.t_drop and dr == hr
    # the forward under the device-chosen threshold, without a host round trip
    tr = torch.empty(2, dtype=torch.float64, device="cuda")
    y, st = pkg.forward_rate(ctx, layer, x, target, kind=kind, keep_top1=keep, normalize=normalize,
                             logits_mode=pkg.LOGITS_EXACT, with_stats=True, t_rate=tr)
    y2, st2 = pkg.forward(ctx, layer, x, dp, logits_mode=pkg.LOGITS_EXACT, with_stats=True)
    assert tr.cpu().tolist() == [dp.t_drop, dr]
    assert st == st2 and st["drop_rate"] == dr
    assert torch.equal(y, y2)


def _host_cal(ctx, layer, x, target, kind, keep, normalize, tol=0.005, iters=40):
    pkg = D()
    lo, hi, best = 0.0, 1.0, None
    for _ in range(iters):
        t = 0.5 * (lo + hi)
        pol = pkg.DropPolicy.two_t_from(t, keep) if kind == "2t" else pkg.DropPolicy.one_t(t, keep)
        pol.normalize = normalize
        r = pkg.route_and_drop(ctx, layer, x, pol, logits_mode=pkg.LOGITS_EXACT).stats["drop_rate"]
        if best is None or abs(r - target) < abs(best[1] - target):
            best = (pol, r)
        if abs(r - target) <= tol:
            break
        lo, hi = (t, hi) if r < target else (lo, t)
    return best


def test_bench_scale_bf16(ctx):
    """C2 shape, 16384 bf16 tokens, tensor-core logits: the device picks the
    threshold bench.py's host bisection picks."""
    pkg = D()
    rng = np.random.default_rng(5)
    d, ffn, E, K = 2048, 1024, 64, 8
    r = lambda *s: O.bf16_round(rng.standard_normal(s, dtype=np.float32) * d ** -0.5)
    L = O.partial_transform(O.Layer(d, ffn, E, K, r(d, E), [(r(d, ffn), r(d, ffn), r(ffn, d)) for _ in range(E)]), 2)
    layer = dev_layer(L, "bf16")
    x = torch.randn(16384, d, device="cuda").bfloat16()
    for target in (0.25, 0.5):
        hp, hr = _host_cal_tensor(ctx, layer, x, target)
        dp, dr = pkg.calibrate_rate(ctx, layer, x, target)
        assert dp.t_drop == hp.t_drop and dr == hr


def _host_cal_tensor(ctx, layer, x, target, tol=0.005):
    pkg = D()
    lo, hi, best = 0.0, 1.0, None
    for _ in range(40):
        t = 0.5 * (lo + hi)
        r = pkg.route_and_drop(ctx, layer, x, pkg.DropPolicy.two_t_from(t)).stats["drop_rate"]
        if best is None or abs(r - target) < abs(best[1] - target):
            best = (pkg.DropPolicy.two_t_from(t), r)
        if abs(r - target) <= tol:
            break
        lo, hi = (t, hi) if r < target else (lo, t)
    return best
