"""CPU: pin the oracle (oracle/dsmoe_oracle.c) before trusting it.

1. The reference's own known-answer tests, restated (file:line under
   /root/reference/proj/tests).
2. Bit-equality with the reference itself compiled from its sources into
   oracle/_ref/ (skipped where that build is absent).
3. Bit-equality with the committed golden fixtures tests/golden/*.npz, which
   tools/make_golden.py generated from the compiled reference.
"""
import os

import numpy as np
import pytest

import oracle as O

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
need_ref = pytest.mark.skipif(not O.ref_available(), reason="compiled reference (oracle/_ref) absent")
f32 = np.float32


# ------------------------------------------------------- known-answer tests
def test_topk_picks_largest_in_index_order():  # test_moe_model.cpp:38-47
    idx, raw = O.topk(np.array([[0.1, 0.4, 0.3, 0.2]], f32), 2)
    assert idx.tolist() == [[1, 2]]
    assert raw.tolist() == [[float(f32(0.4)), float(f32(0.3))]]


def test_topk_ties_go_to_lower_index():  # test_moe_model.cpp:49-55
    assert O.topk(np.full((1, 4), 0.25, f32), 2)[0].tolist() == [[0, 1]]
    assert O.topk(np.array([[0.1, 0.3, 0.3, 0.2]], f32), 2)[0].tolist() == [[1, 2]]


def test_topk_rejects_bad_k():  # test_moe_model.cpp:57-60
    for k in (0, 3):
        with pytest.raises(O.OracleError):
            O.topk(np.array([[0.5, 0.5]], f32), k)


def test_replay_is_copy_major():  # test_moe_model.cpp:186-208
    # logits whose top-2 are experts 3 then 1
    r = O.route_from_logits(np.array([[0.0, 1.0, 0.0, 2.0]], f32), K=2, P=2)
    assert r.idx.tolist() == [[6, 2, 7, 3]]
    assert r.raw[0, 0] == r.raw[0, 2] and r.raw[0, 1] == r.raw[0, 3]
    assert r.frac.tolist() == [[1.0, 1.0, 1.0, 1.0]]


def test_normalize_divides_by_topk_sum():  # test_dropping.cpp:61-70
    n = O.normalize(np.array([[0.4, 0.3]]), K=2)
    assert n[0, 0] == pytest.approx(4 / 7, rel=1e-15)
    assert n[0, 1] == pytest.approx(3 / 7, rel=1e-15)
    with pytest.raises(O.OracleError):
        O.normalize(np.array([[0.0, 0.0]]), K=2)


def test_normalize_uses_base_k_only_after_replay():  # dropping.hpp:64-66
    n = O.normalize(np.array([[0.6, 0.2, 0.6, 0.2]]), K=2, P=2)
    assert n.tolist() == [[0.6 / 0.8, 0.2 / 0.8, 0.6 / 0.8, 0.2 / 0.8]]


def test_1t_inclusive_threshold():  # test_dropping.cpp:88-102
    assert O.apply_bands(O.normalize(np.array([[0.8, 0.2]]), 2), 2, 1, 0.5, 0.5).tolist() == [[1.0, 0.0]]
    assert O.apply_bands(O.normalize(np.array([[0.5, 0.5]]), 2), 2, 1, 0.5, 0.5).tolist() == [[1.0, 1.0]]


def test_keep_top1_guard():  # test_dropping.cpp:104-111
    ns = O.normalize(np.array([[0.3, 0.2]]), 2)  # 0.6, 0.4
    assert O.apply_bands(ns, 2, 1, 0.9, 0.9, keep_top1=True).tolist() == [[1.0, 0.0]]
    assert O.apply_bands(ns, 2, 1, 0.9, 0.9, keep_top1=False).tolist() == [[0.0, 0.0]]


def test_2t_bands():  # test_dropping.cpp:113-128
    ns = np.array([[0.10, 0.08, 0.05, 0.10, 0.08, 0.05]])
    assert O.apply_bands(ns, 3, 2, 0.07, 0.09, keep_top1=False).tolist() == [[1, 1, 0, 1, 0, 0]]
    nb = np.array([[0.09, 0.07, 0.09, 0.07]])
    assert O.apply_bands(nb, 2, 2, 0.07, 0.09, keep_top1=False).tolist() == [[1, 1, 1, 0]]


def test_2t_collapsed_band_equals_1t():  # test_dropping.cpp:130-147
    rng = np.random.default_rng(77)
    for _ in range(25):
        v = 0.05 + rng.random(3)
        v /= v.sum()
        ns = np.concatenate([v, v])[None, :]
        t = 0.05 + 0.5 * rng.random()
        assert np.array_equal(O.apply_bands(ns, 3, 2, t, t), O.apply_bands(ns, 3, 2, t, t))
        one = O.apply_bands(ns[:, :3], 3, 1, t, t)
        assert np.array_equal(O.apply_bands(ns, 3, 2, t, t)[:, :3], one)


def test_p1_middle_band_is_half():  # dropping.hpp:105-110
    ns = np.array([[0.5, 0.3, 0.2]])
    assert O.apply_bands(ns, 3, 1, 0.25, 0.4, keep_top1=False).tolist() == [[1.0, 0.5, 0.0]]


def test_drop_accounting_fixture():  # test_dropping.cpp:149-179
    pre = np.ones(1000)
    post = np.ones(1000)
    post[:100] = 0.0
    post[100:300] = 0.5
    st = O.drop_stats(pre, post, 1, 0, 500, 16, 24)
    assert st["total_routed_units"] == 1000.0 and st["dropped_units"] == 200.0
    assert st["drop_rate"] == pytest.approx(0.20, rel=1e-15)
    assert st["total_flops"] == 1000.0 * 6 * 16 * 24
    assert st["retained_flops"] + st["saved_flops"] == st["total_flops"]
    sh = O.drop_stats(pre, post, 1, 1, 500, 16, 24)
    assert sh["shared_units"] == 500.0
    assert sh["drop_rate"] == pytest.approx(200 / 1500, rel=1e-15)


def test_replayed_half_drop_weighs_half():  # test_dropping.cpp:181-189
    st = O.drop_stats(np.ones(4), np.array([1.0, 1.0, 1.0, 0.0]), 2, 0, 1, 16, 24)
    assert st["total_routed_units"] == 2.0 and st["dropped_units"] == 0.5 and st["drop_rate"] == 0.25


def test_reconstruction_order_stable_descending():  # test_reconstruct.cpp:125-136, :138-183
    assert O.reconstruction_order(np.array([[0.3, 0.9, 0.3, 0.1, 0.9, 0.5]])).tolist() == [[1, 4, 5, 0, 2, 3]]
    assert O.reconstruction_order(np.ones((4, 24))).tolist() == [list(range(24))] * 4
    assert O.reconstruction_order(np.tile([0.1, 0.2, 0.3, 0.4], (3, 1))).tolist() == [[3, 2, 1, 0]] * 3


def test_uniform_reconstruction_equals_partial_p2():  # test_reconstruct.cpp:138-161
    L = O.generate_layer(64, 24, 4, 2, seed=12)
    rec = O.reconstruct(L, np.ones((4, 24)))
    part = O.partial_transform(L, 2)
    assert np.array_equal(rec.flat(), part.flat())


def test_placement_and_loads():  # test_ep_sim.cpp:31-69
    assert O.place_experts(8, 4, round_robin=True).tolist() == [0, 1, 2, 3, 0, 1, 2, 3]
    assert O.place_experts(8, 4).tolist() == [0, 0, 1, 1, 2, 2, 3, 3]
    with pytest.raises(O.OracleError):
        O.place_experts(6, 4)
    with pytest.raises(O.OracleError):
        O.place_experts(3, 4, round_robin=True)
    idx = np.array([0, 2, 1, 3, 4, 6, 5, 7])
    frac = np.array([1.0, 1.0, 1.0, 0.0, 1.0, 0.5, 1.0, 0.0])
    loads = O.device_loads(idx, frac, 2, O.place_experts(8, 2), 2)
    assert loads.tolist() == [1.5, 1.25]


def test_load_aware_thresholds():  # test_ep_sim.cpp:71-91
    ts = O.load_aware_thresholds([120.0, 80.0, 100.0, 100.0], 0.12)
    assert ts[0] == 0.12 and ts[2] == 0.12 and ts[3] == 0.12
    assert ts[1] == pytest.approx(0.096, rel=1e-15)
    assert O.load_aware_thresholds([50.0, 50.0], 0.3).tolist() == [0.3, 0.3]
    assert O.load_aware_thresholds([10.0, 0.0], 0.2)[1] == 0.0
    for bad in ((0.0, [1.0, 1.0]), (1.5, [1.0, 1.0]), (0.5, [0.0, 0.0])):
        with pytest.raises(O.OracleError):
            O.load_aware_thresholds(bad[1], bad[0])


def test_forward_linear_in_raw_score():  # test_moe_model.cpp:118-130
    L = O.generate_layer(64, 32, 4, 2, seed=5)
    x = O.generate_tokens(8, 64, seed=6)
    r = O.route(L, x)
    y1 = O.moe_forward(L, x, r.idx, r.raw, r.frac)
    y2 = O.moe_forward(L, x, r.idx, 2 * r.raw, r.frac)
    assert np.allclose(y2, 2 * y1, rtol=1e-5, atol=1e-6)


def test_shared_experts_unweighted():  # test_moe_model.cpp:161-184
    L = O.generate_layer(64, 32, 4, 2, S=1, seed=5)
    x = O.generate_tokens(8, 64, seed=6)
    r = O.route(L, x)
    y = O.moe_forward(L, x, r.idx, r.raw, np.zeros_like(r.frac))
    only_shared = O.Layer(64, 32, 1, 1, L.gate[:, :1], [L.shared[0]], [])
    ys = O.moe_forward(only_shared, x, np.zeros((8, 1), np.int32), np.ones((8, 1)), np.ones((8, 1)))
    assert np.array_equal(y, ys)


# -------------------------------------------------- vs the compiled reference
@need_ref
def test_generators_match_reference():
    L = O.generate_layer(64, 48, 4, 2, S=1, seed=1234)
    R = O.RefLayer.generate(64, 48, 4, 2, S=1, seed=1234)
    assert np.array_equal(L.flat(), R.to_layer().flat())
    assert np.array_equal(O.generate_tokens(16, 64, 99), O.ref_generate_tokens(16, 64, 99))


@need_ref
@pytest.mark.parametrize("P", [1, 2])
@pytest.mark.parametrize("kind,t", [("none", 0), ("1t", 0.2), ("1t", 0.45), ("2t", 0.2), ("2t", 0.31)])
@pytest.mark.parametrize("keep", [True, False])
def test_routing_matches_reference(P, kind, t, keep):
    if kind == "2t" and P != 2:
        pytest.skip("drop_2t needs P=2")
    rng = np.random.default_rng(3)
    logits = rng.standard_normal((300, 8), dtype=f32)
    logits[:20] = 0.0                      # all-tie rows
    logits[20:40, 1] = logits[20:40, 5]    # pairwise ties
    mine = O.route_from_logits(logits, 2, P, kind, t, keep_top1=keep)
    ref = O.ref().refshim_route_from_logits
    import ctypes as C
    n = 300 * 2 * P
    out = [np.empty(n, np.int32)] + [np.empty(n, np.float64) for _ in range(4)]
    ref.argtypes = [O.f32p, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_double, C.c_double,
                    C.c_double, C.c_int, C.c_int, O.i32p, O.f64p, O.f64p, O.f64p, O.f64p]
    tmaj, tmin = (t - 0.01, t + 0.01) if kind == "2t" else (0.0, 0.0)
    O._chk(ref(logits, 300, 8, 2, P, O.KIND[kind], t, tmaj, tmin, int(keep), 1, *out), "ref")
    for a, b in zip((mine.idx, mine.raw, mine.norm, mine.frac, mine.pre_frac), out):
        assert np.array_equal(a.ravel(), b)


@need_ref
def test_c1_pipeline_matches_reference():
    """C1: generate -> route -> profile(abs_gate) -> reconstruct -> 2T(0.40) -> forward."""
    L = O.generate_layer(512, 1024, 8, 2, seed=1234)
    R = O.RefLayer.generate(512, 1024, 8, 2, seed=1234)
    x = O.generate_tokens(64, 512, 99)
    r0 = O.route(L, x)
    vals = O.profile_importance(L, x, r0.idx, "abs_gate")
    assert np.array_equal(vals, R.profile_importance(x, r0.idx, 8, 1024, "abs_gate"))
    rec = O.reconstruct(L, vals)
    Rr, order = R.reconstruct(vals, 8, 1024)
    assert np.array_equal(order, rec.neuron_order)
    assert np.array_equal(Rr.to_layer().flat(), rec.flat())
    ro = O.route(rec, x, "2t", 0.40)
    rr = Rr.route_and_drop(x, 2, 2, "2t", 0.40)
    for a, b in zip((ro.idx, ro.raw, ro.norm, ro.frac), (rr.idx, rr.raw, rr.norm, rr.frac)):
        assert np.array_equal(a, b)
    assert np.array_equal(O.moe_forward(rec, x, ro.idx, ro.raw, ro.frac),
                          Rr.moe_forward(x, rr.idx, rr.raw, rr.frac))
    assert O.drop_stats(ro.pre_frac, ro.frac, 2, 0, 64, 512, 1024) == Rr.drop_stats(64, rr.pre_frac, rr.frac)


@need_ref
@pytest.mark.parametrize("metric", ["gate", "abs_gate", "gate_up", "abs_gate_up"])
def test_importance_metrics_match_reference(metric):
    L = O.generate_layer(64, 48, 4, 2, seed=21)
    R = O.RefLayer.generate(64, 48, 4, 2, seed=21)
    x = O.generate_tokens(40, 64, 22)
    r = O.route(L, x)
    assert np.array_equal(O.profile_importance(L, x, r.idx, metric), R.profile_importance(x, r.idx, 4, 48, metric))


@need_ref
@pytest.mark.parametrize("complete", [False, True])
def test_transforms_match_reference(complete):
    L = O.generate_layer(64, 48, 4, 2, S=1, seed=8)
    R = O.RefLayer.generate(64, 48, 4, 2, S=1, seed=8)
    mine = O.complete_transform(L, 4) if complete else O.partial_transform(L, 4)
    theirs = R.transform(complete, 4).to_layer()
    assert np.array_equal(mine.flat(), theirs.flat())
    assert (mine.E, mine.K, mine.P) == (theirs.E, theirs.K, theirs.P)


@need_ref
@pytest.mark.parametrize("load_aware", [True, False])
@pytest.mark.parametrize("kind,t", [("1t", 0.25), ("2t", 0.25)])
def test_simulate_step_matches_reference(load_aware, kind, t):
    L = O.generate_layer(64, 48, 8, 2, seed=31)
    x = O.generate_tokens(200, 64, 32)
    x += (1.5 / np.linalg.norm(L.gate[:, 3])) * L.gate[:, 3]  # skew toward expert 3 (acceptance.cpp:381-387)
    x = x.astype(f32)
    rec = O.reconstruct(L, O.profile_importance(L, x, O.route(L, x).idx, "abs_gate"))
    R = O.RefLayer.from_layer(rec)
    mine = O.simulate_step(O.gate_logits(x, rec.gate), rec, 4, kind, t, load_aware=load_aware)
    ref = R.simulate_step(x, 4, 2, 2, kind, t, load_aware=load_aware)
    for k in ("pre_loads", "post_loads", "thresholds", "idx", "frac"):
        assert np.array_equal(mine[k], ref[k]), k
    for k in ("ideal_load", "drop_rate", "speedup"):
        assert mine[k] == ref[k], k


# ------------------------------------------------------------ golden fixtures
def _golden(name):
    p = os.path.join(GOLDEN, name)
    if not os.path.exists(p):
        pytest.skip(f"{name} not generated")
    return np.load(p)


def test_golden_c1_routing_and_forward():
    g = _golden("c1_reference.npz")
    L = O.generate_layer(512, 1024, 8, 2, seed=1234)
    x = O.generate_tokens(int(g["T"]), 512, 99)
    assert np.array_equal(x, g["x"])
    r0 = O.route(L, x)
    vals = O.profile_importance(L, x, r0.idx, "abs_gate")
    assert np.array_equal(vals, g["importance"])
    rec = O.reconstruct(L, vals)
    assert np.array_equal(rec.neuron_order, g["order"])
    ro = O.route(rec, x, "2t", 0.40)
    for k in ("idx", "raw", "norm", "frac"):
        assert np.array_equal(getattr(ro, k), g[k]), k
    sel = g["fwd_rows"]
    y = O.moe_forward(rec, x[sel], ro.idx[sel], ro.raw[sel], ro.frac[sel])
    assert np.array_equal(y, g["y"])
    assert O.drop_stats(ro.pre_frac, ro.frac, 2, 0, x.shape[0], 512, 1024)["drop_rate"] == float(g["drop_rate"])
