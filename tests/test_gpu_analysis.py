"""Rate-targeted drop + gating analysis against the
reference's own dsmoe_sweep / dsmoe_analyze_gating output on the
reference-written container (tests/golden/dsmoe1_small.*)."""
import json
import os

import numpy as np
import pytest

import oracle as O

G = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
BIN, TOK, RES = (os.path.join(G, "dsmoe1_small" + s) for s in (".bin", ".tokens", ".json"))


def oracle_gating(L, x, bins):
    """analyze_gating (dropping.hpp:207-228) restated on the oracle routing."""
    lg = O.gate_logits(x, L.gate)
    r = O.route_from_logits(lg, L.K, 1)
    counts = np.bincount(r.idx.ravel(), minlength=L.E)
    b = lambda v: np.clip((v * bins).astype(np.int64), 0, bins - 1)
    return counts.tolist(), np.bincount(b(r.raw.ravel()), minlength=bins).tolist(), \
        np.bincount(b(r.norm.ravel()), minlength=bins).tolist()


def test_oracle_gating_matches_reference():
    from paper_2508_18376_b200 import container
    g = json.load(open(RES))["gating"]
    hl = container.parse_model(BIN)[0]
    L = O.Layer(64, 128, 8, 2, np.asarray(hl.gate, np.float32), [], [])
    sc, rh, nh = oracle_gating(L, container.load_tokens(TOK), 10)
    assert sc == g["selection_counts"] and rh == g["raw_hist"] and nh == g["norm_hist"]


@pytest.mark.gpu
def test_gpu_gating_matches_reference():
    import torch
    from paper_2508_18376_b200 import analysis, container
    import paper_2508_18376_b200 as D
    g = json.load(open(RES))["gating"]
    layers = container.load_model(BIN, dtype="f32")
    x = torch.from_numpy(container.load_tokens(TOK)).cuda()
    got = analysis.analyze_gating(D.Context(), layers[0], x, 10)
    for k in ("selection_counts", "raw_hist", "norm_hist", "num_tokens", "top_k", "bins"):
        assert got[k] == g[k], k


@pytest.mark.gpu
@pytest.mark.parametrize("kind", ["1t", "2t"])
def test_gpu_sweep_matches_reference(kind):
    import torch
    from paper_2508_18376_b200 import analysis, container
    import paper_2508_18376_b200 as D
    want = json.load(open(RES))["sweep_" + kind]
    layers = container.load_model(BIN, dtype="f32")
    x = torch.from_numpy(container.load_tokens(TOK)).cuda()
    got = analysis.threshold_sweep(D.Context(), layers, x, kind, [r["threshold"] for r in want["rows"]])
    assert got["policy_kind"] == want["policy_kind"]
    for a, b in zip(got["rows"], want["rows"]):
        assert a["drop_rate"] == b["drop_rate"]
        assert a["per_layer_rates"] == b["per_layer_rates"]
        assert abs(a["mean_rel_error"] - b["mean_rel_error"]) <= 1e-4 * max(1.0, b["mean_rel_error"])


@pytest.mark.gpu
def test_gpu_calibrate_rate_hits_target():
    import torch
    import paper_2508_18376_b200 as D
    from paper_2508_18376_b200 import analysis
    L = O.reconstruct(*(lambda b, x: (b, O.profile_importance(b, x, O.route(b, x).idx, "abs_gate")))(
        O.generate_layer(128, 256, 16, 4, seed=9), O.generate_tokens(512, 128, 10)))
    x = O.generate_tokens(2048, 128, 11)
    layer = D.MoeLayer(L.d, L.ffn, L.E, L.K, L.gate, L.blocks, replay_factor=2, dtype="f32")
    ctx = D.Context()
    for target in (0.25, 0.5):
        pol, rate = analysis.calibrate_rate(ctx, layer, torch.from_numpy(x).cuda(), target, tol=0.01)
        assert abs(rate - target) <= 0.01
        ro = O.route(L, x, "2t", pol.t_drop)
        assert O.drop_stats(ro.pre_frac, ro.frac, 2, 0, x.shape[0], 128, 256)["drop_rate"] == rate
