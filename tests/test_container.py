"""DSMOE1 containers: the loader reads what the
reference's own C ABI wrote (tests/golden/dsmoe1_small.*, made by
tools/make_golden.py --container from oracle/_ref/libdsmoe_ref.so) with the
reference's validation and error codes (io.cpp:177-327); on the GPU,
`container.infer` reproduces dsmoe_infer's accounting (capi.cpp:328-368)."""
import json
import os
import struct

import numpy as np
import pytest

import oracle as O

G = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
BIN, TOK, RES = (os.path.join(G, "dsmoe1_small" + s) for s in (".bin", ".tokens", ".json"))


def C():
    from paper_2508_18376_b200 import container
    return container


def test_tokens_match_reference_generator():
    x = C().load_tokens(TOK)
    assert x.shape == (96, 64)
    assert np.array_equal(x, O.generate_tokens(96, 64, seed=77))


def test_parse_matches_reference_reconstruction_chain():
    """Layer l = reconstruct(generate_synthetic(seed_l)) on the residual
    calibration stream, exactly as dsmoe_reconstruct builds it (capi.cpp:281-310)."""
    layers = C().parse_model(BIN)
    assert len(layers) == 2
    cur = C().load_tokens(TOK)
    for l, hl in enumerate(layers):
        assert hl.lineage == "reconstructed" and hl.replay_factor == 2
        base = O.generate_layer(64, 128, 8, 2, S=1, seed=O.splitmix_nth(4242, l))
        r = O.route(base, cur)
        vals = O.profile_importance(base, cur, r.idx, "abs_gate")
        rec = O.reconstruct(base, vals)
        assert np.array_equal(np.asarray(hl.neuron_order, np.int32), rec.neuron_order)
        assert np.array_equal(hl.gate, rec.gate)
        for (a1, a3, a2), (b1, b3, b2) in zip(hl.blocks, rec.blocks):
            assert np.array_equal(a1, b1) and np.array_equal(a3, b3) and np.array_equal(a2, b2)
        for (a1, a3, a2), (b1, b3, b2) in zip(hl.shared, base.shared):
            assert np.array_equal(a1, b1) and np.array_equal(a3, b3) and np.array_equal(a2, b2)
        cur = cur + O.moe_forward(base, cur, r.idx, r.raw, r.frac)


def _corrupt(tmp_path, mutate):
    raw = bytearray(open(BIN, "rb").read())
    raw = mutate(raw)
    p = tmp_path / "bad.bin"
    p.write_bytes(bytes(raw))
    return str(p)


@pytest.mark.parametrize("mutate,code", [
    (lambda r: b"XSMOE1\0\0" + r[8:], 5),                              # bad magic
    (lambda r: r[:12], 6),                                            # shorter than header
    (lambda r: r[:len(r) - 100], 6),                                  # payload truncated
    (lambda r: r[:16] + b"{not json" + r[25:], 7),                     # manifest not JSON
    (lambda r: r[:8] + struct.pack("<Q", 10 ** 9) + r[16:], 6),        # manifest length beyond file
])
def test_corrupt_containers_report_reference_codes(tmp_path, mutate, code):
    from paper_2508_18376_b200.dsmoe import DsmoeError
    with pytest.raises(DsmoeError) as e:
        C().parse_model(_corrupt(tmp_path, mutate))
    assert e.value.code == code


def test_misaligned_offset_is_schema_error(tmp_path):
    from paper_2508_18376_b200.dsmoe import DsmoeError
    raw = bytearray(open(BIN, "rb").read())
    (mlen,) = struct.unpack_from("<Q", raw, 8)
    man = json.loads(raw[16:16 + mlen])
    man["tensors"][1]["offset"] += 4
    body = json.dumps(man, separators=(",", ":")).encode()
    assert len(body) <= mlen
    raw[16:16 + mlen] = body + b" " * (mlen - len(body))
    p = tmp_path / "mis.bin"
    p.write_bytes(bytes(raw))
    with pytest.raises(DsmoeError) as e:
        C().parse_model(str(p))
    assert e.value.code == 7


def test_missing_file_is_io_error():
    from paper_2508_18376_b200.dsmoe import DsmoeError
    with pytest.raises(DsmoeError) as e:
        C().parse_model("/nonexistent/model.bin")
    assert e.value.code == 4


def test_policy_json_defaults():
    p = C().policy_from({"kind": "2t", "t_drop": 0.4}, False)
    assert (p.kind, p.t_major, p.t_minor, p.keep_top1, p.normalize) == ("2t", 0.4 - 0.01, 0.4 + 0.01, True, True)
    assert C().policy_from({"kind": "none"}, True).normalize is False


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["none", "2t", "1t"])
def test_gpu_infer_matches_reference_dsmoe_infer(name):
    golden = json.load(open(RES))[name]
    layers = C().load_model(BIN, dtype="f32")
    got = C().infer(layers, C().load_tokens(TOK), golden["policy"])
    want = golden["result"]
    assert got["drop_rate"] == want["drop_rate"]
    assert got["dropped_units"] == want["dropped_units"] and got["total_units"] == want["total_units"]
    assert got["total_flops"] == want["total_flops"] and got["saved_flops"] == want["saved_flops"]
    for a, b in zip(got["per_layer"], want["per_layer"]):
        for k in ("drop_rate", "dropped_units", "total_routed_units", "shared_units", "retained_flops"):
            assert a[k] == b[k], k
    assert abs(got["rel_error"] - want["rel_error"]) <= 1e-4 * max(1.0, want["rel_error"])
