"""CPU: the reference's C interface served by libdsmoe_b200.so
(include/dsmoe_abi.h) — exports, host-side entry points and error behaviour,
checked against the reference's own libdsmoe.so compiled into oracle/_ref.

No GPU here: generation, DSMOE1 containers, model_info, status names and
the argument / document validation that happens before any device work.
The device entry points are compared with the reference in
tests/test_gpu_abi.py.
"""
import json
import os
import re
import subprocess

import pytest

import oracle as O

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF_LIB = os.path.join(ROOT, "oracle", "_ref", "libdsmoe_ref.so")


def abi():
    from paper_2508_18376_b200 import abi as A
    return A


@pytest.fixture(scope="module")
def ours():
    return abi().DsmoeAbi()


@pytest.fixture(scope="module")
def ref():
    if not os.path.exists(REF_LIB):
        pytest.skip("oracle/_ref not built (the reference compiled from /root/reference/proj)")
    return abi().DsmoeAbi(REF_LIB)


def header_functions():
    src = open(os.path.join(ROOT, "include", "dsmoe_abi.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(dsmoe_[a-z0-9_]+)\s*\(", src)))


def test_exports_every_reference_symbol(ours):
    names = header_functions()
    assert len(names) == 20
    out = subprocess.run(["nm", "-D", "--defined-only", ours.path], capture_output=True, text=True).stdout
    exported = set(re.findall(r"\bT (dsmoe_\w+)", out))
    assert not [n for n in names if n not in exported]
    assert set(abi().SYMBOLS) == set(names)
    if os.path.exists(REF_LIB):  # the same set the reference exports
        out = subprocess.run(["nm", "-D", "--defined-only", REF_LIB], capture_output=True, text=True).stdout
        ref_names = {n for n in re.findall(r"\bT (dsmoe_\w+)", out) if not n.startswith("dsmoe_b200")}
        assert ref_names == set(names)


def test_identity_and_status_names(ours, ref):
    assert ours.version() == ref.version()
    for c in range(-1, 10):
        assert ours.status_name(c) == ref.status_name(c)


CFG = {"d_model": 64, "d_ffn": 96, "num_experts": 6, "top_k": 2, "num_shared_experts": 1, "num_layers": 2}


@pytest.mark.parametrize("width", [4, 8])
def test_generate_and_save_byte_identical(ours, ref, tmp_path, width):
    """generate_synthetic / generate_model (io.cpp:330-360) and save_model
    (io.cpp:111-173): the same container bytes as the reference."""
    a, b = tmp_path / "ours.dsmoe", tmp_path / "ref.dsmoe"
    ours.save(ours.generate_model(CFG, seed=77, scale=1.0, scalar_width=width), str(a))
    ref.save(ref.generate_model(CFG, seed=77, scale=1.0, scalar_width=width), str(b))
    assert a.read_bytes() == b.read_bytes()


def test_generate_tokens_byte_identical(ours, ref, tmp_path):
    a, b = tmp_path / "a.tok", tmp_path / "b.tok"
    ours.generate_tokens(33, 64, 99, str(a), scale=0.5)
    ref.generate_tokens(33, 64, 99, str(b), scale=0.5)
    assert a.read_bytes() == b.read_bytes()


def test_load_reference_container_roundtrip(ours, ref, tmp_path):
    """A container the reference wrote (incl. a reconstructed layer with
    neuron_order, tests/golden/dsmoe1_small.bin) loads, describes and re-saves
    byte for byte."""
    src = os.path.join(ROOT, "tests", "golden", "dsmoe1_small.bin")
    m_o, m_r = ours.load(src), ref.load(src)
    assert ours.info(m_o) == ref.info(m_r)
    a, b = tmp_path / "a.dsmoe", tmp_path / "b.dsmoe"
    ours.save(m_o, str(a))
    ref.save(m_r, str(b))
    assert a.read_bytes() == b.read_bytes() == open(src, "rb").read()


def test_info_matches(ours, ref):
    for cfg in (CFG, {**CFG, "gate_prenormalized": True, "num_shared_experts": 0, "num_layers": 1}):
        assert ours.info(ours.generate_model(cfg, 5)) == ref.info(ref.generate_model(cfg, 5))


def _code(fn):
    try:
        fn()
    except abi().AbiError as e:
        return e.code
    return 0


def test_error_codes_match(ours, ref, tmp_path):
    """Error classes of the reference's entry points (capi.cpp:37-58,
    io.cpp:177-294), reached before any device work."""
    bad = tmp_path / "bad.bin"
    bad.write_bytes(b"NOTDSMOE" + b"\0" * 40)
    short = tmp_path / "short.bin"
    short.write_bytes(b"DSMOE1\0")
    good = os.path.join(ROOT, "tests", "golden", "dsmoe1_small.bin")
    trunc = tmp_path / "trunc.bin"
    trunc.write_bytes(open(good, "rb").read()[:-100])
    cases = [
        lambda L: L.load(str(bad)),
        lambda L: L.load(str(short)),
        lambda L: L.load(str(trunc)),
        lambda L: L.load(str(tmp_path / "missing.bin")),
        lambda L: L.generate_model("{not json"),
        lambda L: L.generate_model({"d_model": 8}),
        lambda L: L.generate_model({**CFG, "top_k": 9}),
        lambda L: L.generate_model(CFG, scalar_width=2),
        lambda L: L.generate_model({**CFG, "num_layers": 0}),
        lambda L: L.generate_tokens(0, 4, 1, str(tmp_path / "t")),
        lambda L: L.infer(L.generate_model(CFG), str(tmp_path / "none.tok"), {"kind": "2t", "t_drop": 0.1}),
        lambda L: L.infer(L.generate_model(CFG), str(tmp_path / "none.tok"), {"kind": "3t"}),
        lambda L: L.infer(L.generate_model(CFG), str(tmp_path / "none.tok"), {"kind": "1t"}),
        lambda L: L.infer(L.generate_model(CFG), str(tmp_path / "none.tok"),
                          {"kind": "2t", "t_drop": 0.1, "t_major": 0.3, "t_minor": 0.2}),
        lambda L: L.infer(L.generate_model(CFG), str(tmp_path / "none.tok"), "[1,"),
        lambda L: L.transform(L.generate_model(CFG), "sideways", 2),
        lambda L: L.reconstruct(L.generate_model(CFG), str(tmp_path / "none.tok"), "loudest"),
        lambda L: L.sweep(L.generate_model(CFG), str(tmp_path / "none.tok"), "2t", [0.3, 0.1]),
        lambda L: L.sweep(L.generate_model(CFG), str(tmp_path / "none.tok"), "xt", [0.1]),
    ]
    for i, fn in enumerate(cases):
        co, cr = _code(lambda: fn(ours)), _code(lambda: fn(ref))
        assert co == cr and co != 0, (i, co, cr, ours.last_error(), ref.last_error())


def test_sim_comm_not_served(ours):
    with pytest.raises(abi().AbiError) as e:
        ours.sim_comm({"ep": 2, "tp": 1, "tokens_per_device": 4, "bytes_per_token": 8, "alpha": 1e-6, "beta": 1e9})
    assert e.value.code == 3


def test_fp64_models_rejected_on_device_entry_points(ours, tmp_path):
    """scalar_width 8 models load / save / describe, but the device compute
    entry points refuse them (the device computes in fp32)."""
    m = ours.generate_model(CFG, scalar_width=8)
    assert ours.info(m)["scalar_width"] == 8
    tok = tmp_path / "t.tok"
    ours.generate_tokens(4, 64, 1, str(tok))
    with pytest.raises(abi().AbiError) as e:
        ours.infer(m, str(tok), {"kind": "none"})
    assert e.value.code == 1 and "scalar_width 8" in ours.last_error()


def test_null_frees(ours):
    ours.L.dsmoe_string_free(None)
    ours.L.dsmoe_model_free(None)
