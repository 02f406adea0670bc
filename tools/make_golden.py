"""Generate tests/golden/*.npz from the REFERENCE ITSELF (oracle/_ref, compiled
from /root/reference/proj by oracle/Makefile).  Run in the build container:

    python tools/make_golden.py

c1_reference.npz — BASELINE config C1 (E=8, K=2, d=512, ffn=1024, fp32):
tokens (seed 99), abs_gate importance on those tokens, the reconstruction
order, 2T(t=0.40) routing of the reconstructed layer and the reference's
moe_forward on a strided subset of rows.
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import oracle as O  # noqa: E402


def main():
    assert O.ref_available(), "build oracle/_ref first (make -C oracle)"
    T = 256
    R = O.RefLayer.generate(512, 1024, 8, 2, seed=1234)
    x = O.ref_generate_tokens(T, 512, 99)
    r0 = R.route_and_drop(x, 2, 1)
    vals = R.profile_importance(x, r0.idx, 8, 1024, "abs_gate")
    Rr, order = R.reconstruct(vals, 8, 1024)
    rr = Rr.route_and_drop(x, 2, 2, "2t", 0.40)
    rows = np.arange(0, T, 8)
    y = Rr.moe_forward(x[rows], rr.idx[rows], rr.raw[rows], rr.frac[rows])
    st = Rr.drop_stats(T, rr.pre_frac, rr.frac)
    os.makedirs(os.path.join(ROOT, "tests", "golden"), exist_ok=True)
    np.savez_compressed(os.path.join(ROOT, "tests", "golden", "c1_reference.npz"), T=T, x=x, importance=vals,
                        order=order, idx=rr.idx, raw=rr.raw, norm=rr.norm, frac=rr.frac, fwd_rows=rows, y=y,
                        drop_rate=st["drop_rate"])
    print("drop_rate", st["drop_rate"])


if __name__ == "__main__" and "--container" not in sys.argv:
    main()


def make_container_fixture():
    """dsmoe1_small.*: a 2-layer model generated, reconstructed (abs_gate),
    saved and inferred by the REFERENCE C ABI (oracle/_ref/libdsmoe_ref.so):
    the container, its calibration/eval token file and dsmoe_infer's JSON."""
    import ctypes as C
    import json
    ref = C.CDLL(os.path.join(ROOT, "oracle", "_ref", "libdsmoe_ref.so"))
    ref.dsmoe_last_error.restype = C.c_char_p
    ref.dsmoe_generate_model.argtypes = [C.c_char_p, C.c_uint64, C.c_double, C.c_int, C.POINTER(C.c_void_p)]
    ref.dsmoe_generate_tokens.argtypes = [C.c_int64, C.c_int64, C.c_uint64, C.c_double, C.c_char_p]
    ref.dsmoe_reconstruct.argtypes = [C.c_void_p, C.c_char_p, C.c_char_p, C.POINTER(C.c_void_p), C.c_void_p]
    ref.dsmoe_model_save.argtypes = [C.c_void_p, C.c_char_p]
    ref.dsmoe_infer.argtypes = [C.c_void_p, C.c_char_p, C.c_char_p, C.POINTER(C.c_char_p)]
    out_dir = os.path.join(ROOT, "tests", "golden")

    def ok(rc):
        assert rc == 0, ref.dsmoe_last_error().decode()

    cfg = json.dumps({"d_model": 64, "d_ffn": 128, "num_experts": 8, "top_k": 2, "num_shared_experts": 1,
                      "gate_prenormalized": False, "num_layers": 2}).encode()
    m = C.c_void_p()
    ok(ref.dsmoe_generate_model(cfg, 4242, 1.0, 4, C.byref(m)))
    tok = os.path.join(out_dir, "dsmoe1_small.tokens").encode()
    ok(ref.dsmoe_generate_tokens(96, 64, 77, 1.0, tok))
    rec = C.c_void_p()
    ok(ref.dsmoe_reconstruct(m, tok, b"abs_gate", C.byref(rec), None))
    ok(ref.dsmoe_model_save(rec, os.path.join(out_dir, "dsmoe1_small.bin").encode()))
    res = {}
    for name, pol in (("none", {"kind": "none"}), ("2t", {"kind": "2t", "t_drop": 0.40}),
                      ("1t", {"kind": "1t", "t_drop": 0.35, "keep_top1": False})):
        js = C.c_char_p()
        ok(ref.dsmoe_infer(rec, tok, json.dumps(pol).encode(), C.byref(js)))
        res[name] = {"policy": pol, "result": json.loads(js.value.decode())}
    ref.dsmoe_sweep.argtypes = [C.c_void_p, C.c_char_p, C.c_char_p, C.POINTER(C.c_double), C.c_size_t, C.c_int,
                                C.POINTER(C.c_char_p), C.POINTER(C.c_char_p)]
    ref.dsmoe_analyze_gating.argtypes = [C.c_void_p, C.c_char_p, C.c_int, C.POINTER(C.c_char_p),
                                         C.POINTER(C.c_char_p)]
    ths = [0.2, 0.3, 0.4, 0.5]
    arr = (C.c_double * len(ths))(*ths)
    for kind in ("1t", "2t"):
        js, cs = C.c_char_p(), C.c_char_p()
        ok(ref.dsmoe_sweep(rec, tok, kind.encode(), arr, len(ths), 1, C.byref(js), C.byref(cs)))
        res["sweep_" + kind] = json.loads(js.value.decode())
    js, cs = C.c_char_p(), C.c_char_p()
    ok(ref.dsmoe_analyze_gating(rec, tok, 10, C.byref(js), C.byref(cs)))
    res["gating"] = json.loads(js.value.decode())
    with open(os.path.join(out_dir, "dsmoe1_small.json"), "w") as f:
        json.dump(res, f, indent=1)
    print("container fixture:", {k: v["result"]["drop_rate"] for k, v in res.items() if "result" in v})


if __name__ == "__main__" and "--container" in sys.argv:
    make_container_fixture()
