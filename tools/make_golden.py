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


if __name__ == "__main__":
    main()
