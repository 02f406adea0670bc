"""GPU: the permutation's superchunk path.  After the fused gate + router
(gate_route_kernel) the permutation takes its chunk offsets from per-
superchunk histograms the router kernel accumulated (double-buffered by a
device epoch, the other buffer cleared by the router's last CTA) instead of
scanning every chunk behind a grid-wide barrier.

Bar: the permutation (row_token, slot_pos, segments) is bit-equal to the CPU
counting sort (oracle.permutation) of the routing the device reports, on one
context through a sequence that mixes batch sizes (one token, partial tiles,
more superchunks than one buffer row, the 64-superchunk cap), route-only
calls (the epoch advances with no permutation reading it), two-kernel
routings (exact logits: the superchunk sums are not used) and forwards —
and the forward output equals the one the chunk-scan path gives
(DSMOE_B200_PERMUTE_SC=0, in a subprocess: the switch is read once)."""
import os
import subprocess
import sys

import numpy as np
import pytest

import oracle as O

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "tests"))

D_MODEL = 256


def _setup(E=64, K=8, P=2):
    import paper_2508_18376_b200 as pkg
    from test_gpu_parity import rand_layer
    L = rand_layer(D_MODEL, 64, E, K, seed=7, P=P)
    layer = pkg.MoeLayer(L.d, L.ffn, L.E, L.K, L.gate, L.blocks, L.shared, replay_factor=L.P, dtype="bf16",
                         gate_prenormalized=L.prenorm)
    return pkg, L, layer


def _x(T, seed):
    return torch.from_numpy(O.bf16_round(np.random.default_rng(seed).standard_normal((T, D_MODEL),
                                                                                      dtype=np.float32))).cuda().to(torch.bfloat16)


# (T, what): "fwd" = forward (tensor logits: fused gate + router + superchunk
# permutation), "route" = route only, "exact" = forward on exact logits (two-kernel routing)
SEQ = [(4133, "fwd"), (1, "fwd"), (777, "route"), (40000, "fwd"), (129, "exact"), (129, "fwd"),
       (300, "route"), (300, "route"), (70000, "fwd"), (4133, "fwd")]


def _check_perm(pkg, ctx, layer, x, pol, mode):
    T, E, K, P = x.shape[0], layer.E, layer.K, layer.P
    r = pkg.route_and_drop(ctx, layer, x, pol, logits_mode=mode)
    idx, _, _, frac = r.host()
    y = pkg.forward(ctx, layer, x, pol, logits_mode=mode)
    rt, sp, sg = ctx.permutation(T, K, E)
    wrt, wsp, wsg = O.permutation(idx.reshape(T, K * P), frac.reshape(T, K * P), K, P, E)
    assert np.array_equal(sg, wsg)
    assert np.array_equal(rt, wrt)
    assert np.array_equal(sp, wsp)
    return y


@pytest.mark.parametrize("E,K,P", [(64, 8, 2), (24, 4, 2), (40, 16, 1)])
def test_superchunk_permutation_sequence(E, K, P):
    pkg, L, layer = _setup(E, K, P)
    ctx = pkg.Context()
    pol = pkg.DropPolicy.two_t_from(0.08) if P == 2 else pkg.DropPolicy.one_t(0.08)  # 2T needs P = 2
    for i, (T, what) in enumerate(SEQ):
        x = _x(T, 50 + i)
        if what == "route":
            pkg.route_and_drop(ctx, layer, x, pol)
            continue
        mode = pkg.LOGITS_EXACT if what == "exact" else pkg.LOGITS_TENSOR
        _check_perm(pkg, ctx, layer, x, pol, mode)
    ctx.check()


def test_superchunk_forward_equals_chunk_scan():
    pkg, L, layer = _setup()
    ctx = pkg.Context()
    pol = pkg.DropPolicy.two_t_from(0.08)
    outs = []
    for i, T in enumerate((4133, 40000)):
        outs.append(pkg.forward(ctx, layer, _x(T, 90 + i), pol).float().cpu().numpy())
    code = ("import sys, numpy as np, torch; sys.path.insert(0, %r); sys.path.insert(0, %r)\n"
            "import test_gpu_superchunk as S\n"
            "pkg, L, layer = S._setup(); ctx = pkg.Context(); pol = pkg.DropPolicy.two_t_from(0.08)\n"
            "for i, T in enumerate((4133, 40000)):\n"
            "    np.save(sys.argv[1] + '_%%d.npy' %% i, pkg.forward(ctx, layer, S._x(T, 90 + i), pol).float().cpu().numpy())\n"
            % (ROOT, os.path.join(ROOT, "tests")))
    import tempfile
    with tempfile.TemporaryDirectory() as td:
        env = dict(os.environ, DSMOE_B200_PERMUTE_SC="0")
        subprocess.run([sys.executable, "-c", code, os.path.join(td, "y")], check=True, env=env, cwd=ROOT)
        for i in range(2):
            assert np.array_equal(outs[i], np.load(os.path.join(td, "y_%d.npy" % i)))
