"""GPU: the expert-parallel data path (ep.py) — dispatch, all-to-all, expert
FFN over received segments, reverse all-to-all, combine — for D virtual ranks
on one GPU (EpEmulator) and for a real 1-rank NCCL group, against the oracle's
simulate_step (ep_sim.hpp:110-160) + moe_forward on all ranks' tokens."""
import os
import socket

import numpy as np
import pytest

import oracle as O

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


def D():
    import paper_2508_18376_b200 as pkg
    return pkg


def skewed(T=400, E=8, K=2, d=128, ffn=192, seed=31, S=0):
    L = O.generate_layer(d, ffn, E, K, S=S, seed=seed)
    x = O.generate_tokens(T, d, seed + 1)
    x += (1.5 / np.linalg.norm(L.gate[:, 3])) * L.gate[:, 3]
    x = x.astype(np.float32)
    rec = O.reconstruct(L, O.profile_importance(L, x, O.route(L, x).idx, "abs_gate"))
    return rec, x


def dev_layer(L):
    return D().MoeLayer(L.d, L.ffn, L.E, L.K, L.gate, L.blocks, L.shared, replay_factor=L.P, dtype="f32")


@pytest.mark.parametrize("devices", [2, 4])
@pytest.mark.parametrize("load_aware", [True, False])
def test_ep_emulator_matches_simulate_step(devices, load_aware):
    from paper_2508_18376_b200 import ep
    rec, x = skewed()
    layer = dev_layer(rec)
    shards = np.array_split(np.arange(x.shape[0]), devices)
    xs = [torch.from_numpy(x[s]).cuda() for s in shards]
    emu = ep.EpEmulator(layer, devices)
    pol = D().DropPolicy.two_t_from(0.3)
    outs, rep = emu.forward(xs, pol, load_aware=load_aware, logits_mode=D().LOGITS_EXACT)
    ref = O.simulate_step(O.gate_logits(x, rec.gate), rec, devices, "2t", 0.3, load_aware=load_aware)
    assert np.array_equal(rep["pre_loads"], ref["pre_loads"])
    assert np.array_equal(rep["thresholds"], ref["thresholds"])
    assert np.array_equal(rep["post_loads"], ref["post_loads"])
    assert rep["speedup"] == ref["speedup"]
    ro = O.route_from_logits(O.gate_logits(x, rec.gate), rec.K, rec.P)
    yo = O.moe_forward(rec, x, ref["idx"], ro.raw, ref["frac"])
    y = torch.cat(outs).cpu().numpy()
    assert np.abs(y - yo).max() / np.abs(yo).max() < 1e-5


def test_ep_emulator_shared_experts_bf16():
    from paper_2508_18376_b200 import ep
    rec, x = skewed(T=300, E=8, K=2, d=128, ffn=128, S=1)
    xb = O.bf16_round(x)
    pkg = D()
    layer = pkg.MoeLayer(rec.d, rec.ffn, rec.E, rec.K, rec.gate, rec.blocks, rec.shared, replay_factor=2,
                         dtype="bf16")
    shards = np.array_split(np.arange(x.shape[0]), 2)
    xs = [torch.from_numpy(xb[s]).cuda().bfloat16() for s in shards]
    outs, rep = ep.EpEmulator(layer, 2).forward(xs, pkg.DropPolicy.two_t_from(0.3), logits_mode=pkg.LOGITS_EXACT)
    recb = rec.round_bf16()
    ref = O.simulate_step(O.gate_logits(xb, recb.gate), recb, 2, "2t", 0.3)
    ro = O.route_from_logits(O.gate_logits(xb, recb.gate), recb.K, 2)
    yo = O.moe_forward(recb, xb, ref["idx"], ro.raw, ref["frac"])
    y = torch.cat(outs).float().cpu().numpy()
    assert np.abs(y - yo).max() / np.abs(yo).max() < 1e-2


def test_ep_nccl_single_rank():
    import torch.distributed as dist
    from paper_2508_18376_b200 import ep
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("nccl", rank=0, world_size=1)
    try:
        rec, x = skewed(T=200)
        layer = dev_layer(rec)
        m = ep.ExpertParallelMoE(layer)
        y, rep = m.forward(torch.from_numpy(x).cuda(), D().DropPolicy.two_t_from(0.3), logits_mode=D().LOGITS_EXACT)
        ref = O.simulate_step(O.gate_logits(x, rec.gate), rec, 1, "2t", 0.3)
        ro = O.route_from_logits(O.gate_logits(x, rec.gate), rec.K, rec.P)
        yo = O.moe_forward(rec, x, ref["idx"], ro.raw, ref["frac"])
        assert np.abs(y.cpu().numpy() - yo).max() / np.abs(yo).max() < 1e-5
        assert np.array_equal(rep["pre_loads"], ref["pre_loads"])
    finally:
        dist.destroy_process_group()
