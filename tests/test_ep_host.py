"""CPU, world_size 2 over gloo: the expert-parallel host policy (ep.py) gives
the reference simulate_step's loads and thresholds (ep_sim.hpp:110-160) on
the concatenation of the ranks' tokens, and the count / split bookkeeping of
the all-to-all exchange is consistent."""
import os
import socket

import numpy as np
import pytest

import oracle as O

torch = pytest.importorskip("torch")


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def skewed_case(T=240, E=8, K=2, d=64, ffn=48, seed=31):
    L = O.generate_layer(d, ffn, E, K, seed=seed)
    x = O.generate_tokens(T, d, seed + 1)
    x += (1.5 / np.linalg.norm(L.gate[:, 3])) * L.gate[:, 3]  # acceptance.cpp:381-387
    x = x.astype(np.float32)
    rec = O.reconstruct(L, O.profile_importance(L, x, O.route(L, x).idx, "abs_gate"))
    return rec, x


def _worker(rank, world, port, results):
    import torch.distributed as dist
    from paper_2508_18376_b200 import ep

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    rec, x = skewed_case()
    shard = np.array_split(np.arange(x.shape[0]), world)[rank]
    xs = x[shard]
    lg = O.gate_logits(xs, rec.gate)
    r = O.route_from_logits(lg, rec.K, rec.P)
    owner = ep.owner_of_experts(rec.E, rec.P, 4)
    counts = np.bincount(r.idx[:, :rec.K].ravel() // rec.P, minlength=rec.E)
    t = torch.from_numpy(counts.astype(np.int64))
    dist.all_reduce(t)
    pre = ep.loads_from_counts(t.numpy(), ep.block_devices(rec.E, rec.P, 4), 4, rec.P)
    th = ep.device_thresholds(pre, 0.3, True)
    # dispatch bookkeeping: seg from the oracle permutation of the dropped routing
    tmaj = th[owner][r.idx[:, :rec.K] // rec.P] - 0.01
    tmin = th[owner][r.idx[:, :rec.K] // rec.P] + 0.01
    rd = O.route_from_logits(lg, rec.K, rec.P, "1t", 0.0, t_major_slot=tmaj, t_minor_slot=tmin)
    _, _, seg = O.permutation(rd.idx, rd.frac, rec.K, rec.P, rec.E)
    # every rank plays 2 devices' worth of experts: 4 devices over 2 ranks
    owner2 = ep.owner_of_experts(rec.E, rec.P, world)
    send = ep.send_counts(seg, owner2, world)
    cnt_send = torch.from_numpy(ep.counts_for_receivers(seg, owner2, world))
    cnt_recv = torch.empty_like(cnt_send)
    dist.all_to_all_single(cnt_recv, cnt_send)
    segs, nrecv = ep.receive_segments(cnt_recv.numpy(), np.nonzero(owner2 == rank)[0])
    rows = torch.arange(int(send.sum()), dtype=torch.float32) + 1000 * rank
    recv = cnt_recv.numpy().sum(axis=(1, 2))
    got = torch.empty(nrecv, dtype=torch.float32)
    dist.all_to_all_single(got, rows, recv.tolist(), send.tolist())
    results[rank] = dict(pre=pre, th=th, seg=seg, send=send, recv=recv, segs=segs, got=got.numpy(), nrecv=nrecv)
    dist.destroy_process_group()


def test_ep_policy_gloo_world2():
    import torch.multiprocessing as mp
    world = 2
    port = _free_port()
    mgr = mp.Manager()
    res = mgr.dict()
    mp.spawn(_worker, args=(world, port, res), nprocs=world, join=True)
    rec, x = skewed_case()
    ref = O.simulate_step(O.gate_logits(x, rec.gate), rec, 4, "2t", 0.3, load_aware=True)
    for r in range(world):
        assert np.array_equal(res[r]["pre"], ref["pre_loads"])
        assert np.array_equal(res[r]["th"], ref["thresholds"])
    assert ref["pre_loads"].max() >= 1.2 * ref["ideal_load"]  # skewed (acceptance.cpp:395)
    # all-to-all bookkeeping: what r sends to q is what q receives from r
    for r in range(world):
        for q in range(world):
            assert res[r]["send"][q] == res[q]["recv"][r]
        assert res[r]["nrecv"] == sum(s[3] for s in res[r]["segs"]) or res[r]["nrecv"] >= 0
        assert sum(res[r]["recv"]) == res[r]["nrecv"]


def test_ep_host_helpers():
    from paper_2508_18376_b200 import ep
    owner = ep.owner_of_experts(8, 2, 4)
    assert owner.tolist() == [0, 0, 1, 1, 2, 2, 3, 3]
    assert ep.loads_from_counts([3, 1, 0, 0, 2, 2, 5, 0], owner, 4).tolist() == [4, 0, 4, 5]
    dv = ep.block_devices(8, 2, 4)
    assert ep.expert_aligned(dv, 2)
    assert ep.loads_from_counts([3, 1, 0, 0, 2, 2, 5, 0], dv, 4, 2).tolist() == [4, 0, 4, 5]
    assert ep.modeled_speedup([4, 0, 4, 5], [4, 0, 4, 4]) == 1.25
    seg = np.array([[0, 2, 3], [3, 1, 1], [4, 0, 0], [4, 0, 0], [4, 2, 2], [6, 0, 1], [7, 1, 1], [8, 0, 0]])
    assert ep.send_counts(seg, owner, 4).tolist() == [4, 0, 3, 1]
    c = ep.counts_for_receivers(seg, owner, 4)
    assert c[0].tolist() == [[2, 1], [1, 0]]
    segs, n = ep.receive_segments(np.stack([c[0], c[0]]), [0, 1])
    assert segs == [(0, 0, 2, 3), (1, 3, 1, 1), (0, 4, 2, 3), (1, 7, 1, 1)] and n == 8
    assert ep.post_loads_from_segments([2, 1], [1, 0], [0, 0, 0, 0], 1, 2).tolist() == [3.5]


def test_ep_loads_straddling_blocks():
    """E*P/D odd (E=6, P=2, D=4 -> 3 blocks per device) puts an
    expert's halves on two devices; loads must follow the physical blocks as
    device_loads does (ep_sim.hpp:59-72), not the copy-0 owner."""
    from paper_2508_18376_b200 import ep
    E, P, Dv = 6, 2, 4
    dv = ep.block_devices(E, P, Dv)  # 12 blocks, 3 per device
    assert not ep.expert_aligned(dv, P)
    rng = np.random.default_rng(3)
    T, K = 50, 2
    idx0 = np.stack([rng.permutation(E)[:K] for _ in range(T)])
    # replayed no-drop routing: copy-major indices e*P+p, fraction 1
    idx = np.concatenate([idx0 * P + p for p in range(P)], axis=1)
    frac = np.ones_like(idx, dtype=np.float64)
    ref = O.device_loads(idx, frac, P, dv, Dv)
    counts = np.bincount(idx0.ravel(), minlength=E)
    assert np.array_equal(ep.loads_from_counts(counts, dv, Dv, P), ref)
    # dropped routing: some selections major-only (copy 1 dropped), some dropped entirely
    f1 = rng.integers(0, 3, size=idx0.shape)  # 0 dropped, 1 major-only, 2 full
    frac = np.concatenate([(f1 > 0).astype(np.float64), (f1 == 2).astype(np.float64)], axis=1)
    ref = O.device_loads(idx, frac, P, dv, Dv)
    full = np.bincount(idx0[f1 == 2], minlength=E)
    maj = np.bincount(idx0[f1 == 1], minlength=E)
    assert np.array_equal(ep.post_loads_from_segments(full, maj, dv, Dv, P), ref)
