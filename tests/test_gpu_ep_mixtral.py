"""GPU: expert parallelism at the benched Mixtral shape (BASELINE C5) — two
processes (gloo; they share the one GPU here, NCCL on a multi-GPU box), each
holding only its expert shard of the C3 layer exactly as bench.py builds it
(seeded weights, complete_transform P=4 on the device, device importance
profile + reconstruction: 32 experts of width 3584 as 1792-wide major /
minor halves, top-8, d=4096, bf16), skewed routing (acceptance.cpp:381-387),
load-aware 2T thresholds.  Loads, thresholds, post loads and the modeled
speed-up equal the reference simulate_step (ep_sim.hpp:110-160) on the
concatenated batch bit for bit; the outputs of every token match the
oracle's moe_forward within the bf16 scaled residual."""
import os
import socket

import numpy as np
import pytest

import oracle as O

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

T_RANK = 768
WORLD = 2


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _tokens(rank):
    import bench as B
    gate = B.make_weights("c3")[0]
    return B.bench_tokens("c3", T_RANK, rank=rank, skew=B.SKEW, gate=gate)


def _worker(rank, port, t_drop, load_aware, q):
    import torch.distributed as dist
    import bench as B
    import paper_2508_18376_b200 as D
    from paper_2508_18376_b200 import ep
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=WORLD)
    torch.cuda.set_device(0)
    ctx = D.Context()
    layer, _ = B.build_layer("c5", ctx)
    m = ep.ExpertParallelMoE(layer)
    assert m.layer.shard == tuple(range(32 * rank, 32 * rank + 32))  # this rank's 16 experts' 32 blocks
    del layer
    x = _tokens(rank).cuda()
    y, rep = m.forward(x, D.DropPolicy.two_t_from(t_drop), load_aware=load_aware, logits_mode=D.LOGITS_EXACT)
    q.put((rank, y.float().cpu().numpy(), rep["pre_loads"], rep["thresholds"], rep["post_loads"], rep["speedup"]))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("load_aware", [True])
def test_ep_mixtral_shape_two_ranks(load_aware):
    import torch.multiprocessing as mp
    import bench as B
    import paper_2508_18376_b200 as D
    torch.cuda.set_device(0)
    ctx = D.Context()
    info = {}
    rec, host = B.build_layer("c5", ctx, info=info)
    gate, experts, shared, E, K, ffn = host
    f = lambda t: t.float().cpu().numpy()
    L = O.Layer(gate.shape[0], ffn, E, K, f(gate), [tuple(f(w) for w in ex) for ex in experts], [])
    del experts, host
    Lr = O.reconstruct(L, info["values"].cpu().numpy())
    del L
    x = torch.cat([_tokens(r) for r in range(WORLD)])
    xh = x.float().numpy()
    lg = O.gate_logits(xh, Lr.gate)
    # uniform t for a ~25% global drop, as bench.py calibrates it
    pol, _ = B.calibrate(ctx, rec, x.cuda(), 0.25)
    del rec, info
    torch.cuda.empty_cache()
    ref = O.simulate_step(lg, Lr, WORLD, "2t", pol.t_drop, load_aware=load_aware)
    assert ref["pre_loads"].max() >= 1.2 * ref["ideal_load"]  # skewed (acceptance.cpp:395)
    mpc = mp.get_context("spawn")
    q = mpc.Queue()
    port = _free_port()
    procs = [mpc.Process(target=_worker, args=(r, port, pol.t_drop, load_aware, q)) for r in range(WORLD)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=900) for _ in range(WORLD)], key=lambda t: t[0])
    for p in procs:
        p.join(timeout=300)
        assert p.exitcode == 0
    for _, _, pre, th, post, sp in res:
        assert np.array_equal(pre, ref["pre_loads"])
        assert np.array_equal(th, ref["thresholds"])
        assert np.array_equal(post, ref["post_loads"])
        assert sp == ref["speedup"]
    y = np.concatenate([r[1] for r in res])
    ro = O.route_from_logits(lg, Lr.K, Lr.P)
    sel = np.arange(xh.shape[0])  # every token of both ranks
    yo = O.moe_forward(Lr, xh[sel], ref["idx"][sel], ro.raw[sel], ref["frac"][sel], threads=os.cpu_count() or 1)
    err = np.abs(y[sel] - yo).max() / max(np.abs(yo).max(), np.abs(y[sel]).max())
    assert err < 1e-2, err
