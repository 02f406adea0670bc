"""GPU, real multi-process expert parallelism: ExpertParallelMoE (ep.py; the
one-row-per-(token, rank) path `forward` and the per-selection `forward_rows`) with
world_size 2 and 3 — separate processes, each with its own token shard,
context and stream, exchanging counts, rows, scores and expert outputs through
torch.distributed (gloo: the ranks share the one GPU available here; on a
multi-GPU box the same code runs over NCCL).  The concatenated outputs and the
load / threshold reports must equal the oracle's simulate_step
(ep_sim.hpp:110-160) + moe_forward on all ranks' tokens."""
import os
import socket

import numpy as np
import pytest

import oracle as O

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


def skewed(T=420, E=12, K=2, d=128, ffn=192, seed=61):
    L = O.generate_layer(d, ffn, E, K, seed=seed)
    x = O.generate_tokens(T, d, seed + 1)
    x += (1.5 / np.linalg.norm(L.gate[:, 5])) * L.gate[:, 5]
    x = x.astype(np.float32)
    rec = O.reconstruct(L, O.profile_importance(L, x, O.route(L, x).idx, "abs_gate"))
    return rec, x


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, load_aware, method, q, strategy="contiguous", E=12, chunks=None):
    import torch.distributed as dist
    import paper_2508_18376_b200 as D
    from paper_2508_18376_b200 import ep
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    rec, x = skewed(E=E)
    layer = D.MoeLayer(rec.d, rec.ffn, rec.E, rec.K, rec.gate, rec.blocks, rec.shared, replay_factor=rec.P,
                       dtype="f32")
    shard = np.array_split(np.arange(x.shape[0]), world)[rank]
    m = ep.ExpertParallelMoE(layer, strategy=strategy, chunks=chunks)
    y, rep = getattr(m, method)(torch.from_numpy(x[shard]).cuda(), D.DropPolicy.two_t_from(0.3),
                                load_aware=load_aware, logits_mode=D.LOGITS_EXACT)
    q.put((rank, y.cpu().numpy(), rep["pre_loads"], rep["thresholds"], rep["post_loads"], rep["speedup"]))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("load_aware", [True, False])
@pytest.mark.parametrize("method", ["forward", "forward_rows"])
def test_ep_multiprocess_matches_simulate_step(world, load_aware, method):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, load_aware, method, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=300) for _ in range(world)], key=lambda t: t[0])
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    rec, x = skewed()
    ref = O.simulate_step(O.gate_logits(x, rec.gate), rec, world, "2t", 0.3, load_aware=load_aware)
    for _, _, pre, th, post, sp in res:
        assert np.array_equal(pre, ref["pre_loads"])
        assert np.array_equal(th, ref["thresholds"])
        assert np.array_equal(post, ref["post_loads"])
        assert sp == ref["speedup"]
    ro = O.route_from_logits(O.gate_logits(x, rec.gate), rec.K, rec.P)
    yo = O.moe_forward(rec, x, ref["idx"], ro.raw, ref["frac"])
    y = np.concatenate([r[1] for r in res])
    assert np.abs(y - yo).max() / np.abs(yo).max() < 1e-5


@pytest.mark.parametrize("chunks", [1, 3])
def test_ep_token_chunks(chunks):
    """The overlapped step (token chunks on their own streams) gives the same
    reports and outputs for any chunk count."""
    import torch.multiprocessing as mp
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, True, "forward", q, "contiguous", 12, chunks))
             for r in range(world)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=300) for _ in range(world)], key=lambda t: t[0])
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    rec, x = skewed()
    ref = O.simulate_step(O.gate_logits(x, rec.gate), rec, world, "2t", 0.3, load_aware=True)
    for _, _, pre, th, post, sp in res:
        assert np.array_equal(pre, ref["pre_loads"]) and np.array_equal(post, ref["post_loads"])
        assert np.array_equal(th, ref["thresholds"]) and sp == ref["speedup"]
    ro = O.route_from_logits(O.gate_logits(x, rec.gate), rec.K, rec.P)
    yo = O.moe_forward(rec, x, ref["idx"], ro.raw, ref["frac"])
    y = np.concatenate([r[1] for r in res])
    assert np.abs(y - yo).max() / np.abs(yo).max() < 1e-5


@pytest.mark.parametrize("strategy,world,E", [("round_robin", 2, 12), ("contiguous", 4, 6)])
def test_ep_sub_blocks_on_different_ranks(strategy, world, E):
    """S-ETP placement: round-robin puts block 2e on rank 0
    and its minor half 2e+1 on rank 1; contiguous with 3 blocks per rank
    splits every other expert's halves.  A full selection goes to both
    holders, each evaluating its half, a major-only one to block 0's rank;
    loads, thresholds and outputs still equal simulate_step + moe_forward."""
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, True, "forward", q, strategy, E)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=300) for _ in range(world)], key=lambda t: t[0])
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    rec, x = skewed(E=E)
    ref = O.simulate_step(O.gate_logits(x, rec.gate), rec, world, "2t", 0.3, load_aware=True,
                          round_robin=strategy == "round_robin")
    for _, _, pre, th, post, sp in res:
        assert np.array_equal(pre, ref["pre_loads"])
        assert np.array_equal(th, ref["thresholds"])
        assert np.array_equal(post, ref["post_loads"])
        assert sp == ref["speedup"]
    ro = O.route_from_logits(O.gate_logits(x, rec.gate), rec.K, rec.P)
    yo = O.moe_forward(rec, x, ref["idx"], ro.raw, ref["frac"])
    y = np.concatenate([r[1] for r in res])
    assert np.abs(y - yo).max() / np.abs(yo).max() < 1e-5


def _worker_bf16(rank, world, port, q):
    import torch.distributed as dist
    import paper_2508_18376_b200 as D
    from paper_2508_18376_b200 import ep
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    rec, x = _bf16_case()
    layer = D.MoeLayer(rec.d, rec.ffn, rec.E, rec.K, rec.gate, rec.blocks, rec.shared, replay_factor=rec.P,
                       dtype="bf16")
    shard = np.array_split(np.arange(x.shape[0]), world)[rank]
    m = ep.ExpertParallelMoE(layer)
    y, _ = m.forward(torch.from_numpy(x[shard]).cuda().bfloat16(), D.DropPolicy.two_t_from(0.25),
                     logits_mode=D.LOGITS_EXACT)
    q.put((rank, y.float().cpu().numpy()))
    dist.barrier()
    dist.destroy_process_group()


def _bf16_case():
    L = O.generate_layer(256, 192, 16, 4, S=1, seed=71)
    x = O.bf16_round(O.generate_tokens(333, 256, 72))
    rec = O.reconstruct(L, O.profile_importance(L, x, O.route(L, x).idx, "abs_gate")).round_bf16()
    return rec, x


def test_ep_multiprocess_bf16_shared_experts():
    """bf16 layer with a shared expert (computed once per token on its own rank)."""
    import torch.multiprocessing as mp
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker_bf16, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=300) for _ in range(world)], key=lambda t: t[0])
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    rec, x = _bf16_case()
    ref = O.simulate_step(O.gate_logits(x, rec.gate), rec, world, "2t", 0.25)
    ro = O.route_from_logits(O.gate_logits(x, rec.gate), rec.K, rec.P)
    yo = O.moe_forward(rec, x, ref["idx"], ro.raw, ref["frac"])
    y = np.concatenate([r[1] for r in res])
    assert np.abs(y - yo).max() / np.abs(yo).max() < 1e-2
