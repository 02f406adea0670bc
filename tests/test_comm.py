"""ETP vs S-ETP (comm.py): the model restated from comm_sim.cpp against the
reference's own dsmoe_sim_comm / dsmoe_sim_comm_sweep output
(tests/golden/comm_reference.json, tools/make_comm_golden.py), the
acceptance-test invariants (acceptance.cpp:540-700, test 10), and the real
payload movement over gloo (world 2 and 4, CPU)."""
import json
import os
import socket

import numpy as np
import pytest

from paper_2508_18376_b200 import comm

torch = pytest.importorskip("torch")
GOLD = os.path.join(os.path.dirname(__file__), "golden", "comm_reference.json")


def _cases():
    with open(GOLD) as f:
        return json.load(f)


@pytest.mark.parametrize("i", range(5))
def test_model_equals_reference(i):
    case = _cases()[i]
    sc = comm.CommScenario.from_json(case["scenario"])
    for name, fn in (("etp", comm.simulate_etp), ("setp", comm.simulate_setp)):
        assert comm.report_json(fn(sc)) == case["report"][name], name
    assert comm.compare_schemes(sc) == case["report"]["comparison"]
    rows = comm.sweep_comm(sc, case["sweep_sizes"])
    assert rows == case["sweep"]["rows"]


def test_launches_halved_and_payload_conservation():
    rng = np.random.default_rng(4)
    for ep, tp in ((2, 4), (4, 2), (9, 8)):
        for _ in range(5):
            sc = comm.CommScenario(ep, tp, 3, 64, 1e-6, 1e9, 2 * ep)
            sc.routing = rng.integers(0, sc.num_experts, sc.total_tokens())
            etp, setp = comm.simulate_etp(sc), comm.simulate_setp(sc)
            assert etp.launches == 2 * setp.launches if tp > 1 else etp.launches == setp.launches
            # every token reaches tp hosts in S-ETP: wire bytes = off-device deliveries
            src = np.arange(sc.total_tokens()) // sc.tokens_per_device
            grp = sc.group_of_expert(sc.routing)
            off = sum(int(((grp * tp + r) != src).sum()) for r in range(tp))
            assert int(setp.phases[0].link_bytes.sum()) == off * sc.bytes_per_token
            acc = 0.0  # sequential double sum (builtin sum() compensates since Python 3.12)
            for p in etp.phases:
                acc += p.time
            assert acc == etp.total_time


def test_full_swap_equal_bytes_favors_single_dispatch():
    sc = comm.CommScenario(2, 2, 8, 4096, 1e-6, 1e9, 2)
    t = np.arange(sc.total_tokens())
    sc.routing = np.where((t // sc.tokens_per_device) // sc.tp_degree == 0, 1, 0)
    etp, setp = comm.simulate_etp(sc), comm.simulate_setp(sc)
    for ph in etp.phases + setp.phases:
        assert ph.max_device_bytes == 16 * sc.bytes_per_token
    assert setp.total_time < etp.total_time


def test_improvement_decays_with_payload():
    for ep, tp, tpd, E, seed in ((2, 4, 16, 4, 909), (9, 8, 2, 18, 910)):
        sc = comm.CommScenario(ep, tp, tpd, 1024, 1e-5, 1e9, E)
        sc.routing = np.array([v % E for v in comm.xoshiro_u64(seed, sc.total_tokens())])
        rows = comm.sweep_comm(sc, [512, 2048, 8192, 32768, 131072])
        imp = [r["improvement_pct"] for r in rows]
        assert all(b < a for a, b in zip(imp, imp[1:]))


def test_invalid_scenarios_rejected():
    with pytest.raises(ValueError):
        comm.CommScenario.from_json({"ep": 0, "tp": 2, "tokens_per_device": 4, "bytes_per_token": 8, "alpha": 0,
                                     "beta": 1})
    sc = comm.CommScenario(2, 1, 2, 8, 0.0, 1.0, 3)
    sc.routing = np.zeros(4, np.int64)
    with pytest.raises(ValueError):
        sc.validate()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, ep, tp, q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    sc = comm.CommScenario.from_json({"ep": ep, "tp": tp, "tokens_per_device": 6, "bytes_per_token": 256,
                                      "alpha": 1e-6, "beta": 1e9, "num_experts": 2 * ep, "seed": 5})
    b = comm.CommBench(sc, device="cpu")
    res = b.run(iters=2, warmup=1)
    D = sc.devices()
    want = sum(int(ph.link_bytes.reshape(D, D)[rank].sum()) for ph in b.setp.phases)
    q.put((rank, res["setp"]["bytes_sent"], want, res["etp"]["seconds"] > 0))
    dist.destroy_process_group()


@pytest.mark.parametrize("ep,tp", [(2, 1), (1, 2), (2, 2)])
def test_commbench_moves_model_payloads_gloo(ep, tp):
    import torch.multiprocessing as mp
    world = ep * tp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, ep, tp, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, sent, want, ok in out:
        assert sent == want, rank
        assert ok
