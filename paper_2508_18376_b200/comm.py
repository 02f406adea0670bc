"""ETP vs S-ETP expert communication.

DualSparse-MoE splits every expert into tp partial sub-experts
(partial_transform, /root/reference/proj/include/dsmoe/transform.hpp:100-131)
hosted by the tp ranks of the expert's EP group.  The reference only models
the two ways to move tokens to those hosts
(/root/reference/proj/src/comm_sim.cpp, include/dsmoe/comm_sim.hpp):

  ETP    all-to-all among the EP group leads, chain all-gather inside each TP
         group, chain reduce-scatter back, all-to-all back (4 collectives);
  S-ETP  one all-to-all over all ep x tp ranks straight to every partition
         host, one all-to-all back (2 collectives).

This module restates that model (`simulate_etp`, `simulate_setp`,
`compare_schemes`, `sweep_comm`, the scenario's xoshiro256++ routing) with the
reference's arithmetic, so its reports equal `dsmoe_sim_comm` field for field,
and adds the real thing: `CommBench` moves the scenario's payloads with the
collectives of each scheme over torch.distributed (NCCL on the GPUs of one
box; gloo point-to-point on CPU for the tests) and times them — the measured
counterpart of the model's `total_time`.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

_M64 = (1 << 64) - 1


# ------------------------------------------------------------------ routing
def _splitmix64(state):
    """SplitMix64::next (rng.hpp:19-24); returns (value, new state)."""
    state = (state + 0x9E3779B97F4A7C15) & _M64
    z = state
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & _M64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & _M64
    return z ^ (z >> 31), state


def _rotl(x, k):
    return ((x << k) | (x >> (64 - k))) & _M64


def xoshiro_u64(seed: int, n: int) -> list[int]:
    """First n outputs of Xoshiro256pp(seed).next_u64 (rng.hpp:30-47)."""
    st, sm = [], seed & _M64
    for _ in range(4):
        v, sm = _splitmix64(sm)
        st.append(v)
    out = []
    for _ in range(n):
        out.append((_rotl((st[0] + st[3]) & _M64, 23) + st[0]) & _M64)
        t = (st[1] << 17) & _M64
        st[2] ^= st[0]
        st[3] ^= st[1]
        st[1] ^= st[2]
        st[0] ^= st[3]
        st[2] ^= t
        st[3] = _rotl(st[3], 45)
    return out


# ----------------------------------------------------------------- scenario
@dataclass
class CommScenario:
    """CommScenario (comm_sim.hpp:14-43): ep_degree x tp_degree devices,
    id = group * tp + rank; token t lives on device t // tokens_per_device;
    experts map to EP groups in contiguous blocks."""

    ep_degree: int = 1
    tp_degree: int = 1
    tokens_per_device: int = 0
    bytes_per_token: int = 0
    alpha: float = 0.0
    beta: float = 1.0
    num_experts: int = 0
    routing: np.ndarray = field(default_factory=lambda: np.zeros(0, np.int64))

    @staticmethod
    def from_json(j: dict) -> "CommScenario":
        """scenario_from (/root/reference/proj/src/capi.cpp:114-132): routing
        = xoshiro256++(seed) % num_experts per token."""
        sc = CommScenario(int(j["ep"]), int(j["tp"]), int(j["tokens_per_device"]), int(j["bytes_per_token"]),
                          float(j["alpha"]), float(j["beta"]), int(j.get("num_experts", j["ep"])))
        seed = int(j.get("seed", 1))
        if sc.ep_degree < 1 or sc.tp_degree < 1 or sc.tokens_per_device < 1:
            raise ValueError("scenario: degrees and tokens_per_device must be >= 1")
        if sc.num_experts < 1:
            raise ValueError("scenario: num_experts must be >= 1")
        sc.routing = np.array([v % sc.num_experts for v in xoshiro_u64(seed, sc.total_tokens())], np.int64)
        sc.validate()
        return sc

    def devices(self) -> int:
        return self.ep_degree * self.tp_degree

    def total_tokens(self) -> int:
        return self.devices() * self.tokens_per_device

    def group_of_expert(self, e):
        return e // (self.num_experts // self.ep_degree)

    def validate(self):
        """CommScenario::validate (comm_sim.hpp:26-42)."""
        if not (self.ep_degree >= 1 and self.tp_degree >= 1):
            raise ValueError("comm scenario: degrees must be >= 1")
        if not (self.tokens_per_device >= 1 and self.bytes_per_token >= 1):
            raise ValueError("comm scenario: tokens and bytes per token must be >= 1")
        if not (self.alpha >= 0.0 and self.beta > 0.0):
            raise ValueError("comm scenario: alpha must be >= 0 and beta > 0")
        if not (self.num_experts >= self.ep_degree and self.num_experts % self.ep_degree == 0):
            raise ValueError("comm scenario: num_experts must be a positive multiple of ep_degree")
        if len(self.routing) != self.total_tokens():
            raise ValueError("comm scenario: routing must cover every token")
        if len(self.routing) and (self.routing.min() < 0 or self.routing.max() >= self.num_experts):
            raise ValueError("comm scenario: routed expert out of range")


# ------------------------------------------------------------------- phases
@dataclass
class CommPhase:
    kind: str
    participants: int
    link_bytes: np.ndarray          # devices x devices int64, diagonal zero
    max_link_bytes: int = 0
    max_device_bytes: int = 0
    time: float = 0.0


@dataclass
class CommReport:
    scheme: str
    phases: list = field(default_factory=list)
    launches: int = 0
    total_time: float = 0.0
    total_bytes: int = 0


def _make_phase(kind, participants, links, alpha, beta) -> CommPhase:
    """make_phase (comm_sim.cpp:22-41)."""
    ph = CommPhase(kind, participants, links)
    ph.max_link_bytes = int(links.max()) if links.size else 0
    out_b, in_b = links.sum(axis=1), links.sum(axis=0)
    ph.max_device_bytes = int(np.maximum(in_b, out_b).max()) if links.size else 0
    ph.time = alpha + float(ph.max_device_bytes) / beta
    return ph


def _finish(rep: CommReport) -> CommReport:
    """finish_report (comm_sim.cpp:43-51): sequential double sum of phase times."""
    for ph in rep.phases:
        rep.total_time += ph.time
        rep.total_bytes += int(ph.link_bytes.sum())
    rep.launches = len(rep.phases)
    return rep


def _add(links, src, dst, amount):
    """LinkMatrix::add (comm_sim.cpp:15-18), vectorised: local handoffs carry no bytes."""
    m = src != dst
    np.add.at(links, (src[m], dst[m]), amount)


def simulate_etp(sc: CommScenario) -> CommReport:
    """simulate_etp (comm_sim.cpp:55-109)."""
    sc.validate()
    tp, D = sc.tp_degree, sc.devices()
    t = np.arange(sc.total_tokens())
    src_group = (t // sc.tokens_per_device) // tp
    dst_group = sc.group_of_expert(sc.routing)
    rep = CommReport("etp")
    a2a = np.zeros((D, D), np.int64)
    _add(a2a, src_group * tp, dst_group * tp, sc.bytes_per_token)
    group_payload = np.bincount(dst_group, minlength=sc.ep_degree).astype(np.int64) * sc.bytes_per_token
    rep.phases.append(_make_phase("all_to_all", sc.ep_degree, a2a, sc.alpha, sc.beta))
    if tp > 1:
        ag = np.zeros((D, D), np.int64)
        rs = np.zeros((D, D), np.int64)
        for g in range(sc.ep_degree):
            for r in range(tp - 1):
                ag[g * tp + r, g * tp + r + 1] += group_payload[g]
            for r in range(tp - 1, 0, -1):
                rs[g * tp + r, g * tp + r - 1] += group_payload[g]
        rep.phases.append(_make_phase("all_gather", tp, ag, sc.alpha, sc.beta))
        rep.phases.append(_make_phase("reduce_scatter", tp, rs, sc.alpha, sc.beta))
    back = np.zeros((D, D), np.int64)
    _add(back, dst_group * tp, src_group * tp, sc.bytes_per_token)
    rep.phases.append(_make_phase("all_to_all", sc.ep_degree, back, sc.alpha, sc.beta))
    return _finish(rep)


def simulate_setp(sc: CommScenario) -> CommReport:
    """simulate_setp (comm_sim.cpp:111-138)."""
    sc.validate()
    tp, D = sc.tp_degree, sc.devices()
    t = np.arange(sc.total_tokens())
    src = t // sc.tokens_per_device
    dst_group = sc.group_of_expert(sc.routing)
    rep = CommReport("setp")
    a2a = np.zeros((D, D), np.int64)
    back = np.zeros((D, D), np.int64)
    for r in range(tp):
        _add(a2a, src, dst_group * tp + r, sc.bytes_per_token)
        _add(back, dst_group * tp + r, src, sc.bytes_per_token)
    rep.phases.append(_make_phase("all_to_all", D, a2a, sc.alpha, sc.beta))
    rep.phases.append(_make_phase("all_to_all", D, back, sc.alpha, sc.beta))
    return _finish(rep)


def compare_schemes(sc: CommScenario) -> dict:
    """compare_schemes (comm_sim.cpp:140-156)."""
    etp, setp = simulate_etp(sc), simulate_setp(sc)
    if not (etp.total_time > 0.0 and setp.total_time > 0.0):
        raise ValueError("compare_schemes: degenerate scenario with zero modeled time; use alpha > 0")
    inp = float(sc.tokens_per_device) * float(sc.bytes_per_token)
    eb, sb = inp / etp.total_time, inp / setp.total_time
    return {"etp_time": etp.total_time, "setp_time": setp.total_time, "etp_bandwidth": eb, "setp_bandwidth": sb,
            "improvement_pct": (sb - eb) / eb * 100.0, "etp_launches": etp.launches, "setp_launches": setp.launches}


def sweep_comm(sc: CommScenario, sizes) -> list[dict]:
    """sweep_comm (comm_sim.cpp:158-170)."""
    if len(sizes) == 0:
        raise ValueError("sweep_comm: empty size list")
    rows = []
    for s in sizes:
        if s < 1:
            raise ValueError("sweep_comm: sizes must be >= 1")
        sc.bytes_per_token = int(s)
        c = compare_schemes(sc)
        rows.append({"bytes": int(s), "etp_bw": c["etp_bandwidth"], "setp_bw": c["setp_bandwidth"],
                     "improvement_pct": c["improvement_pct"]})
    return rows


def report_json(rep: CommReport) -> dict:
    """The JSON shape of json_text(CommReport) (/root/reference/proj/src/reports.cpp:126-134)."""
    return {"scheme": rep.scheme, "launches": rep.launches, "total_time": rep.total_time,
            "total_bytes": rep.total_bytes,
            "phases": [{"kind": p.kind, "participants": p.participants, "max_link_bytes": p.max_link_bytes,
                        "max_device_bytes": p.max_device_bytes, "time": p.time,
                        "link_bytes": [int(v) for v in p.link_bytes.ravel()]} for p in rep.phases]}


# ------------------------------------------------------ real communication
class CommBench:
    """Moves one scenario's token payloads with each scheme's collectives.

    Rank d of the world (ep x tp ranks, d = group * tp + rank) sends the rows
    of its tokens_per_device tokens (bytes_per_token each, as bf16/uint8
    payload) exactly along the scenario's links:

      S-ETP  all_to_all_single over the world with per-destination splits =
             the model's a2a link bytes from d, then the reverse;
      ETP    lead-to-lead all_to_all_single (non-leads send and receive
             nothing), all_gather inside the TP group (group payload), a
             reduce_scatter of the partial results back (the model's chain
             phases as NCCL ring collectives), lead-to-lead return.

    With the NCCL backend the all-to-alls are `all_to_all_single`; with gloo
    (CPU tests) they are posted isend/irecv pairs.  `run` returns measured
    seconds per scheme (max over ranks) and the bytes every rank actually
    moved, which must equal the model's link_bytes rows.
    """

    def __init__(self, sc: CommScenario, group=None, device="cuda"):
        import torch.distributed as dist
        self.sc = sc
        self.dist = dist
        self.group = group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        if self.world != sc.devices():
            raise ValueError(f"comm bench: world {self.world} != ep x tp {sc.devices()}")
        self.nccl = dist.get_backend(group) == "nccl"
        self.device = device if self.nccl else "cpu"  # gloo point-to-point moves host tensors
        tp = sc.tp_degree
        g, r = divmod(self.rank, tp)
        self.tp_group = None
        if tp > 1:  # every rank must create every subgroup, in the same order
            for gg in range(sc.ep_degree):
                pg = dist.new_group(list(range(gg * tp, gg * tp + tp)))
                if gg == g:
                    self.tp_group = pg
        self.etp = simulate_etp(sc)
        self.setp = simulate_setp(sc)

    # -- primitive: all-to-all with explicit per-peer byte counts
    def _a2a(self, send_counts, recv_counts):
        import torch
        sc = self.sc
        dev = self.device
        sbuf = torch.empty(int(sum(send_counts)), dtype=torch.uint8, device=dev)
        rbuf = torch.empty(int(sum(recv_counts)), dtype=torch.uint8, device=dev)
        if self.nccl:
            self.dist.all_to_all_single(rbuf, sbuf, [int(v) for v in recv_counts], [int(v) for v in send_counts],
                                        group=self.group)
        else:
            reqs, so, ro = [], 0, 0
            for peer in range(self.world):
                if send_counts[peer] and peer != self.rank:
                    reqs.append(self.dist.isend(sbuf[so:so + send_counts[peer]], peer, group=self.group))
                if recv_counts[peer] and peer != self.rank:
                    reqs.append(self.dist.irecv(rbuf[ro:ro + recv_counts[peer]], peer, group=self.group))
                so += int(send_counts[peer])
                ro += int(recv_counts[peer])
            for q in reqs:
                q.wait()
        del sc
        return int(sum(send_counts[p] for p in range(self.world) if p != self.rank))

    def _phase_a2a(self, ph: CommPhase):
        D = self.world
        L = ph.link_bytes.reshape(D, D)
        return self._a2a(L[self.rank], L[:, self.rank])

    def _setp(self):
        sent = 0
        for ph in self.setp.phases:
            sent += self._phase_a2a(ph)
        return sent

    def _etp(self):
        import torch
        sc = self.sc
        tp = sc.tp_degree
        sent = self._phase_a2a(self.etp.phases[0])
        if tp > 1:
            g = self.rank // tp
            payload = int(np.bincount(sc.group_of_expert(sc.routing), minlength=sc.ep_degree)[g]) * sc.bytes_per_token
            chunk = max(1, -(-payload // tp))  # ring collectives move equal chunks
            buf = torch.empty(chunk * tp, dtype=torch.uint8, device=self.device)
            part = torch.empty(chunk, dtype=torch.uint8, device=self.device)
            if self.nccl:
                self.dist.all_gather_into_tensor(buf, part, group=self.tp_group)
                red = torch.empty(chunk * tp, dtype=torch.float16, device=self.device)
                outp = torch.empty(chunk, dtype=torch.float16, device=self.device)
                self.dist.reduce_scatter_tensor(outp, red, group=self.tp_group)
            else:
                parts = [torch.empty_like(part) for _ in range(tp)]
                self.dist.all_gather(parts, part, group=self.tp_group)
                red = torch.zeros(chunk, dtype=torch.float32, device=self.device)
                self.dist.all_reduce(red, group=self.tp_group)
            sent += 2 * chunk * (tp - 1)
        sent += self._phase_a2a(self.etp.phases[-1])
        return sent

    def run(self, iters=20, warmup=3):
        """Mean seconds per scheme (max over ranks) + bytes this rank sent."""
        import time
        import torch
        out = {}
        for name, fn in (("setp", self._setp), ("etp", self._etp)):
            for _ in range(warmup):
                fn()
            if self.nccl:
                torch.cuda.synchronize()
            self.dist.barrier(group=self.group)
            if self.nccl:
                s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                s.record()
                for _ in range(iters):
                    sent = fn()
                e.record()
                torch.cuda.synchronize()
                sec = s.elapsed_time(e) * 1e-3 / iters
            else:
                t0 = time.perf_counter()
                for _ in range(iters):
                    sent = fn()
                sec = (time.perf_counter() - t0) / iters
            t = torch.tensor([sec], dtype=torch.float64, device=self.device if self.nccl else "cpu")
            self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX, group=self.group)
            out[name] = {"seconds": float(t.item()), "bytes_sent": int(sent)}
        out["measured_speedup_setp_vs_etp"] = out["etp"]["seconds"] / out["setp"]["seconds"]
        out["model"] = compare_schemes(self.sc)
        return out
