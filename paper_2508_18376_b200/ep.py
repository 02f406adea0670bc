"""Expert parallelism across the GPUs of one box (north-star item 6).

The reference only simulates EP (/root/reference/proj/include/dsmoe/ep_sim.hpp):
it places physical expert blocks on devices (place_experts :38), measures
per-device loads in compute units (device_loads :59), derives load-aware
per-device thresholds (load_aware_thresholds :76) and applies each selection's
owner-device threshold (simulate_step :110-160), reporting
speedup = max(pre load) / max(post load).  Here the same policy drives a real
data path, one process per GPU over torch.distributed (NCCL):

  1. every rank routes its own tokens without drop and the per-expert
     selection counts are all-reduced (integers, so every rank derives the
     bit-identical loads the reference's device_loads would give on the
     concatenation of all ranks' tokens);
  2. loads -> thresholds (uniform or load-aware) -> per-expert owner
     threshold table t_unit; the device router re-routes with it
     (dsmoe_b200_dispatch) and gathers the kept rows, experts ascending, so
     under contiguous placement each destination rank's rows are one run;
  3. per-expert (full, major-only) row counts and then the rows + raw scores
     travel with all_to_all_single (dispatch);
  4. each rank runs the grouped SwiGLU FFN over the received segments
     (dsmoe_b200_expert_ffn), major-only rows skipping the minor sub-block;
  5. the expert outputs travel back with the reverse all_to_all_single and
     are combined in slot order (dsmoe_b200_combine).

The host-side policy arithmetic (owner table, loads, thresholds, splits,
receive segments) is plain numpy below and is unit-tested with gloo on CPU.
EpEmulator runs the same data path for D virtual ranks on one GPU (the
all-to-alls become slices), which is how the path is checked against the
oracle here, where only one GPU is available.
"""
from __future__ import annotations

import numpy as np

from . import dsmoe as D


# --------------------------------------------------------------- host policy
def block_devices(num_experts: int, replay_factor: int, devices: int, strategy: str = "contiguous"):
    """Placement::device_of (ep_sim.hpp:38-54): the device of every physical
    block e*P + p."""
    return D.place_experts(num_experts * replay_factor, devices, strategy)


def owner_of_experts(num_experts: int, replay_factor: int, devices: int, strategy: str = "contiguous"):
    """Device whose threshold an original expert's selections use = the device
    of its copy-0 (whole or major) block (ep_sim.hpp:139-141)."""
    return block_devices(num_experts, replay_factor, devices, strategy)[np.arange(num_experts) * replay_factor]


def expert_aligned(device_of, replay_factor: int) -> bool:
    """True when every expert's P blocks sit on one device (the data path
    then moves whole selections; contiguous placement with E*P/D a multiple
    of P, ep_sim.hpp:48-52)."""
    dv = np.asarray(device_of).reshape(-1, replay_factor)
    return bool((dv == dv[:, :1]).all())


def loads_from_counts(counts, device_of, devices, replay_factor: int = 1):
    """device_loads (ep_sim.hpp:59-72) of a no-drop routing from per-expert
    selection counts: each selection adds fraction/P = 1/P to the device of
    each of its P blocks.  P is a power of two in every caller, so each
    partial sum is an exact multiple of 1/P and the double sums do not
    depend on their order.  `device_of` has E*P entries (block devices)."""
    P = int(replay_factor)
    dv = np.asarray(device_of).reshape(-1, P)
    c = np.asarray(counts, np.float64)
    loads = np.zeros(devices, np.float64)
    for p in range(P):
        np.add.at(loads, dv[:, p], c * (1.0 / P))
    return loads


def post_loads_from_segments(seg_full, seg_major, device_of, devices, replay_factor):
    """device_loads of the dropped routing from per-expert (full, major-only)
    kept-selection counts: a full selection keeps every copy (1/P each), a
    major-only one copy 0 only — fraction 1.0 at weight 1/P for P > 1, or
    fraction 0.5 for P = 1 (dropping.hpp:105-116).  Exact for P a power of two."""
    P = int(replay_factor)
    dv = np.asarray(device_of).reshape(-1, P)
    full = np.asarray(seg_full, np.float64)
    maj = np.asarray(seg_major, np.float64)
    loads = np.zeros(devices, np.float64)
    if P == 1:
        np.add.at(loads, dv[:, 0], full + 0.5 * maj)
        return loads
    w = 1.0 / P
    np.add.at(loads, dv[:, 0], (full + maj) * w)
    for p in range(1, P):
        np.add.at(loads, dv[:, p], full * w)
    return loads


def device_thresholds(loads, t_drop, load_aware):
    """simulate_step (ep_sim.hpp:133-138): load-aware or uniform thresholds."""
    if load_aware:
        return D.load_aware_thresholds(loads, t_drop)
    return np.full(len(loads), float(t_drop))


def send_counts(seg, owner, devices):
    """Rows this rank sends to each rank: the kept rows of the experts it owns."""
    out = np.zeros(devices, np.int64)
    np.add.at(out, np.asarray(owner), np.asarray(seg)[:, 2].astype(np.int64))
    return out


def counts_for_receivers(seg, owner, devices):
    """(devices x n_local x 2) int32: for each destination rank, (full rows,
    major-only rows) of each expert it owns, in expert order."""
    owner = np.asarray(owner)
    n_local = np.bincount(owner, minlength=devices).max()
    out = np.zeros((devices, n_local, 2), np.int32)
    for r in range(devices):
        es = np.nonzero(owner == r)[0]
        out[r, :len(es), 0] = seg[es, 1]
        out[r, :len(es), 1] = seg[es, 2] - seg[es, 1]
    return out


def receive_segments(cnt_recv, local_experts):
    """Segments of the receive buffer: source-rank major, then expert, each
    (unit, start, n_full, n_tot) — the order the sources' runs arrive in."""
    segs, start = [], 0
    for src in range(cnt_recv.shape[0]):
        for j, e in enumerate(local_experts):
            nf, nm = int(cnt_recv[src, j, 0]), int(cnt_recv[src, j, 1])
            if nf + nm:
                segs.append((int(e), start, nf, nf + nm))
            start += nf + nm
    return segs, start


def modeled_speedup(pre, post):
    """EpReport::speedup (ep_sim.hpp:154-158)."""
    mp, mq = float(np.max(pre)), float(np.max(post))
    return mp / mq if mq > 0 else (float("inf") if mp > 0 else 1.0)


# ------------------------------------------------------------ distributed
class _Coll:
    """The three collectives the EP step needs.  NCCL: native on device
    tensors.  Any other backend (gloo — the multi-process tests, several
    ranks sharing one GPU): host copies, all-to-all as posted isend/irecv."""

    def __init__(self, dist, group):
        self.dist, self.group = dist, group
        self.nccl = dist.get_backend(group) == "nccl"
        self.rank, self.world = dist.get_rank(group), dist.get_world_size(group)

    def all_reduce(self, t):
        if self.nccl:
            self.dist.all_reduce(t, group=self.group)
            return t
        h = t.cpu()
        self.dist.all_reduce(h, group=self.group)
        return h.to(t.device)

    def all_to_all(self, out, inp, out_splits, in_splits):
        """out/inp: first-dim splits (rows) per peer, as in all_to_all_single."""
        if self.nccl:
            self.dist.all_to_all_single(out, inp, out_splits, in_splits, group=self.group)
            return
        hi, ho = inp.contiguous().cpu(), out.cpu()
        reqs, keep, so, ro = [], [], 0, 0
        for peer in range(self.world):
            ns, nr = int(in_splits[peer]), int(out_splits[peer])
            if peer == self.rank:
                ho[ro:ro + nr] = hi[so:so + ns]
            else:
                if ns:
                    keep.append(hi[so:so + ns])
                    reqs.append(self.dist.isend(keep[-1], peer, group=self.group))
                if nr:  # first-dim slices of a contiguous tensor: irecv writes in place
                    reqs.append(self.dist.irecv(ho[ro:ro + nr], peer, group=self.group))
            so += ns
            ro += nr
        for q in reqs:
            q.wait()
        out.copy_(ho.to(out.device))


class ExpertParallelMoE:
    """One rank of an expert-parallel MoE layer.  Every rank holds the full
    (replicated) layer object but evaluates only the experts it owns."""

    def __init__(self, layer: D.MoeLayer, group=None, strategy: str = "contiguous"):
        import torch.distributed as dist
        self.dist = dist
        self.group = group
        self.layer = layer
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        if strategy != "contiguous":
            raise D.DsmoeError(1, "expert-parallel data path needs contiguous placement")
        self.device_of = block_devices(layer.E, layer.P, self.world, strategy)
        if not expert_aligned(self.device_of, layer.P):
            raise D.DsmoeError(1, "expert-parallel data path: an expert's sub-blocks straddle two ranks "
                                  "(contiguous placement needs E*P/world to be a multiple of P)")
        self.owner = owner_of_experts(layer.E, layer.P, self.world, strategy)
        self.local = np.nonzero(self.owner == self.rank)[0]
        self.ctx = D.Context()
        self.ctx_exp = D.Context()
        self.coll = _Coll(dist, group)

    def forward(self, x, policy: D.DropPolicy | None = None, load_aware=True, logits_mode=D.LOGITS_TENSOR,
                timing=False, stats=True):
        """One EP step moving one row per (token, rank) (dsmoe_b200_ep_pack /
        _ep_expert / _ep_combine): a token goes once to each rank that owns
        one of its kept selections, with one record per selection; the rank
        returns one row per token (its experts' weighted sum).  stats=False
        skips the post-drop load report (an all-reduce + host sync)."""
        import torch
        L, W = self.layer, self.world
        policy = policy or D.DropPolicy()
        T = x.shape[0]
        dev = x.device
        # 1. global pre-drop loads -> thresholds (simulate_step, ep_sim.hpp:110-138)
        seg0, _, _ = D.dispatch(self.ctx, L, x, D.DropPolicy(), logits_mode=logits_mode)
        counts = self.coll.all_reduce(torch.from_numpy(seg0[:, 2].astype(np.int64)).to(dev))
        pre = loads_from_counts(counts.cpu().numpy(), self.device_of, W, L.P)
        t_unit, th = None, np.zeros(W)
        if policy.kind != "none":
            th = device_thresholds(pre, policy.t_drop, load_aware)
            t_unit = torch.from_numpy(th[self.owner]).to(dev)
        # 2. re-route under the owner thresholds (logits of step 1); shared experts run here
        seg, _, st = D.dispatch(self.ctx, L, x, policy, t_unit=t_unit, logits_mode=D.LOGITS_REUSE, with_stats=stats)
        # 3. one row per (token, destination) + one record per kept selection
        cap_rows = T * min(W, L.K) + 1
        send = torch.empty((cap_rows, L.d), dtype=x.dtype, device=dev)
        rc = torch.empty(T * L.K + 1, dtype=torch.int32, device=dev)
        rr = torch.empty_like(rc)
        rw = torch.empty(T * L.K + 1, dtype=torch.float32, device=dev)
        nu, ns = D.ep_pack(self.ctx, L, x, W, self.owner, send, rc, rr, rw)
        # 4. counts, then rows and records
        cnt = torch.from_numpy(np.stack([nu, ns], axis=1)).to(dev)
        cnt_recv = torch.empty_like(cnt)
        self.coll.all_to_all(cnt_recv, cnt, [1] * W, [1] * W)
        cr = cnt_recv.cpu().numpy()
        ru, rs = cr[:, 0], cr[:, 1]
        U, S = int(ru.sum()), int(rs.sum())
        xr = torch.empty((U + 1, L.d), dtype=x.dtype, device=dev)
        rcr = torch.empty(S + 1, dtype=torch.int32, device=dev)
        rrr = torch.empty_like(rcr)
        rwr = torch.empty(S + 1, dtype=torch.float32, device=dev)
        self.coll.all_to_all(xr[:U], send[:int(nu.sum())], ru.tolist(), nu.tolist())
        for dst, src in ((rcr, rc), (rrr, rr), (rwr, rw)):
            self.coll.all_to_all(dst[:S], src[:int(ns.sum())], rs.tolist(), ns.tolist())
        # 5. this rank's experts, one output row per received row
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)] if timing else None
        if timing:
            ev[0].record()
        yl = D.ep_expert(self.ctx_exp, L, xr, U, rcr, rrr, rwr, S, np.concatenate([[0], np.cumsum(ru)]),
                         np.concatenate([[0], np.cumsum(rs)]))
        if timing:
            ev[1].record()
        # 6. rows back in send order, summed per token over ranks (+ shared experts)
        ret = torch.empty((int(nu.sum()) + 1, L.d), dtype=x.dtype, device=dev)
        self.coll.all_to_all(ret[:int(nu.sum())], yl[:U], nu.tolist(), ru.tolist())
        out = D.ep_combine(self.ctx, L, ret, T)
        rep = {"pre_loads": pre, "thresholds": th, "rows_sent": nu, "rows_received": U, "records_sent": ns}
        if stats:
            post = torch.from_numpy(np.stack([seg[:, 1], seg[:, 2] - seg[:, 1]]).astype(np.int64)).to(dev)
            post = self.coll.all_reduce(post).cpu().numpy()
            rep["post_loads"] = post_loads_from_segments(post[0], post[1], self.device_of, W, L.P)
            rep["speedup"] = modeled_speedup(pre, rep["post_loads"])
            rep["local_drop_stats"] = st
        if timing:
            torch.cuda.synchronize()
            rep["expert_ms"] = ev[0].elapsed_time(ev[1])
        return out, rep

    def forward_rows(self, x, policy: D.DropPolicy | None = None, load_aware=True, logits_mode=D.LOGITS_TENSOR,
                     timing=False, stats=True):
        """The first EP data path: one row per kept SELECTION both ways (more
        bytes; kept for comparison).  stats=False skips the post-drop load
        report (one all-reduce + host sync)."""
        import torch
        dist, L = self.dist, self.layer
        policy = policy or D.DropPolicy()
        T = x.shape[0]
        dev = x.device
        # 1. global pre-drop loads
        seg0, _, _ = D.dispatch(self.ctx, L, x, D.DropPolicy(), logits_mode=logits_mode)
        counts = torch.from_numpy(seg0[:, 2].astype(np.int64)).to(dev)
        counts = self.coll.all_reduce(counts)
        pre = loads_from_counts(counts.cpu().numpy(), self.device_of, self.world, L.P)
        t_unit, th = None, np.zeros(self.world)
        if policy.kind != "none":
            th = device_thresholds(pre, policy.t_drop, load_aware)
            t_unit = torch.from_numpy(th[self.owner]).to(dev)
        # 2. owner-threshold routing + gather
        xp = torch.empty((T * L.K + 128, L.d), dtype=x.dtype, device=dev)
        sp = torch.empty(T * L.K + 128, dtype=torch.float32, device=dev)
        # same batch, new thresholds: re-route from the logits step 1 left on this context
        seg, R, st = D.dispatch(self.ctx, L, x, policy, t_unit=t_unit, rows_out=xp, scale_out=sp,
                                logits_mode=D.LOGITS_REUSE, with_stats=stats)
        send = send_counts(seg, self.owner, self.world)
        # 3. exchange counts, then rows and scores
        cnt_send = torch.from_numpy(counts_for_receivers(seg, self.owner, self.world)).to(dev)
        cnt_recv = torch.empty_like(cnt_send)
        self.coll.all_to_all(cnt_recv, cnt_send, [1] * self.world, [1] * self.world)
        cnt_recv = cnt_recv.cpu().numpy()
        segs, nrecv = receive_segments(cnt_recv, self.local)
        recv = cnt_recv.sum(axis=(1, 2)).astype(np.int64)
        xr = torch.empty((nrecv + 128, L.d), dtype=x.dtype, device=dev)
        sr = torch.empty(nrecv + 128, dtype=torch.float32, device=dev)
        self.coll.all_to_all(xr[:nrecv], xp[:R], recv.tolist(), send.tolist())
        self.coll.all_to_all(sr[:nrecv], sp[:R], recv.tolist(), send.tolist())
        # 4. local experts
        yr = torch.empty_like(xr)
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)] if timing else None
        if timing:
            ev[0].record()
        if segs:
            D.expert_ffn(self.ctx_exp, L, xr, sr, segs, y_out=yr)
        if timing:
            ev[1].record()
        # 5. return + combine
        yb = torch.empty((R + 128, L.d), dtype=x.dtype, device=dev)
        self.coll.all_to_all(yb[:R], yr[:nrecv], send.tolist(), recv.tolist())
        out = D.combine(self.ctx, L, yb, T)
        if not stats:
            rep = {"pre_loads": pre, "thresholds": th, "rows_sent": send, "rows_received": int(nrecv)}
            if timing:
                torch.cuda.synchronize()
                rep["expert_ms"] = ev[0].elapsed_time(ev[1])
            return out, rep
        post = torch.from_numpy(np.stack([seg[:, 1], seg[:, 2] - seg[:, 1]]).astype(np.int64)).to(dev)
        post = self.coll.all_reduce(post)
        post = post.cpu().numpy()
        post_loads = post_loads_from_segments(post[0], post[1], self.device_of, self.world, L.P)
        rep = {"pre_loads": pre, "post_loads": post_loads, "thresholds": th, "speedup": modeled_speedup(pre, post_loads),
               "local_drop_stats": st, "rows_sent": send, "rows_received": int(nrecv)}
        if timing:
            torch.cuda.synchronize()
            rep["expert_ms"] = ev[0].elapsed_time(ev[1])
        return out, rep


# ---------------------------------------------------------------- emulator
class EpEmulator:
    """The expert-parallel data path for `devices` virtual ranks on one GPU:
    per-rank contexts, real kernels, the all-to-alls as slice/concat copies.
    Used to check the path against the oracle and to time each rank's expert
    FFN under uniform vs load-aware thresholds."""

    def __init__(self, layer: D.MoeLayer, devices: int):
        self.layer = layer
        self.D = devices
        self.device_of = block_devices(layer.E, layer.P, devices)
        if not expert_aligned(self.device_of, layer.P):
            raise D.DsmoeError(1, "EpEmulator: an expert's sub-blocks straddle two devices")
        self.owner = owner_of_experts(layer.E, layer.P, devices)
        self.ctx = [D.Context() for _ in range(devices)]
        self.ctx_exp = [D.Context() for _ in range(devices)]

    def forward(self, xs, policy: D.DropPolicy | None = None, load_aware=True, logits_mode=D.LOGITS_TENSOR,
                timing=False):
        import torch
        L, Dv = self.layer, self.D
        policy = policy or D.DropPolicy()
        counts = np.zeros(L.E, np.int64)
        for r in range(Dv):
            seg0, _, _ = D.dispatch(self.ctx[r], L, xs[r], D.DropPolicy(), logits_mode=logits_mode)
            counts += seg0[:, 2]
        pre = loads_from_counts(counts, self.device_of, Dv, L.P)
        t_unit, th = None, np.zeros(Dv)
        if policy.kind != "none":
            th = device_thresholds(pre, policy.t_drop, load_aware)
            t_unit = torch.from_numpy(th[self.owner]).cuda()
        xp, sp, seg, R, send = [], [], [], [], []
        for r in range(Dv):
            T = xs[r].shape[0]
            a = torch.empty((T * L.K + 128, L.d), dtype=xs[r].dtype, device="cuda")
            b = torch.empty(T * L.K + 128, dtype=torch.float32, device="cuda")
            sg, n, _ = D.dispatch(self.ctx[r], L, xs[r], policy, t_unit=t_unit, rows_out=a, scale_out=b,
                                  logits_mode=D.LOGITS_REUSE)
            xp.append(a), sp.append(b), seg.append(sg), R.append(n)
            send.append(send_counts(sg, self.owner, Dv))
        cnt = [counts_for_receivers(seg[r], self.owner, Dv) for r in range(Dv)]
        offs = [np.concatenate([[0], np.cumsum(send[r])]) for r in range(Dv)]
        ys_back = [torch.empty((R[r] + 128, L.d), dtype=xs[r].dtype, device="cuda") for r in range(Dv)]
        expert_ms = []
        for dst in range(Dv):
            cnt_recv = np.stack([cnt[src][dst] for src in range(Dv)])
            segs, nrecv = receive_segments(cnt_recv, np.nonzero(self.owner == dst)[0])
            xr = torch.empty((nrecv + 128, L.d), dtype=xs[0].dtype, device="cuda")
            sr = torch.empty(nrecv + 128, dtype=torch.float32, device="cuda")
            pos = 0
            for src in range(Dv):  # all-to-all: src's run for dst
                a, b = offs[src][dst], offs[src][dst + 1]
                xr[pos:pos + b - a] = xp[src][a:b]
                sr[pos:pos + b - a] = sp[src][a:b]
                pos += b - a
            yr = torch.empty_like(xr)
            if timing:
                torch.cuda.synchronize()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
            if segs:
                D.expert_ffn(self.ctx_exp[dst], L, xr, sr, segs, y_out=yr)
            if timing:
                e1.record()
                torch.cuda.synchronize()
                expert_ms.append(e0.elapsed_time(e1))
            pos = 0
            for src in range(Dv):  # reverse all-to-all
                a, b = offs[src][dst], offs[src][dst + 1]
                ys_back[src][a:b] = yr[pos:pos + b - a]
                pos += b - a
        outs = [D.combine(self.ctx[r], L, ys_back[r], xs[r].shape[0]) for r in range(Dv)]
        full = np.zeros(L.E, np.int64)
        maj = np.zeros(L.E, np.int64)
        for r in range(Dv):
            full += seg[r][:, 1]
            maj += seg[r][:, 2] - seg[r][:, 1]
        post = post_loads_from_segments(full, maj, self.device_of, Dv, L.P)
        rep = {"pre_loads": pre, "post_loads": post, "thresholds": th, "speedup": modeled_speedup(pre, post)}
        if timing:
            rep["expert_ms"] = expert_ms
        return outs, rep
