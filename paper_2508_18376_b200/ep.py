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
    """One rank of an expert-parallel MoE layer.  With shard=True (default)
    the rank keeps only the weights of the physical blocks the placement puts
    on it (dsmoe_b200_layer_shard_blocks: the gate and the shared experts are
    whole) and evaluates only them."""

    def __init__(self, layer: D.MoeLayer, group=None, strategy: str = "contiguous", shard: bool = True,
                 chunks: int | None = None):
        import torch
        import torch.distributed as dist
        self.dist = dist
        self.group = group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        W, P = self.world, layer.P
        # Placement::device_of of the physical blocks (ep_sim.hpp:38-54): any
        # placement, including ones that put an expert's sub-blocks on
        # different ranks (S-ETP; contiguous with E*P/W odd)
        self.device_of = block_devices(layer.E, P, W, strategy)
        self.aligned = expert_aligned(self.device_of, P)
        self.owner = owner_of_experts(layer.E, P, W, strategy)  # threshold owner: block 0's device
        self.held = (self.device_of == self.rank).astype(np.uint8)
        self.local = np.nonzero(self.owner == self.rank)[0]
        dv = self.device_of.reshape(-1, P)
        dest = np.zeros((layer.E, 2), np.int64)
        for p in range(P):
            dest[:, 0] |= 1 << dv[:, p]       # a full selection: every rank holding one of its blocks
        dest[:, 1] = 1 << dv[:, 0]             # a major-only selection: the rank holding block 0
        self.ctx = D.Context()
        self.ctx_exp = D.Context()
        self.full = layer
        if shard and W > 1:
            layer = D.layer_shard_blocks(self.ctx, layer, self.held)
        self.layer = layer
        self.coll = _Coll(dist, group)
        dev = torch.device("cuda", torch.cuda.current_device())
        self.d_device_of = torch.from_numpy(self.device_of.astype(np.int32)).to(dev)
        self.d_dest = torch.from_numpy(dest.astype(np.uint32).view(np.int32)).to(dev)
        self._bufs = {}
        self._chunks = []
        # token chunks per step: the dispatch all-to-all of chunk c+1 overlaps
        # the expert GEMMs of chunk c (one chunk when there is nothing to overlap)
        self.chunks = chunks if chunks is not None else (2 if W > 1 else 1)

    def _buf(self, name, shape, dtype, dev):
        import torch
        b = self._bufs.get(name)
        if b is None or b.shape != shape or b.dtype != dtype:
            b = torch.empty(shape, dtype=dtype, device=dev)
            self._bufs[name] = b
        return b

    def _chunk_state(self, c):
        import torch
        while len(self._chunks) <= c:
            st = torch.cuda.Stream()
            self._chunks.append({"stream": st, "ctx": D.Context(stream=st), "ctx_exp": D.Context(stream=st),
                                 "host": torch.empty(4 * self.world, dtype=torch.int64).pin_memory(),
                                 "ev": torch.cuda.Event()})
        return self._chunks[c]

    def forward(self, x, policy: D.DropPolicy | None = None, load_aware=True, logits_mode=D.LOGITS_TENSOR,
                timing=False, stats=True, chunks=None):
        """One EP step with one host synchronisation point (the split sizes):
        1. no-drop routing of the whole batch -> per-expert counts ->
           all-reduce (device);
        2. device_loads -> thresholds -> owner table on the device
           (simulate_step, ep_sim.hpp:110-149);
        then per token chunk, each on its own stream and contexts:
        3. re-route the chunk under the owner thresholds from the step-1
           logits, pack one row per (token, destination rank) + one record per
           (kept selection, destination), local shared experts
           (dsmoe_b200_ep_dispatch);
        4. all-to-all of the per-destination counts, copied to pinned host
           memory; the host waits for all chunks' counts once;
        5. all-to-all of rows and records; this rank's experts (one output
           row per received row); rows back; summed per token over ranks +
           shared experts.
        The collectives are issued chunk-interleaved (rows of every chunk,
        then experts, then the returns), so on the one NCCL stream chunk c+1's
        dispatch all-to-all overlaps chunk c's expert GEMMs and chunk c's
        return overlaps chunk c+1's.  stats=True adds the post-drop load report
        (one all-reduce + sync)."""
        import torch
        L, W, ctx = self.layer, self.world, self.ctx
        policy = policy or D.DropPolicy()
        T = x.shape[0]
        dev = x.device
        drop = policy.kind != "none"
        nch = max(1, min(self.chunks if chunks is None else int(chunks), T))
        main = torch.cuda.current_stream()
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)] if timing else None
        if timing:
            ev[0].record(main)
        counts = D.ep_route_counts(ctx, L, x, policy, self._buf("counts", (L.E, 2), torch.int64, dev), logits_mode)
        counts = self.coll.all_reduce(counts)
        t_unit, loads = D.ep_thresholds(ctx, L, counts, W, self.d_device_of, policy.t_drop if drop else 1.0,
                                        load_aware and drop, self._buf("t_unit", (L.E,), torch.float64, dev),
                                        self._buf("loads", (W,), torch.float64, dev))
        lg, ld, _ = D.ctx_logits(ctx)
        ready = torch.cuda.Event()
        ready.record(main)
        out = torch.empty((T, L.d), dtype=x.dtype, device=dev)
        bounds = np.linspace(0, T, nch + 1).astype(np.int64)
        ch = []
        for c in range(nch):  # 3-4: dispatch + count exchange, all chunks
            c0, c1 = int(bounds[c]), int(bounds[c + 1])
            st = self._chunk_state(c)
            Tc = c1 - c0
            with torch.cuda.stream(st["stream"]):
                st["stream"].wait_event(ready)
                send = self._buf(f"send{c}", (Tc * min(W, L.K * L.P) + 1, L.d), x.dtype, dev)
                rec = self._buf(f"rec{c}", (Tc * L.K * min(W, L.P) + 1, 3), torch.int32, dev)
                cnt = self._buf(f"cnt{c}", (2, W, 2), torch.int64, dev)
                D.ep_dispatch(st["ctx"], L, x[c0:c1], policy, t_unit if drop else None, W, self.d_dest, send, rec,
                              cnt[0], logits=(lg + c0 * ld * 4, ld))
                self.coll.all_to_all(cnt[1], cnt[0], [1] * W, [1] * W)
                st["host"].copy_(cnt.view(-1), non_blocking=True)
                st["ev"].record(st["stream"])
            ch.append({"c0": c0, "c1": c1, "T": Tc, "st": st, "send": send, "rec": rec})
        for k in ch:  # the host synchronisation point: split sizes of every chunk
            k["st"]["ev"].synchronize()
            h = k["st"]["host"].numpy()
            k["nu"], k["ns"] = h[0:2 * W:2].copy(), h[1:2 * W:2].copy()
            k["ru"], k["rs"] = h[2 * W:4 * W:2].copy(), h[2 * W + 1:4 * W:2].copy()
            k["U"], k["S"], k["NU"], k["NS"] = (int(k["ru"].sum()), int(k["rs"].sum()), int(k["nu"].sum()),
                                                int(k["ns"].sum()))
        tev = []
        for c, k in enumerate(ch):  # 5: rows and records, every chunk
            with torch.cuda.stream(k["st"]["stream"]):
                k["xr"] = self._buf(f"xr{c}", (max(k["U"], 1) + 1, L.d), x.dtype, dev)
                k["rr"] = self._buf(f"rr{c}", (max(k["S"], 1) + 1, 3), torch.int32, dev)
                e = [torch.cuda.Event(enable_timing=True) for _ in range(4)] if timing else None
                if timing:
                    e[0].record()
                self.coll.all_to_all(k["xr"][:k["U"]], k["send"][:k["NU"]], k["ru"].tolist(), k["nu"].tolist())
                self.coll.all_to_all(k["rr"][:k["S"]], k["rec"][:k["NS"]], k["rs"].tolist(), k["ns"].tolist())
                if timing:
                    e[1].record()
                tev.append(e)
        for c, k in enumerate(ch):  # this rank's experts
            with torch.cuda.stream(k["st"]["stream"]):
                k["yl"] = D.ep_expert_packed(k["st"]["ctx_exp"], L, k["xr"], k["U"], k["rr"], k["S"],
                                             np.concatenate([[0], np.cumsum(k["ru"])]),
                                             np.concatenate([[0], np.cumsum(k["rs"])]),
                                             out=self._buf(f"yl{c}", (max(k["U"], 1) + 1, L.d), x.dtype, dev))
                if timing:
                    tev[c][2].record()
        for c, k in enumerate(ch):  # rows back, combine into this chunk's output rows
            with torch.cuda.stream(k["st"]["stream"]):
                ret = self._buf(f"ret{c}", (k["NU"] + 1, L.d), x.dtype, dev)
                self.coll.all_to_all(ret[:k["NU"]], k["yl"][:k["U"]], k["nu"].tolist(), k["ru"].tolist())
                if timing:
                    tev[c][3].record()
                D.ep_combine(k["st"]["ctx"], L, ret, k["T"], out=out[k["c0"]:k["c1"]])
                if stats or timing:  # this chunk's kept (full, major-only) selections per expert
                    D.ep_last_counts(k["st"]["ctx"], L, k["T"], self._buf(f"post{c}", (L.E, 2), torch.int64, dev))
        for k in ch:
            main.wait_stream(k["st"]["stream"])
        if timing:
            ev[1].record(main)
        sm = lambda key: np.sum([k[key] for k in ch], axis=0)
        rep = {"rows_sent": sm("nu"), "rows_received": int(sm("U")), "records_sent": sm("ns"),
               "records_received": int(sm("S")), "chunks": nch}
        if stats or timing:
            post = self._bufs["post0"].clone()
            for c in range(1, nch):
                post += self._bufs[f"post{c}"]
            post = self.coll.all_reduce(post).cpu().numpy()
            pre = loads.cpu().numpy()
            rep["pre_loads"] = pre
            rep["thresholds"] = device_thresholds(pre, policy.t_drop, load_aware) if drop else np.zeros(W)
            rep["post_loads"] = post_loads_from_segments(post[:, 0], post[:, 1], self.device_of, W, L.P)
            rep["speedup"] = modeled_speedup(pre, rep["post_loads"])
        if timing:
            torch.cuda.synchronize()
            rep["exchange_ms"] = float(sum(e[0].elapsed_time(e[1]) + e[2].elapsed_time(e[3]) for e in tev))
            rep["expert_ms"] = float(sum(e[1].elapsed_time(e[2]) for e in tev))
            rep["step_ms"] = ev[0].elapsed_time(ev[1])
            # this rank's expert FLOPs: 6 d x (the widths of the blocks it holds that each record needs)
            bw = np.asarray(self.full.widths()[0], np.float64).reshape(-1, L.P) * self.held.reshape(-1, L.P)
            fl, nbytes = 0.0, 0
            for k in ch:
                codes = k["rr"][:k["S"], 0].cpu().numpy()
                unit, full = codes >> 2, (codes & 3) == 2
                fl += float(6.0 * L.d * np.where(full, bw.sum(axis=1)[unit], bw[unit, 0]).sum())
                nbytes += int((k["NU"] + k["U"]) * L.d * x.element_size() + (k["NS"] + k["S"]) * 12)
            rep["expert_flops"] = fl
            rep["exchange_bytes"] = nbytes  # this rank: sent + received, both directions
        return out, rep

    def forward_rows(self, x, policy: D.DropPolicy | None = None, load_aware=True, logits_mode=D.LOGITS_TENSOR,
                     timing=False, stats=True):
        """The first EP data path: one row per kept SELECTION both ways (more
        bytes; kept for comparison).  stats=False skips the post-drop load
        report (one all-reduce + host sync)."""
        import torch
        if not self.aligned:
            raise D.DsmoeError(1, "forward_rows: the per-selection path needs expert-aligned placement")
        dist, L = self.dist, self.full
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
