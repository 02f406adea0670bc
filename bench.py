"""MoE-module forward throughput on B200 (BASELINE.json metric: "MoE-module
tokens/s vs drop rate (0/25/50%) at 1/2/4/8 B200; EP speedup").

    python bench.py [--gpus N --steps K --warmup W] [--config c2|c3|c4|c5] [--drop 0.25]
    python bench.py --impl reference ...      (the reference's CPU path, host cores)

A step is one MoE-module forward (gate -> route/drop -> permute -> grouped
SwiGLU GEMMs -> combine) over T synthetic tokens already resident in HBM.
Default workload at N = 1: BASELINE config C2 (OLMoE-1B-7B layer: 64 experts,
top-8, d=2048, ffn=1024, reconstructed into major/minor halves, bf16,
T=16384).  `value` is at the --drop target (2T policy, threshold calibrated on
the device); the 0/25/50% sweep and its speed-ups over 0% ride at the end of
the line.  Weights are random-init of the named shapes (no checkpoints
offline), drawn on the host from a seeded torch CPU generator so the
reference arm (`--impl reference`) runs the very same layer.
N > 1 (torchrun, one process per GPU): default config C5 = the Mixtral layer
(C3) under expert parallelism with skewed synthetic routing
(acceptance.cpp:381-387), load-aware vs uniform thresholds (ep.py).
Prints ONE compact JSON line on rank 0; the full record goes to
gpurun_out/bench_detail_<config>_n<N>.json.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    # name: (d, ffn, E, K, S, workload label)
    "c2": (2048, 1024, 64, 8, 0, "OLMoE-1B-7B MoE layer (64 experts, top-8, d=2048, ffn=1024), reconstructed P=2"),
    "c3": (4096, 14336, 8, 2, 0, "Mixtral-8x7B MoE layer (8 experts, top-2, d=4096, ffn=14336), complete P=4 "
                                 "(32 experts, top-8, ffn 3584) then reconstructed P=2"),
    "c4": (2048, 1408, 64, 6, 2, "DeepSeek-V2-Lite MoE layer (64 routed + 2 shared, top-6, d=2048, ffn=1408), "
                                 "reconstructed P=2"),
}
CONFIGS["c5"] = CONFIGS["c3"][:5] + ("Mixtral-8x7B MoE layer (C3: complete P=4, reconstructed P=2) under "
                                      "expert parallelism, skewed synthetic routing",)
# calibration tokens for the offline importance profile (both arms, same
# tokens): the reference's profile_importance runs ~0.2 GFLOP/s on one core,
# so the set is sized for its arm to finish in well under a minute
CALIB = {"c2": 128, "c3": 32, "c4": 128, "c5": 32}
SKEW = 1.5  # acceptance.cpp:381-387: x += (1.5 / |W_g[:,hot]|) W_g[:,hot]
HOT = 3
METRIC = "MoE-module tokens/s vs drop rate (0/25/50%) at 1/2/4/8 B200; EP speedup"
PROFILE_EVERY = 8  # headline loop: stage events on every 8th step


def base_cfg(cfg):
    return "c3" if cfg == "c5" else cfg


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return d.get("bf16_tflops", 1625.1), d.get("bf16_tflops_sustained", 1384.5), d.get("hbm_gbs", 6530.0), \
            "MEASURED_PEAKS.json"
    # fallback: /opt/skills/guides/B200_PROFILING.md
    return 2250.0, 2250.0, 7700.0, "B200_PROFILING.md fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed regions."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index=0):
        self.index = index
        self.samples = []
        self._stop = threading.Event()
        self._t = None

    def _nvml(self):
        """NVML directly (microseconds per query, so the sampler keeps up with
        a sub-second timed region); None when unavailable."""
        try:
            import pynvml as N
            N.nvmlInit()
            h = N.nvmlDeviceGetHandleByIndex(self.index)
            mx = N.nvmlDeviceGetMaxClockInfo(h, N.NVML_CLOCK_SM)
            bits = {"hw_slowdown": N.nvmlClocksEventReasonHwSlowdown,
                    "hw_thermal_slowdown": N.nvmlClocksEventReasonHwThermalSlowdown,
                    "sw_thermal_slowdown": N.nvmlClocksEventReasonSwThermalSlowdown,
                    "sw_power_cap": N.nvmlClocksEventReasonSwPowerCap}

            def q():
                sm = N.nvmlDeviceGetClockInfo(h, N.NVML_CLOCK_SM)
                r = N.nvmlDeviceGetCurrentClocksEventReasons(h)
                return [str(sm), str(mx), hex(r)] + ["Active" if r & b else "Not Active" for b in bits.values()]
            q()
            return q
        except Exception:
            return None

    def _run(self):
        q = self._nvml()
        while not self._stop.is_set():
            try:
                if q is not None:
                    self.samples.append(q())
                else:
                    out = subprocess.run(["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits"], capture_output=True, text=True,
                                         timeout=5).stdout.strip()
                    if out:
                        self.samples.append([v.strip() for v in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.005 if q is not None else 0.02)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({n for s in self.samples for n, v in zip(names, s[3:7]) if v.strip() == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": float(self.samples[0][1]) if self.samples[0][1].replace(".", "").isdigit() else None,
                "reasons": reasons, "samples": len(self.samples)}


# ------------------------------------------------------------------ layers
def make_weights(cfg, seed=0):
    """Random-init weights of the named shapes in the reference layout (gate
    d x E, w1/w3 d x ffn, w2 ffn x d), N(0, 1/d) rounded to bf16, drawn on the
    host from a seeded CPU generator (identical in both bench arms)."""
    import torch
    d, ffn, E, K, S, _ = CONFIGS[cfg]
    g = torch.Generator().manual_seed(seed)
    sd = d ** -0.5

    def rnd(*s):
        return (torch.randn(*s, generator=g) * sd).to(torch.bfloat16)

    gate = rnd(d, E)
    experts = [(rnd(d, ffn), rnd(d, ffn), rnd(ffn, d)) for _ in range(E)]
    shared = [(rnd(d, ffn), rnd(d, ffn), rnd(ffn, d)) for _ in range(S)]
    return gate, experts, shared


def calib_tokens(cfg, n):
    import torch
    d = CONFIGS[cfg][0]
    return torch.randn(n, d, generator=torch.Generator().manual_seed(98)).to(torch.bfloat16)


def bench_tokens(cfg, T, rank=0, skew=0.0, gate=None):
    """The timed batch: N(0,1) tokens (seed 99 + rank), optionally biased toward
    expert HOT (acceptance.cpp:381-387) for the skewed-routing EP configs."""
    import torch
    d = CONFIGS[cfg][0]
    x = torch.randn(T, d, generator=torch.Generator().manual_seed(99 + rank))
    if skew:
        hot = gate.float().cpu()[:, HOT]
        x = x + (skew / hot.norm()) * hot
    return x.to(torch.bfloat16)


def build_layer(cfg, ctx, calib=None, seed=0, info=None):
    """Base layer -> (C3/C5: complete P=4 on the device) -> device importance
    profile on the calibration tokens -> device reconstruction into
    major/minor (P=2).  Returns (reconstructed MoeLayer, host) with host =
    (gate, experts, shared, E, K, ffn) of the (transformed) base layer as host
    bf16 tensors; `info` (dict, optional) receives the calibration set,
    importance values, neuron order and offline timings."""
    import torch
    import paper_2508_18376_b200 as D
    bc = base_cfg(cfg)
    d, ffn, E, K, S, _ = CONFIGS[bc]
    gate, experts, shared = make_weights(bc, seed)
    base = D.MoeLayer(d, ffn, E, K, gate, experts, shared, dtype="bf16")
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    if bc == "c3":
        base = D.transform(ctx, base, "complete", 4)  # complete_transform (transform.hpp:66-95) on the device
        E, K, ffn = base.E, base.K, base.ffn
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    n_cal = calib if calib is not None else CALIB[cfg]
    xc = calib_tokens(bc, n_cal).cuda()
    r = D.route_and_drop(ctx, base, xc)
    vals = D.profile_importance(ctx, base, xc, r.indices, "abs_gate")
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    rec, order = D.reconstruct_experts(ctx, base, vals)
    torch.cuda.synchronize()
    t3 = time.perf_counter()
    if bc == "c3":
        tg, tex, tsh = D.layer_weights(ctx, base)  # the transformed layer, read back from the device
        host = (tg, tex, tsh, E, K, ffn)
    else:
        host = (gate, experts, shared, E, K, ffn)
    if info is not None:
        info.update(calib=xc, values=vals, order=order, base=base,
                    offline={"calib_tokens": n_cal, "metric": "abs_gate", "transform_ms": (t1 - t0) * 1e3,
                             "profile_ms": (t2 - t1) * 1e3, "reconstruct_ms": (t3 - t2) * 1e3})
    return rec, host


def calibrate(ctx, layer, x, target, tol=0.005, kind="2t", t_unit=None):
    """Threshold bisection to a target drop rate (acceptance.cpp:342-352 method).
    kind "2t": band (t-0.01, t+0.01), minor halves drop first; "1t": whole
    selections below t drop (drop_1t, dropping.hpp:133)."""
    import paper_2508_18376_b200 as D
    if target <= 0:
        return D.DropPolicy(), 0.0
    if t_unit is None:  # the same bisection in one device kernel (dsmoe_b200_calibrate_rate): the same t
        return D.calibrate_rate(ctx, layer, x, target, kind=kind, tol=tol)
    mk = D.DropPolicy.two_t_from if kind == "2t" else D.DropPolicy.one_t
    lo, hi = 0.0, 1.0
    best = None
    for _ in range(40):
        t = 0.5 * (lo + hi)
        st = D.route_and_drop(ctx, layer, x, mk(t), t_unit=t_unit).stats
        if best is None or abs(st["drop_rate"] - target) < abs(best[1] - target):
            best = (t, st["drop_rate"])
        if abs(st["drop_rate"] - target) <= tol:
            break
        if st["drop_rate"] < target:
            lo = t
        else:
            hi = t
    return mk(best[0]), best[1]


# ---------------------------------------------------------------- timing
def time_steps(fn, steps, warmup, dist=None):
    import torch
    for _ in range(warmup):
        fn()
    torch.cuda.synchronize()
    if dist is not None:
        dist.barrier()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(steps):
        fn()
    e.record()
    torch.cuda.synchronize()
    ms = s.elapsed_time(e)
    if dist is not None:
        t = torch.tensor([ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dist.barrier()
        ms = float(t.item())
    return ms


# ------------------------------------------------------- the reference path
def ref_layer(cfg, calib=None):
    """The reference's own offline pipeline on the same weights and
    calibration tokens: (C3: complete_transform) -> route_tokens ->
    profile_importance -> reconstruct_experts (oracle/_ref: the reference
    compiled from /root/reference/proj).  Returns (RefLayer, E, K, ffn)."""
    import numpy as np
    import oracle as O
    bc = base_cfg(cfg)
    d, ffn, E, K, S, _ = CONFIGS[bc]
    if not O.ref_available():
        raise RuntimeError("oracle/_ref not built (the reference compiled from /root/reference/proj)")
    gate, experts, shared = make_weights(bc)
    f = lambda t: t.float().numpy()
    R = O.RefLayer.from_layer(O.Layer(d, ffn, E, K, f(gate), [tuple(f(w) for w in ex) for ex in experts],
                                      [tuple(f(w) for w in s) for s in shared]))
    del gate, experts, shared
    if bc == "c3":
        R = R.transform(True, 4)
        E, K, ffn = E * 4, K * 4, ffn // 4
    xc = np.ascontiguousarray(f(calib_tokens(bc, calib if calib is not None else CALIB[cfg])))
    r = R.route_and_drop(xc, K, 1)
    vals = R.profile_importance(xc, r.idx, E, ffn, "abs_gate")
    rec, _ = R.reconstruct(vals, E, ffn, "abs_gate")
    return rec, E, K, ffn


def ref_calibrate(R, x, K, target, tol=0.005):
    """The reference's route_and_drop (2T band t -/+ 0.01) bisected to the
    target drop rate on a routing sample (acceptance.cpp:342-352)."""
    if target <= 0:
        return 0.0, 0.0
    lo, hi, best = 0.0, 1.0, None
    for _ in range(40):
        t = 0.5 * (lo + hi)
        r = R.route_and_drop(x, K, 2, "2t", t)
        rate = R.drop_stats(x.shape[0], r.pre_frac, r.frac)["drop_rate"]
        if best is None or abs(rate - target) < abs(best[1] - target):
            best = (t, rate)
        if abs(rate - target) <= tol:
            break
        lo, hi = (t, hi) if rate < target else (lo, t)
    return best


def ref_rate(R, x, K, t, threads):
    """One reference step on the sample: route_and_drop + moe_forward (the
    forward over `threads` host threads on contiguous token shards — pure and
    per-token separable, moe.hpp:253-269, bit-identical to one call)."""
    t0 = time.perf_counter()
    if t > 0:
        r = R.route_and_drop(x, K, 2, "2t", t)
    else:
        r = R.route_and_drop(x, K, 2)
    R.moe_forward(x, r.idx, r.raw, r.frac, threads=threads)
    dt = time.perf_counter() - t0
    return x.shape[0] / dt, dt, r


def run_reference(args, world):
    """--impl reference: the reference's CPU path on this box's host cores, on
    the same reconstructed layer (same weights, same calibration tokens, the
    reference's own profile / reconstruct) at the same 2T drop target."""
    import numpy as np
    cfg = args.config
    d, ffn, E, K, S, label = CONFIGS[cfg]
    ncores = os.cpu_count() or 1
    t_setup = time.perf_counter()
    R, E, K, ffn = ref_layer(cfg)
    bc = base_cfg(cfg)
    skew = SKEW if cfg == "c5" else 0.0
    gate = make_weights(bc)[0] if skew else None
    xs = np.ascontiguousarray(bench_tokens(bc, 1024, skew=skew, gate=gate).float().numpy())
    t_drop, rate = ref_calibrate(R, xs, K, args.drop)
    sample = args.cpu_sample or {"c2": 256, "c3": 8, "c4": 256, "c5": 8}[cfg]
    x = np.ascontiguousarray(xs[:sample])
    setup_s = time.perf_counter() - t_setup
    ref_rate(R, x[:max(2, sample // 4)], K, t_drop, ncores)  # warm-up
    for _ in range(max(0, args.warmup - 1)):
        ref_rate(R, x, K, t_drop, ncores)
    rates, rr = [], None
    for _ in range(args.steps):
        v, _, rr = ref_rate(R, x, K, t_drop, ncores)
        rates.append(v)
    v = statistics.median(rates)
    samp = (f"{sample} tokens/step of the benchmark batch (N(0,1), seed 99), route_and_drop + moe_forward "
            f"over {ncores} threads, median of {args.steps} steps")
    line = {"metric": METRIC, "value": v, "unit": "tokens/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": sample / v * 1e3, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f32", "data": "synthetic tokens N(0,1), random-init weights of the named "
            "shapes (seeded, identical to the GPU arm)", "impl": "reference",
            "config": {"workload": label, "config_id": cfg, "drop_target": args.drop, "drop_rate": round(rate, 4),
                       "drop_rate_sample": round(R.drop_stats(sample, np.ones_like(rr.frac), rr.frac)["drop_rate"], 4),
                       "policy": "2T (t-0.01, t+0.01)", "t_drop": t_drop,
                       "calib_tokens": CALIB[cfg], "reconstruction": "reference profile_importance(abs_gate) + "
                       "reconstruct_experts on the calibration tokens", "tokens_per_step": sample,
                       "setup_s": round(setup_s, 1)},
            "cpu_baseline": {"value": v, "unit": "tokens/s", "cores": ncores, "kind": "reference", "sample": samp},
            "e2e": {"value": v, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line))


# ------------------------------------------------------------------ e2e
def e2e_pipelined(D, ctx_stream, ctx, layer, pol, x, steps):
    """Same metric through the public API with HOST buffers: per step the
    token batch is copied H2D from pinned memory and the MoE output D2H to
    pinned memory.  Copies run on their own streams, double-buffered, so the
    copy of step i+1 / i-1 overlaps the forward of step i."""
    import torch
    T, d = x.shape
    xh = [x.cpu().pin_memory() for _ in range(2)]
    oh = [torch.empty_like(xh[0]).pin_memory() for _ in range(2)]
    xd = [torch.empty_like(x) for _ in range(2)]
    od = [torch.empty_like(x) for _ in range(2)]
    s_in, s_out = torch.cuda.Stream(), torch.cuda.Stream()
    ev_in = [torch.cuda.Event() for _ in range(2)]
    ev_fw = [torch.cuda.Event() for _ in range(2)]
    ev_out = [torch.cuda.Event() for _ in range(2)]
    for e in ev_out:
        e.record(s_out)

    def run(n):
        for i in range(n):
            b = i & 1
            with torch.cuda.stream(s_in):
                s_in.wait_event(ev_fw[b]) if i >= 2 else None
                xd[b].copy_(xh[b], non_blocking=True)
                ev_in[b].record(s_in)
            ctx_stream.wait_event(ev_in[b])
            ctx_stream.wait_event(ev_out[b])
            D.forward(ctx, layer, xd[b], pol, out=od[b])
            ev_fw[b].record(ctx_stream)
            with torch.cuda.stream(s_out):
                s_out.wait_event(ev_fw[b])
                oh[b].copy_(od[b], non_blocking=True)
                ev_out[b].record(s_out)

    run(3)
    torch.cuda.synchronize()
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    t0.record(ctx_stream)
    run(steps)
    s_out.synchronize()
    t1.record(s_out)
    torch.cuda.synchronize()
    ms = t0.elapsed_time(t1) / steps
    return {"value": T / (ms * 1e-3), "unit": "tokens/s", "ms_per_step": ms,
            "h2d_bytes_per_step": xh[0].numel() * xh[0].element_size(),
            "d2h_bytes_per_step": oh[0].numel() * oh[0].element_size(),
            "mode": "double-buffered H2D / forward / D2H on separate streams"}


def ep_emulated(D, cfg="c2", devices=8, tokens_per_rank=4096, target=0.25, skew=1.5):
    """EP data path for `devices` virtual ranks on one GPU (ep.EpEmulator):
    skewed synthetic routing (acceptance.cpp:381-387), contiguous placement.
    Step time of EP = the slowest rank's expert FFN (the all-to-alls are
    copies here); compares no drop, uniform thresholds and load-aware
    thresholds, uniform matched to load-aware's global drop rate."""
    import torch
    from paper_2508_18376_b200 import ep
    ctx = D.Context()
    layer, host = build_layer(cfg, ctx)
    hot = host[0].float().cpu()[:, HOT]
    d = hot.shape[0]
    g = torch.Generator().manual_seed(7)
    xs = []
    for r in range(devices):
        x = torch.randn(tokens_per_rank, d, generator=g)
        x = x + (skew / hot.norm()) * hot
        xs.append(x.to(torch.bfloat16).cuda())
    emu = ep.EpEmulator(layer, devices)
    xall = torch.cat(xs)
    pol_u, rate_u = calibrate(ctx, layer, xall, target)
    seg0, _, _ = D.dispatch(ctx, layer, xall, D.DropPolicy())
    pre = ep.loads_from_counts(seg0[:, 2], emu.device_of, devices, layer.P)

    def aware_rate(t):
        th = ep.device_thresholds(pre, t, True)
        t_unit = torch.from_numpy(th[emu.owner]).cuda()
        return D.route_and_drop(ctx, layer, xall, D.DropPolicy.two_t_from(t), t_unit=t_unit).stats["drop_rate"]

    lo, hi, best = 0.0, 1.0, None
    for _ in range(30):
        t = 0.5 * (lo + hi)
        r = aware_rate(t)
        if best is None or abs(r - rate_u) < abs(best[1] - rate_u):
            best = (t, r)
        if abs(r - rate_u) < 0.002:
            break
        lo, hi = (t, hi) if r < rate_u else (lo, t)
    pol_a, rate_a = D.DropPolicy.two_t_from(best[0]), best[1]

    def run(policy, aware):
        best = None
        for _ in range(3):
            _, rep = emu.forward(xs, policy, load_aware=aware, timing=True)
            m = max(rep["expert_ms"])
            if best is None or m < best[0]:
                best = (m, rep)
        return best

    none = run(D.DropPolicy(), False)
    uni = run(pol_u, False)
    aware = run(pol_a, True)
    return {"devices": devices, "tokens_per_rank": tokens_per_rank, "skew": skew,
            "drop_rate": {"uniform": round(rate_u, 4), "load_aware": round(rate_a, 4)},
            "max_rank_expert_ms": {"no_drop": none[0], "uniform": uni[0], "load_aware": aware[0]},
            "pre_loads": none[1]["pre_loads"].tolist(), "post_loads_load_aware": aware[1]["post_loads"].tolist(),
            "modeled_speedup_load_aware": aware[1]["speedup"],
            "speedup_load_aware_vs_no_drop": none[0] / aware[0],
            "speedup_uniform_vs_no_drop": none[0] / uni[0],
            "speedup_load_aware_vs_uniform_matched_rate": uni[0] / aware[0]}


def detail_path(cfg, n):
    out = os.path.join(ROOT, "gpurun_out")
    os.makedirs(out, exist_ok=True)
    return os.path.join(out, f"bench_detail_{cfg}_n{n}.json")


def r4(v):
    return None if v is None else float(f"{v:.4g}")


# ------------------------------------------------------------------ main
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default=None, choices=list(CONFIGS),
                    help="default: c2 at N=1, c5 (Mixtral EP, skewed routing) at N>1")
    ap.add_argument("--drop", type=float, default=0.25)
    ap.add_argument("--tokens", type=int, default=16384)
    ap.add_argument("--cpu-sample", type=int, default=0, help="tokens for the CPU baseline sample (0 = auto)")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-ep", action="store_true", help="skip the single-GPU EP emulation")
    ap.add_argument("--ep", action="store_true", help="run the NCCL expert-parallel path even at N=1")
    ap.add_argument("--extra", default="c3,c4", help="comma list of extra configs to sweep (default c3,c4; '' for none)")
    args = ap.parse_args()

    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local = int(os.environ.get("LOCAL_RANK", 0))
    use_ep = world > 1 or args.ep
    if args.config is None:
        args.config = "c5" if use_ep else "c2"

    if args.impl == "reference":
        if rank != 0:
            return
        run_reference(args, world)
        return

    import torch
    import torch.distributed as dist
    # one process per GPU; DSMOE_B200_EP_BACKEND=gloo (smoke tests of the N > 1
    # path with several ranks sharing one GPU) maps ranks onto the visible GPUs
    torch.cuda.set_device(local % max(1, torch.cuda.device_count()))
    if use_ep:
        if "MASTER_ADDR" not in os.environ:  # --ep without torchrun: a 1-rank group
            import socket
            sk = socket.socket()
            sk.bind(("127.0.0.1", 0))
            os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(sk.getsockname()[1]), RANK="0",
                              WORLD_SIZE="1")
            sk.close()
        dist.init_process_group(os.environ.get("DSMOE_B200_EP_BACKEND", "nccl"))
        run_ep(args, dist, rank, world, local)
        dist.destroy_process_group()
        return
    run_single(args, local)


def run_ep(args, dist, rank, world, local):
    """N > 1: expert parallelism over NCCL (ep.py)."""
    import numpy as np
    import torch
    import paper_2508_18376_b200 as D
    from paper_2508_18376_b200 import ep
    cfg = args.config
    bc = base_cfg(cfg)
    d, ffn, E, K, S, label = CONFIGS[cfg]
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    ctx = D.Context(stream)
    info = {}
    layer, host = build_layer(cfg, ctx, info=info)
    T = args.tokens
    skew = SKEW if cfg == "c5" else 0.0
    x = bench_tokens(bc, T, rank=rank, skew=skew, gate=host[0]).cuda()
    peak_burst, peak_sust, hbm, peak_src = load_peaks()
    m = ep.ExpertParallelMoE(layer)
    # uniform threshold for the drop target on the union of all ranks' tokens
    xall = [torch.empty_like(x) for _ in range(world)]
    dist.all_gather(xall, x)
    pol, rate_main = calibrate(ctx, layer, torch.cat(xall), args.drop)
    del xall
    res = {}
    with ClockSampler(local) as clk:
        for name, p_, aware in (("no_drop", D.DropPolicy(), False), ("uniform", pol, False),
                                ("load_aware", pol, True)):
            res[name] = time_steps(lambda: m.forward(x, p_, load_aware=aware, stats=False), args.steps,
                                   max(3, args.warmup), dist) / args.steps
    l0 = D.total_launch_count()
    _, rep = m.forward(x, pol, load_aware=True, timing=True)
    launches_per_step = D.total_launch_count() - l0
    ms_step = res["load_aware"]
    # S-ETP placement: round-robin blocks put the major and
    # minor halves of an expert on different ranks; a full selection then
    # travels to both (measured next to the contiguous placement)
    setp = None
    if world > 1:
        try:
            m_rr = ep.ExpertParallelMoE(layer, strategy="round_robin")
            ms_rr = time_steps(lambda: m_rr.forward(x, pol, load_aware=True, stats=False), args.steps,
                               max(3, args.warmup), dist) / args.steps
            _, rep_rr = m_rr.forward(x, pol, load_aware=True, timing=True)
            setp = {"placement": "round_robin (halves of an expert on different ranks)", "ms_per_step": r4(ms_rr),
                    "speedup_vs_contiguous": r4(ms_step / ms_rr), "modeled_speedup": r4(rep_rr["speedup"]),
                    "exchange_bytes_rank0": rep_rr.get("exchange_bytes")}
            del m_rr
        except Exception as e:  # noqa: BLE001 — the line must still print
            setp = {"error": str(e)}
    # e2e through the public API with host buffers
    xh = x.cpu().pin_memory()
    oh = torch.empty_like(xh).pin_memory()
    xd = torch.empty_like(x)

    def e2e_step():
        xd.copy_(xh, non_blocking=True)
        y, _ = m.forward(xd, pol, load_aware=True, stats=False)
        oh.copy_(y, non_blocking=True)
    n_e2e = max(5, args.steps // 2)
    ms_e2e = time_steps(e2e_step, n_e2e, 2, dist) / n_e2e
    # roofline of the expert side: the slowest rank's grouped-GEMM FLOPs / its expert time
    t = torch.tensor([rep.get("expert_ms") or 0.0, rep.get("expert_flops") or 0.0, rep.get("exchange_ms") or 0.0,
                      rep.get("exchange_bytes") or 0.0], device="cuda", dtype=torch.float64)
    tall = [torch.empty_like(t) for _ in range(world)]
    dist.all_gather(tall, t)
    tall = torch.stack(tall).cpu().numpy()
    slow = int(tall[:, 0].argmax())
    tf = tall[slow, 1] / (tall[slow, 0] * 1e-3) / 1e12 if tall[slow, 0] > 0 else None
    cpu = None
    if rank == 0 and not args.no_cpu:
        try:
            cpu = cpu_baseline_ep(cfg, world, pol.t_drop)
        except Exception as e:  # noqa: BLE001
            cpu = {"value": None, "unit": "tokens/s", "cores": os.cpu_count(), "kind": "reference",
                   "sample": f"unavailable: {e}"}
    value = T * world / (ms_step * 1e-3)
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "bf16",
            "data": "synthetic tokens N(0,1) biased toward one hot expert, random-init weights of the named shapes",
            "config": {"workload": label, "config_id": cfg, "tokens_per_gpu": T,
                       "parallelism": f"ep{world} (contiguous placement, NCCL all-to-all)",
                       "drop_target": args.drop, "drop_rate": round(rate_main, 4),
                       "policy": "2T load-aware (t_max = uniform t)", "l2": "inputs > L2"},
            "roofline": {"bound": "tensor", "kernel": "expert grouped GEMMs of the slowest rank",
                         "achieved": r4(tf), "peak": peak_burst, "unit": "TFLOP/s",
                         "frac": r4(tf / peak_burst) if tf else None, "traffic": None,
                         "peak_kind": f"bf16 burst ({peak_src})",
                         "exchange": {"what": "all-to-all rows + records, both directions, per rank",
                                      "bytes_max_rank": int(tall[:, 3].max()),
                                      "ms_max_rank": r4(float(tall[:, 2].max())),
                                      "GBps_per_rank": r4(float((tall[:, 3] / np.maximum(tall[:, 2], 1e-9)).min()
                                                                / 1e6))}},
            "cpu_baseline": cpu,
            "e2e": {"value": T * world / (ms_e2e * 1e-3), "unit": "tokens/s",
                    "h2d_bytes_per_step": xh.numel() * xh.element_size() * world,
                    "d2h_bytes_per_step": oh.numel() * oh.element_size() * world},
            "gpu_launches": launches_per_step * args.steps, "clocks": clk.summary(),
            "ep": {"ms_per_step": {k: r4(v) for k, v in res.items()},
                   "speedup_load_aware_vs_no_drop": r4(res["no_drop"] / res["load_aware"]),
                   "speedup_load_aware_vs_uniform": r4(res["uniform"] / res["load_aware"]),
                   "pre_loads": rep["pre_loads"].tolist(), "post_loads": rep["post_loads"].tolist(),
                   "modeled_speedup": r4(rep["speedup"]), "setp": setp}}
        json.dump({"line": line, "report": {k: (v.tolist() if hasattr(v, "tolist") else v) for k, v in rep.items()
                                            if k != "local_drop_stats"}},
                  open(detail_path(cfg, world), "w"), indent=1, default=str)
        print(json.dumps(line))


def cpu_baseline_ep(cfg, world, t_drop):
    """The reference's simulate_step (ep_sim.hpp:110-160) + moe_forward on the
    host (oracle/_ref), on a bounded token sample of the same skewed batch."""
    R, E, K, ffn = ref_layer(cfg)
    bc = base_cfg(cfg)
    x = bench_tokens(bc, 8, skew=SKEW, gate=make_weights(bc)[0]).float().numpy()
    ncores = os.cpu_count() or 1
    t0 = time.perf_counter()
    rep = R.simulate_step(x, world, K, 2, "2t", t_drop, load_aware=True)
    raw = R.route_and_drop(x, K, 2).raw  # simulate_step keeps the pre-drop raw scores
    R.moe_forward(x, rep["idx"], raw, rep["frac"], threads=ncores)
    dt = time.perf_counter() - t0
    return {"value": x.shape[0] / dt, "unit": "tokens/s", "cores": ncores, "kind": "reference",
            "sample": f"{x.shape[0]} tokens: simulate_step (load-aware, {world} devices) + moe_forward over "
                      f"{ncores} threads, {dt:.1f} s"}


def stage_bytes(T, d, E, K, R, S, es=2, fused=False):
    """Algorithmic HBM bytes per launch of the non-GEMM kernels:
    the gate reads X and W_g and writes fp32 logits; the router reads the
    logits and writes one (code, score) pair per selection; the permutation
    reads those and writes row_token / row_scale per kept row and slot_pos per
    selection; the combine reads the R weighted expert rows (+ S*T shared
    rows) and writes the output."""
    if fused:  # K0 + K1 in one kernel: x and W_g in, logits + one (code, score) pair per selection out
        first = {"gate_route": T * d * es + d * E * es + T * E * 4 + T * K * 8}
    else:
        first = {"gate": T * d * es + d * E * es + T * E * 4, "router": T * E * 4 + T * K * 8}
    return {**first,
            "permute_plan": T * K * 8 + R * 8 + T * K * 4,
            "combine": (R + S * T) * d * es + T * d * es}


def run_single(args, local):
    import torch
    import paper_2508_18376_b200 as D
    cfg = args.config
    d, ffn, E, K, S, label = CONFIGS[cfg]
    ncores = os.cpu_count() or 1
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    ctx = D.Context(stream)
    info = {}
    layer, host = build_layer(cfg, ctx, info=info)
    E, K, ffn = host[3], host[4], host[5]
    T = args.tokens
    skew = SKEW if cfg == "c5" else 0.0
    x = bench_tokens(base_cfg(cfg), T, skew=skew, gate=host[0]).cuda()
    out = torch.empty_like(x)
    peak_burst, peak_sust, hbm, peak_src = load_peaks()

    # ---- drop sweep (0 / 25 / 50 %, 2T; 25 / 50 % 1T) timed in interleaved
    # rounds so slow drifts of the power-capped clock bias none of the ratios
    targets = sorted({0.0, 0.25, 0.5, args.drop})
    pols = {("2t", tg): calibrate(ctx, layer, x, tg) for tg in targets}
    for tg in (0.25, 0.5):
        pols[("1t", tg)] = calibrate(ctx, layer, x, tg, kind="1t")
    rounds, blk = 5, max(4, args.steps // 10)
    acc = {k: 0.0 for k in pols}
    with ClockSampler(local) as clk:
        for _ in range(rounds):
            for k, (pol, _) in pols.items():
                acc[k] += time_steps(lambda: D.forward(ctx, layer, x, pol, out=out), blk, 2)
        # ---- headline timed region (device-resident inputs); per-stage CUDA
        # events on every PROFILE_EVERY-th step (non-blocking event ring)
        pol_main, rate_main = pols[("2t", args.drop)]
        fwd = lambda: D.forward(ctx, layer, x, pol_main, out=out)
        for _ in range(max(3, args.warmup)):
            fwd()
        ctx.set_profiling(True, every=PROFILE_EVERY)
        ms = time_steps(fwd, args.steps, 0)
        prof = ctx.profile()
        ctx.set_profiling(False)
    nst = rounds * blk
    base_ms = acc[("2t", 0.0)] / nst
    sweep = {}
    for (kind, tg), (pol, rate) in pols.items():
        m_ = acc[(kind, tg)] / nst
        sweep[f"{kind}_{tg:.2f}"] = {"drop_rate": round(rate, 4), "ms": r4(m_), "speedup_vs_0": r4(base_ms / m_)}
    launches_per_step = D.last_launch_count()
    ms_step = ms / args.steps
    value = T / (ms_step * 1e-3)

    # ---- per-kernel device times (CUDA events on the context stream, same region)
    _, st = D.forward(ctx, layer, x, pol_main, out=out, with_stats=True)
    rt, _, _ = ctx.permutation(T, K, E)
    R = int(rt.size)
    per = {k: prof[k] / max(1, prof["calls"]) for k in ctx.STAGES}
    g1_flops = st["retained_flops"] * 2.0 / 3.0   # [W1|W3]: 4*d*width per kept row
    g2_flops = st["retained_flops"] / 3.0         # W2: 2*d*width per kept row
    g1_tf = g1_flops / (per["gemm1"] * 1e-3) / 1e12
    g2_tf = g2_flops / (per["gemm2"] * 1e-3) / 1e12
    traffic = None
    tp = os.path.join(ROOT, "profiles", f"ncu_gemm1_{cfg}.json")
    if os.path.exists(tp):
        try:
            traffic = json.load(open(tp)).get("dram_bytes_per_launch")
        except Exception:
            traffic = None
    fused = per["router"] == 0.0  # gate + router fused: the one kernel is timed as stage "gate"
    if fused:
        per["gate_route"] = per["gate"]
    kb = stage_bytes(T, d, E, K, R, S, fused=fused)
    kernels = {k: {"us": r4(per[k] * 1e3), "GBps": r4(b / (per[k] * 1e-3) / 1e9),
                   "frac_hbm": r4(b / (per[k] * 1e-3) / 1e9 / hbm)} for k, b in kb.items() if per[k] > 0}
    kernels["gemm2"] = {"us": r4(per["gemm2"] * 1e3), "TFLOPs": r4(g2_tf), "frac": r4(g2_tf / peak_burst)}
    roofline = {"bound": "tensor", "achieved": r4(g1_tf), "peak": peak_burst, "unit": "TFLOP/s",
                "frac": r4(g1_tf / peak_burst), "traffic": traffic,
                "kernel": "gemm1 (grouped [W1|W3] GEMM + SwiGLU, tcgen05 CTA pairs)",
                "peak_kind": f"bf16 burst ({peak_src}); frac of sustained {peak_sust}: {g1_tf / peak_sust:.3f}",
                "flops_per_launch": g1_flops, "us_per_launch": r4(per["gemm1"] * 1e3),
                "share_of_step": r4(per["gemm1"] / ms_step), "kernels": kernels,
                "stages_sampled": f"CUDA events on every {PROFILE_EVERY}th step of the timed region"}

    # ---- e2e through the public API with host buffers
    e2e = e2e_pipelined(D, stream, ctx, layer, pol_main, x, max(5, args.steps // 2))

    # ---- CPU baseline: the reference on the same reconstructed layer, same tokens
    cpu = None
    if not args.no_cpu:
        try:
            import numpy as np
            Rl, _, _, _ = ref_layer(cfg)
            sample = args.cpu_sample or {"c2": 512, "c3": 16, "c4": 512, "c5": 16}[cfg]
            xs = np.ascontiguousarray(x[:sample].float().cpu().numpy())
            rate, dt, rr = ref_rate(Rl, xs, K, pol_main.t_drop, ncores)
            cpu = {"value": rate, "unit": "tokens/s", "cores": ncores, "kind": "reference",
                   "sample": f"first {sample} tokens of the timed batch, same weights and calibration, "
                             f"reference profile/reconstruct, route_and_drop (2T t={pol_main.t_drop:.4f}: "
                             f"{Rl.drop_stats(sample, np.ones_like(rr.frac), rr.frac)['drop_rate']:.3f} drop) "
                             f"+ moe_forward over {ncores} threads, {dt:.1f} s"}
            del Rl
        except Exception as e:  # noqa: BLE001
            cpu = {"value": None, "unit": "tokens/s", "cores": ncores, "kind": "reference",
                   "sample": f"unavailable: {e}"}

    detail = {"offline": info.get("offline"), "per_stage_ms": per, "stats": st, "rows": R, "e2e": e2e,
              "sweep_full": {f"{k[0]}_{k[1]:.2f}": {"t_drop": p.t_drop, "drop_rate": r_, "ms": acc[k] / nst}
                             for k, (p, r_) in pols.items()}}
    epx = None
    if not args.no_ep:
        try:
            epx = ep_emulated(D, cfg)
            detail["ep_emulated"] = epx
        except Exception as e:  # noqa: BLE001
            epx = {"error": str(e)}
    extra = {}
    for c in [c for c in args.extra.split(",") if c and c != cfg]:
        try:
            extra[c] = extra_sweep(D, c, stream, T)
            detail.setdefault("extra", {})[c] = extra[c]
        except Exception as e:  # noqa: BLE001
            extra[c] = {"error": str(e)}

    line = {"metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": 1, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "bf16",
            "data": "synthetic tokens N(0,1), random-init weights of the named shapes",
            "config": {"workload": label, "config_id": cfg, "tokens_per_gpu": T, "drop_target": args.drop,
                       "drop_rate": round(rate_main, 4), "t_drop": pol_main.t_drop, "policy": "2T (t-0.01, t+0.01)",
                       "calib_tokens": CALIB[cfg],
                       "l2": "inputs > L2 (weights %.2f GB read per step)" % ((E * 3 * d * ffn + S * 3 * d * ffn) * 2 / 1e9),
                       "parallelism": "single GPU"},
            "roofline": roofline, "cpu_baseline": cpu,
            "e2e": {k: e2e[k] for k in ("value", "unit", "h2d_bytes_per_step", "d2h_bytes_per_step")},
            "gpu_launches": launches_per_step * args.steps, "gpu_launches_per_step": launches_per_step,
            "clocks": clk.summary(), "detail": os.path.relpath(detail_path(cfg, 1), ROOT)}
    if epx and "error" not in epx:
        line["ep_emulated"] = {k: r4(epx[k]) for k in ("speedup_load_aware_vs_no_drop",
                                                       "speedup_load_aware_vs_uniform_matched_rate")}
    line["extra_speedup_vs_0"] = {c: ({k: v["speedup_vs_0"] for k, v in e["sweep"].items()} if "sweep" in e else e)
                                  for c, e in extra.items()}
    line["sweep"] = sweep  # the metric's own axis last: it survives any tail truncation
    detail["line"] = line
    json.dump(detail, open(detail_path(cfg, 1), "w"), indent=1, default=str)
    print(json.dumps(line))


def extra_sweep(D, c, stream, T, rounds=5, blk=10):
    """0/25/50% 2T sweep of another BASELINE config, interleaved rounds."""
    import torch
    ctx2 = D.Context(stream)
    l2, h2 = build_layer(c, ctx2)
    x2 = bench_tokens(base_cfg(c), T).cuda()
    o2 = torch.empty_like(x2)
    p2s = {tg: calibrate(ctx2, l2, x2, tg) for tg in (0.0, 0.25, 0.5)}
    acc2 = {tg: 0.0 for tg in p2s}
    for _ in range(rounds):
        for tg, (p2, _) in p2s.items():
            acc2[tg] += time_steps(lambda: D.forward(ctx2, l2, x2, p2, out=o2), blk, 2)
    sw = {}
    for tg, (p2, r2) in p2s.items():
        ms2 = acc2[tg] / (rounds * blk)
        _, st2 = D.forward(ctx2, l2, x2, p2, out=o2, with_stats=True)
        sw[f"{tg:.2f}"] = {"drop_rate": round(r2, 4), "ms": r4(ms2), "tokens_per_s": r4(T / (ms2 * 1e-3)),
                           "gemm_tflops_step": r4(st2["retained_flops"] / (ms2 * 1e-3) / 1e12)}
    for v in sw.values():
        v["speedup_vs_0"] = r4(sw["0.00"]["ms"] / v["ms"])
    del l2, ctx2, x2, o2
    torch.cuda.empty_cache()
    return {"workload": CONFIGS[c][5], "method": f"{rounds} interleaved rounds x {blk} steps", "sweep": sw}


if __name__ == "__main__":
    main()
