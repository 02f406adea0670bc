"""Rate-targeted drop policies and gating analysis on the device (SURVEY §8(f)
next #2): the reference's threshold_sweep (dropping.hpp:310-345) and
analyze_gating (:207-228), plus `calibrate_rate`, which turns a target drop
rate into the 2T threshold that reaches it (the bisection of
acceptance.cpp:342-352) — the "rate-based" drop mask of the north star as a
calibrated threshold on the bit-exact threshold path."""
from __future__ import annotations

import ctypes as C

import numpy as np

from .dsmoe import (Context, DropPolicy, DsmoeError, LOGITS_EXACT, _chk, _x, lib, model_forward_dropped,
                    route_and_drop)


def analyze_gating(ctx: Context, layer, x, bins: int, logits_mode=LOGITS_EXACT) -> dict:
    """GatingDistributionReport (dropping.hpp:198-205) of one layer."""
    x = _x(x, layer)
    sc = np.zeros(layer.E, np.int64)
    rh = np.zeros(max(bins, 1), np.int64)
    nh = np.zeros(max(bins, 1), np.int64)
    _chk(lib().dsmoe_b200_analyze_gating(ctx.h, layer.h, C.c_void_p(x.data_ptr()), x.shape[0], bins, logits_mode,
                                         sc.ctypes.data, rh.ctypes.data, nh.ctypes.data))
    return {"bins": bins, "num_tokens": int(x.shape[0]), "top_k": layer.K, "selection_counts": sc.tolist(),
            "raw_hist": rh.tolist(), "norm_hist": nh.tolist()}


def mean_relative_error(a, b) -> float:
    """mean_relative_error (dropping.hpp:278-293): mean over tokens of
    ||a_t - b_t|| / ||b_t|| (||a_t - b_t|| when b_t = 0), in double."""
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    diff = np.sqrt(((a - b) ** 2).sum(axis=1))
    nb = np.sqrt((b ** 2).sum(axis=1))
    rel = np.where(nb > 0, diff / np.where(nb > 0, nb, 1.0), diff)
    return float(rel.mean()) if len(rel) else 0.0


def threshold_sweep(ctx: Context, layers, x, kind: str, thresholds, keep_top1=True, normalize=True,
                    logits_mode=LOGITS_EXACT) -> dict:
    """threshold_sweep (dropping.hpp:310-345): per threshold the aggregate and
    per-layer drop rates of model_forward_dropped and its mean relative error
    against the no-drop model_forward.  2T derives (t - 0.01, t + 0.01)."""
    thresholds = list(thresholds)
    if not thresholds:
        raise DsmoeError(1, "threshold_sweep: empty threshold list")
    if thresholds != sorted(thresholds):
        raise DsmoeError(1, "threshold_sweep: thresholds must be sorted ascending")
    if kind not in ("1t", "2t"):
        raise DsmoeError(1, "threshold_sweep: pick a drop policy kind")
    base, _ = model_forward_dropped(ctx, layers, x, DropPolicy(normalize=normalize), logits_mode=logits_mode)
    b = base.double().cpu().numpy()
    rows = []
    for t in thresholds:
        pol = DropPolicy.one_t(t, keep_top1) if kind == "1t" else DropPolicy.two_t_from(t, keep_top1)
        pol.normalize = normalize
        y, stats = model_forward_dropped(ctx, layers, x, pol, logits_mode=logits_mode)
        dropped = sum(s["dropped_units"] for s in stats)
        denom = sum(s["total_routed_units"] + s["shared_units"] for s in stats)
        rows.append({"threshold": t, "drop_rate": dropped / denom if denom > 0 else 0.0,
                     "per_layer_rates": [s["drop_rate"] for s in stats],
                     "mean_rel_error": mean_relative_error(y.double().cpu().numpy(), b)})
    return {"policy_kind": kind, "rows": rows}


def calibrate_rate(ctx: Context, layer, x, target: float, kind="2t", keep_top1=True, tol=0.005, iters=40,
                   logits_mode=LOGITS_EXACT):
    """Smallest-error bisection of t so drop_stats(route_and_drop).drop_rate
    lands within `tol` of `target` (acceptance.cpp:342-352).  Returns
    (DropPolicy, achieved rate).  Monotone: a larger t drops more."""
    if target <= 0:
        return DropPolicy(), 0.0
    lo, hi = 0.0, 1.0
    best = None
    for _ in range(iters):
        t = 0.5 * (lo + hi)
        pol = DropPolicy.one_t(t, keep_top1) if kind == "1t" else DropPolicy.two_t_from(t, keep_top1)
        rate = route_and_drop(ctx, layer, x, pol, logits_mode=logits_mode).stats["drop_rate"]
        if best is None or abs(rate - target) < abs(best[1] - target):
            best = (pol, rate)
        if abs(rate - target) <= tol:
            break
        if rate < target:
            lo = t
        else:
            hi = t
    return best


def calibrate_per_layer(ctx: Context, layers, x, target: float, kind="2t", keep_top1=True, tol=0.005,
                        logits_mode=LOGITS_EXACT):
    """Per-layer thresholds for model_forward_dropped: the
    threshold that reaches `target` differs by layer, so layer
    l's t is calibrated on the activations that reach it under the policies
    already chosen for layers 0..l-1.  Returns ([DropPolicy per layer],
    [achieved rate per layer])."""
    import torch
    from .dsmoe import forward
    cur = x
    pols, rates = [], []
    for layer in layers:
        pol, rate = calibrate_rate(ctx, layer, cur, target, kind, keep_top1, tol, logits_mode=logits_mode)
        pols.append(pol)
        rates.append(rate)
        nxt = torch.empty_like(cur)
        forward(ctx, layer, cur, pol, out=nxt, logits_mode=logits_mode, residual=True)
        cur = nxt
    return pols, rates
