"""Quick C2 (OLMoE-shape) timing probe: per-stage device ms at 0/25/50% drop."""
import os, sys, time, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2508_18376_b200 as D

def build_layer(d, ffn, E, K, P=2, S=0, seed=0):
    g = torch.Generator(device="cuda").manual_seed(seed)
    sd = d ** -0.5
    gate = (torch.randn(d, E, device="cuda", generator=g) * sd).bfloat16()
    blocks = []
    w = ffn // P
    for _ in range(E * P):
        blocks.append(tuple((torch.randn(*s, device="cuda", generator=g) * sd).bfloat16() for s in ((d, w), (d, w), (w, d))))
    shared = [tuple((torch.randn(*s, device="cuda", generator=g) * sd).bfloat16() for s in ((d, ffn), (d, ffn), (ffn, d))) for _ in range(S)]
    return D.MoeLayer(d, ffn, E, K, gate, blocks, shared, replay_factor=P, dtype="bf16")

def calibrate(ctx, layer, x, target):
    if target == 0: return D.DropPolicy()
    lo, hi = 0.0, 1.0
    for _ in range(30):
        t = (lo + hi) / 2
        r = D.route_and_drop(ctx, layer, x, D.DropPolicy.two_t_from(t))
        if r.stats["drop_rate"] < target: lo = t
        else: hi = t
        if abs(r.stats["drop_rate"] - target) < 0.005: break
    return D.DropPolicy.two_t_from(t)

def main():
    T = int(os.environ.get("T", 16384))
    cfg = os.environ.get("CFG", "c2")
    shapes = {"c2": (2048, 1024, 64, 8, 2, 0), "c3": (4096, 3584, 32, 8, 2, 0), "c4": (2048, 1408, 64, 6, 2, 2)}
    d, ffn, E, K, P, S = shapes[cfg]
    torch.cuda.set_device(0)
    layer = build_layer(d, ffn, E, K, P, S)
    ctx = D.Context()
    x = torch.randn(T, d, device="cuda").bfloat16()
    res = {}
    for target in (0.0, 0.25, 0.5):
        pol = calibrate(ctx, layer, x, target)
        y, st = D.forward(ctx, layer, x, pol, with_stats=True)
        for _ in range(3): D.forward(ctx, layer, x, pol)
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        n = int(os.environ.get("ITERS", 30))
        s.record()
        for _ in range(n): D.forward(ctx, layer, x, pol)
        e.record(); torch.cuda.synchronize()
        ms = s.elapsed_time(e) / n
        ctx.set_profiling(True)
        for _ in range(5): D.forward(ctx, layer, x, pol)
        prof = ctx.profile(); ctx.set_profiling(False)
        prof = {k: (v / prof["calls"] if k != "calls" else v) for k, v in prof.items()}
        g = prof["gemm1"] + prof["gemm2"]
        res[target] = dict(drop=st["drop_rate"], ms=ms, tok_s=T / ms * 1e3, gemm_tflops=st["retained_flops"] / (g * 1e-3) / 1e12,
                           g1_tflops=st["retained_flops"] * 2 / 3 / (prof["gemm1"] * 1e-3) / 1e12,
                           g2_tflops=st["retained_flops"] / 3 / (prof["gemm2"] * 1e-3) / 1e12, prof=prof, launches=D.last_launch_count())
        print(target, json.dumps(res[target]), flush=True)
    print("speedup 25%:", res[0.0]["ms"] / res[0.25]["ms"], "50%:", res[0.0]["ms"] / res[0.5]["ms"])

if __name__ == "__main__":
    main()
