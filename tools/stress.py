"""Back-to-back forwards with changing token counts, drop policies and
return_logits (PDL chains across differently shaped launches), checked
against a second context run in isolation."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
import paper_2508_18376_b200 as D
torch.cuda.set_device(0)
ctx, ref_ctx = D.Context(), D.Context(stream=torch.cuda.Stream())
layer, _ = bench.build_layer("c2", ctx)
g = torch.Generator(device="cuda").manual_seed(1)
Ts = [1, 33, 512, 4096, 16384, 7, 2049]
xs = {T: torch.randn(T, 2048, device="cuda", generator=g).bfloat16() for T in Ts}
pols = [D.DropPolicy(), D.DropPolicy.two_t_from(0.08), D.DropPolicy.one_t(0.1)]
t0 = time.time()
outs = []
for i in range(700):
    T = Ts[i % len(Ts)]
    pol = pols[(i // len(Ts)) % len(pols)]
    if i % 5 == 0:
        D.route_and_drop(ctx, layer, xs[T], pol, return_logits=True)
    y = D.forward(ctx, layer, xs[T], pol)
    if i >= 700 - len(Ts) * len(pols):
        outs.append((T, pol, y))
torch.cuda.synchronize()
bad = 0
for T, pol, y in outs:
    with torch.cuda.stream(torch.cuda.Stream()):
        r = D.forward(ref_ctx, layer, xs[T], pol)
        torch.cuda.synchronize()
    bad += int(not torch.equal(r, y))
print(f"700 forwards in {time.time() - t0:.1f} s, mismatches vs isolated runs: {bad}")
sys.exit(1 if bad else 0)
