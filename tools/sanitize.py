"""Small end-to-end cases for compute-sanitizer (memcheck / racecheck):
bf16 forward with fused gather + CTA-pair GEMM2, shared experts, fp32 path,
reconstruction, and the EP pack / expert / combine kernels on one rank."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import oracle as O
import paper_2508_18376_b200 as D

torch.cuda.set_device(0)
ctx = D.Context()
rng = np.random.default_rng(3)


def layer(d, ffn, E, K, S=0, P=2, dtype="bf16", seed=1):
    L = O.generate_layer(d, ffn, E, K, S=S, seed=seed)
    L = O.partial_transform(L, P) if P > 1 else L
    return L, D.MoeLayer(L.d, L.ffn, L.E, L.K, L.gate, L.blocks, L.shared, replay_factor=L.P, dtype=dtype)


for (d, ffn, E, K, S, T, dt) in [(256, 256, 8, 2, 0, 300, "bf16"), (256, 192, 16, 4, 1, 257, "bf16"),
                                 (128, 128, 8, 2, 0, 100, "f32")]:
    L, dl = layer(d, ffn, E, K, S, dtype=dt)
    x = torch.from_numpy(O.generate_tokens(T, d, 5)).cuda()
    if dt == "bf16":
        x = x.bfloat16()
    y = D.forward(ctx, dl, x, D.DropPolicy.two_t_from(0.3))
    torch.cuda.synchronize()
    print("forward ok", d, ffn, E, K, S, T, dt, float(y.float().abs().max()))

# reconstruction on device
L = O.generate_layer(128, 128, 8, 2, seed=9)
base = D.MoeLayer(L.d, L.ffn, L.E, L.K, L.gate, L.blocks, L.shared, dtype="bf16")
xc = torch.from_numpy(O.generate_tokens(64, 128, 7)).cuda().bfloat16()
r = D.route_and_drop(ctx, base, xc)
vals = D.profile_importance(ctx, base, xc, r.indices, "abs_gate")
rec, _ = D.reconstruct_experts(ctx, base, vals)
torch.cuda.synchronize()
print("reconstruct ok")

# EP kernels on one rank (ep_pack / ep_expert / ep_combine)
L, dl = layer(256, 256, 8, 2, S=1)
T = 200
x = torch.from_numpy(O.generate_tokens(T, 256, 11)).cuda().bfloat16()
ctx2 = D.Context()
seg, R, _ = D.dispatch(ctx, dl, x, D.DropPolicy.two_t_from(0.3))
send = torch.empty((T * 2 + 1, 256), dtype=x.dtype, device="cuda")
rc = torch.empty(T * 2 + 1, dtype=torch.int32, device="cuda")
rr = torch.empty_like(rc)
rw = torch.empty(T * 2 + 1, dtype=torch.float32, device="cuda")
owner = np.zeros(8, np.int32)
from paper_2508_18376_b200 import dsmoe as DS
nu, ns = DS.ep_pack(ctx, dl, x, 1, owner, send, rc, rr, rw)
yl = DS.ep_expert(ctx2, dl, send, int(nu[0]), rc, rr, rw, int(ns[0]), [0, int(nu[0])], [0, int(ns[0])])
out = DS.ep_combine(ctx, dl, yl, T)
torch.cuda.synchronize()
print("ep ok", int(nu[0]), int(ns[0]))
