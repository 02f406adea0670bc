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
                                 (128, 128, 8, 2, 0, 100, "f32"),
                                 (128, 64, 32, 8, 0, 12000, "bf16")]:  # gate_route: two tiles per CTA
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

# round 2 kernels: transforms + read-back, block-view moe_forward, EP v2 (counts, device thresholds,
# sync-free dispatch with interleaved records, shard of held blocks), reference-ABI compare rows
Lb = O.generate_layer(128, 192, 6, 2, S=1, seed=21)
base = D.MoeLayer(Lb.d, Lb.ffn, Lb.E, Lb.K, Lb.gate, Lb.blocks, Lb.shared, dtype="bf16")
for mode, p in (("complete", 4), ("partial", 3), ("partial", 2)):
    t = D.transform(ctx, base, mode, p)
    g, blocks, shared = D.layer_weights(ctx, t)
    if mode == "partial":
        D.transform(ctx, t, "reverse")
torch.cuda.synchronize()
print("transforms ok")
t2 = D.partial_transform(ctx, base, 2)
xt = torch.from_numpy(O.generate_tokens(70, 128, 3)).cuda().bfloat16()
idx = torch.from_numpy(rng.integers(0, 12, size=(70, 4)).astype(np.int32)).cuda()
raw = torch.from_numpy(rng.uniform(0.1, 0.5, size=(70, 4))).cuda()
frac = torch.from_numpy(rng.choice([0.0, 0.5, 1.0], size=(70, 4))).cuda()
D.moe_forward(ctx, t2, xt, (idx, raw, frac))
torch.cuda.synchronize()
print("block view ok")
T = 200
x = torch.from_numpy(O.generate_tokens(T, 256, 11)).cuda().bfloat16()
held = np.zeros(16, np.uint8)
held[::2] = 1  # S-ETP-like: only the major halves
sh = D.layer_shard_blocks(ctx, dl, held)
cnt = D.ep_route_counts(ctx, dl, x, D.DropPolicy())
dv = torch.zeros(16, dtype=torch.int32, device="cuda")
t_unit, loads = D.ep_thresholds(ctx, dl, cnt, 1, dv, 0.3, True)
send = torch.empty((T * 2 + 1, 256), dtype=x.dtype, device="cuda")
rec = torch.empty((T * 4 + 1, 3), dtype=torch.int32, device="cuda")
cn = torch.empty((1, 2), dtype=torch.int64, device="cuda")
dest = torch.full((8, 2), 1, dtype=torch.int32, device="cuda")
D.ep_dispatch(ctx, dl, x, D.DropPolicy.two_t_from(0.3), t_unit, 1, dest, send, rec, cn)
c = cn.cpu().numpy()[0]
yl = D.ep_expert_packed(ctx2, sh, send, int(c[0]), rec, int(c[1]), [0, int(c[0])], [0, int(c[1])])
out = DS.ep_combine(ctx, dl, yl, T)
D.ep_last_counts(ctx, dl, T)
torch.cuda.synchronize()
print("ep v2 ok", c.tolist())
from paper_2508_18376_b200 import abi as A
import tempfile
tmp = tempfile.mkdtemp()
lib = A.DsmoeAbi()
m = lib.generate_model({"d_model": 128, "d_ffn": 128, "num_experts": 8, "top_k": 2}, 3)
lib.generate_tokens(40, 128, 4, tmp + "/x.tok")
rm, _ = lib.reconstruct(m, tmp + "/x.tok", "abs_gate")
lib.infer(rm, tmp + "/x.tok", {"kind": "2t", "t_drop": 0.3})
lib.sim_ep(rm, tmp + "/x.tok", 2, "round_robin", {"kind": "2t", "t_drop": 0.3})
print("abi ok")
