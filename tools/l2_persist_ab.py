"""Experiment: keep the token matrix x (67 MB at C2) resident in L2 across a
forward with a persisting access-policy window on the context's stream, and
time GEMM1 / GEMM2 in the back-to-back loop with the diagnostic timeline
build (DSMOE_B200_LIB pointing at a -DDSB_GEMM_TIMES=1 build).
    L2P=0|1 python tools/l2_persist_ab.py"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
import paper_2508_18376_b200 as D
from cuda.bindings import runtime as rt

torch.cuda.set_device(0)
s = torch.cuda.Stream()
ctx = D.Context(stream=s)
layer, _ = bench.build_layer("c2", ctx)
x = bench.bench_tokens("c2", 16384).cuda()
pol = D.DropPolicy.two_t_from(0.085)
if os.environ.get("L2P", "0") == "1":
    frac = float(os.environ.get("L2P_HIT", "1.0"))
    mx = rt.cudaDeviceGetAttribute(rt.cudaDeviceAttr.cudaDevAttrMaxPersistingL2CacheSize, 0)[1]
    want = min(mx, int(os.environ.get("L2P_MB", "80")) << 20)
    (err,) = rt.cudaDeviceSetLimit(rt.cudaLimit.cudaLimitPersistingL2CacheSize, want)[:1]
    print("max persisting L2", mx >> 20, "MB, set", want >> 20, "MB", file=sys.stderr)
    v = rt.cudaStreamAttrValue()
    w = v.accessPolicyWindow
    w.base_ptr = x.data_ptr()
    w.num_bytes = x.numel() * x.element_size()
    w.hitRatio = frac
    w.hitProp = rt.cudaAccessProperty.cudaAccessPropertyPersisting
    w.missProp = rt.cudaAccessProperty.cudaAccessPropertyStreaming
    v.accessPolicyWindow = w
    r = rt.cudaStreamSetAttribute(s.cuda_stream, rt.cudaStreamAttrID.cudaLaunchAttributeAccessPolicyWindow, v)
    print("persisting window:", err, r, file=sys.stderr)
with torch.cuda.stream(s):
    for _ in range(3):
        D.forward(ctx, layer, x, pol)
    torch.cuda.synchronize()
    for _ in range(int(os.environ.get("STEPS", "12"))):
        D.forward(ctx, layer, x, pol)
    torch.cuda.synchronize()
