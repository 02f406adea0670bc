"""The forward is CUDA-graph capturable (no host synchronisation, allocation or
pageable copy once the context's workspace exists for a token count): a
captured forward replays bit-identically to the eager one, including after
the input changes in place."""
import numpy as np
import pytest

import oracle as O

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


# (T, E, K, ffn): the last case has >= 16 GEMM1 tiles per CTA pair, so GEMM1
# claims its tiles dynamically (the claim counter re-arms itself in every replay)
@pytest.mark.parametrize("T,E,K,ffn", [(1, 16, 4, 256), (77, 16, 4, 256), (1000, 16, 4, 256), (20000, 64, 8, 512)])
def test_graph_replay_matches_eager(T, E, K, ffn):
    import paper_2508_18376_b200 as D
    torch.cuda.set_device(0)
    s = torch.cuda.Stream()
    ctx = D.Context(stream=s)
    L = O.partial_transform(O.generate_layer(256, ffn, E, K, S=1, seed=5), 2)
    layer = D.MoeLayer(L.d, L.ffn, L.E, L.K, L.gate, L.blocks, L.shared, replay_factor=2, dtype="bf16")
    pol = D.DropPolicy.two_t_from(0.2)
    x = torch.from_numpy(O.bf16_round(O.generate_tokens(T, 256, seed=T))).cuda().bfloat16()
    out = torch.empty_like(x)
    with torch.cuda.stream(s):
        D.forward(ctx, layer, x, pol, out=out)  # workspace + tile tables for this T
        s.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            D.forward(ctx, layer, x, pol, out=out)
        for seed in (1, 2):
            x.copy_(torch.from_numpy(O.bf16_round(O.generate_tokens(T, 256, seed=100 + seed))).cuda().bfloat16())
            g.replay()
            s.synchronize()
            got = out.clone()
            ref = D.forward(ctx, layer, x, pol)
            s.synchronize()
            assert torch.equal(got, ref)
