"""Back-to-back forwards with changing token counts and policies on one
context (programmatic-dependent-launch chains across differently shaped
launches, split-K gate on and off, logits copies in between) produce exactly
what isolated runs on a fresh context produce."""
import pytest

import oracle as O

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


def test_mixed_shape_chain_matches_isolated_runs():
    import paper_2508_18376_b200 as D
    torch.cuda.set_device(0)
    L = O.partial_transform(O.generate_layer(512, 384, 16, 4, S=1, seed=9), 2)
    layer = D.MoeLayer(L.d, L.ffn, L.E, L.K, L.gate, L.blocks, L.shared, replay_factor=2, dtype="bf16")
    ctx = D.Context()
    Ts = [1, 33, 300, 2500, 20000, 7]
    xs = {T: torch.from_numpy(O.bf16_round(O.generate_tokens(T, 512, seed=T))).cuda().bfloat16() for T in Ts}
    pols = [D.DropPolicy(), D.DropPolicy.two_t_from(0.2), D.DropPolicy.one_t(0.25)]
    last = {}
    for i in range(3 * len(Ts) * len(pols)):
        T, p = Ts[i % len(Ts)], (i // len(Ts)) % len(pols)
        if i % 4 == 0:
            D.route_and_drop(ctx, layer, xs[T], pols[p], return_logits=True)
        last[(T, p)] = D.forward(ctx, layer, xs[T], pols[p])
    torch.cuda.synchronize()
    for (T, p), y in last.items():
        ref = D.forward(D.Context(), layer, xs[T], pols[p])
        torch.cuda.synchronize()
        assert torch.equal(ref, y), (T, p)


def test_two_contexts_on_two_streams_concurrently():
    """Per-context device state (superchunk sums and their epoch, the GEMM1
    tile-claim counter, routing buffers) is isolated: two contexts whose
    forwards are issued interleaved on two streams, with no synchronisation
    between them, give exactly the outputs of isolated runs."""
    import paper_2508_18376_b200 as D
    torch.cuda.set_device(0)
    L = O.partial_transform(O.generate_layer(512, 384, 16, 4, S=0, seed=11), 2)
    layer = D.MoeLayer(L.d, L.ffn, L.E, L.K, L.gate, L.blocks, L.shared, replay_factor=2, dtype="bf16")
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    c1, c2 = D.Context(s1), D.Context(s2)
    Ts = [4133, 20000, 300]
    xs = {T: torch.from_numpy(O.bf16_round(O.generate_tokens(T, 512, seed=T + 1))).cuda().bfloat16() for T in Ts}
    pol = D.DropPolicy.two_t_from(0.2)
    outs = {(k, T): torch.empty_like(xs[T]) for k in (1, 2) for T in Ts}
    torch.cuda.synchronize()
    for rep in range(4):
        for T in Ts:
            with torch.cuda.stream(s1):
                D.forward(c1, layer, xs[T], pol, out=outs[(1, T)])
            with torch.cuda.stream(s2):
                D.forward(c2, layer, xs[Ts[(Ts.index(T) + 1) % len(Ts)]], pol,
                          out=outs[(2, Ts[(Ts.index(T) + 1) % len(Ts)])])
    torch.cuda.synchronize()
    for (k, T), y in outs.items():
        ref = D.forward(D.Context(), layer, xs[T], pol)
        torch.cuda.synchronize()
        assert torch.equal(ref, y), (k, T)
