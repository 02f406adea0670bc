"""Host<->device copy bandwidth on this box (pinned memory, the e2e leg of
bench.py): H2D alone, D2H alone, both at once on separate streams."""
import torch

n = 16384 * 2048  # one C2 batch of bf16 tokens = 67 MB
h_in = torch.empty(n, dtype=torch.bfloat16).pin_memory()
h_out = torch.empty(n, dtype=torch.bfloat16).pin_memory()
d_in = torch.empty(n, dtype=torch.bfloat16, device="cuda")
d_out = torch.empty(n, dtype=torch.bfloat16, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def timed(fn, reps=20):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    s1.synchronize()
    s2.synchronize()
    torch.cuda.current_stream().wait_stream(s1)
    torch.cuda.current_stream().wait_stream(s2)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def h2d():
    with torch.cuda.stream(s1):
        d_in.copy_(h_in, non_blocking=True)


def d2h():
    with torch.cuda.stream(s2):
        h_out.copy_(d_out, non_blocking=True)


def both():
    h2d()
    d2h()


b = n * 2
for name, fn in (("h2d", h2d), ("d2h", d2h), ("both", both)):
    ms = timed(fn)
    print(f"{name}: {ms:.3f} ms per 67 MB batch, {b / (ms * 1e-3) / 1e9:.1f} GB/s per direction")
