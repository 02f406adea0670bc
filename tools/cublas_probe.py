import torch
torch.cuda.set_device(0)
a = torch.randn(131072, 2048, device="cuda").bfloat16()
b = torch.randn(2048, 2048, device="cuda").bfloat16()
for _ in range(3):
    c = a @ b.t()
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()
c = a @ b.t()
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record()
for _ in range(20):
    c = a @ b.t()
e.record(); torch.cuda.synchronize()
ms = s.elapsed_time(e) / 20
print("cublas ms", ms, "TF/s", 2 * 131072 * 2048 * 2048 / ms / 1e9)
