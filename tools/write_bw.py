#!/usr/bin/env python
"""Write-only HBM bandwidth on this GPU (the roof of the pairwise matrix):
cudaMemsetAsync and torch fill_ over a 40 GB float32 buffer, CUDA-event timed."""
import torch
n = 100_000 * 100_000
x = torch.empty(n, dtype=torch.float32, device="cuda")
for name, fn in (("fill_", lambda: x.fill_(0.0)), ("zero_", lambda: x.zero_())):
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(); fn(); fn(); fn(); b.record(); torch.cuda.synchronize()
    ms = a.elapsed_time(b) / 3
    print(f"{name}: {ms:.3f} ms  {4 * n / ms / 1e6:.0f} GB/s")
y = torch.empty(1 << 30, dtype=torch.bfloat16, device="cuda")
z = torch.empty_like(y)
for _ in range(2):
    z.copy_(y)
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record(); z.copy_(y); b.record(); torch.cuda.synchronize()
print(f"copy 1Gi bf16: {a.elapsed_time(b):.3f} ms {4 * (1 << 30) / a.elapsed_time(b) / 1e6:.0f} GB/s (r+w)")
