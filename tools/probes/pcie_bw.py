"""Probe: pinned host <-> device copy bandwidth on this box (H2D, D2H, both at once)."""
import torch

dev = torch.device("cuda:0")
n = 1 << 28   # 1 GiB of float32
h1 = torch.empty(n, dtype=torch.float32).pin_memory()
h2 = torch.empty(n, dtype=torch.float32).pin_memory()
d1 = torch.empty(n, dtype=torch.float32, device=dev)
d2 = torch.empty(n, dtype=torch.float32, device=dev)
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
E = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731
for name, both in (("h2d", 0), ("d2h", 1), ("both", 2)):
    for _ in range(2):
        a, b = E(), E()
        torch.cuda.synchronize()
        a.record()
        if both in (0, 2):
            with torch.cuda.stream(s1):
                d1.copy_(h1, non_blocking=True)
        if both in (1, 2):
            with torch.cuda.stream(s2):
                h2.copy_(d2, non_blocking=True)
        torch.cuda.current_stream().wait_stream(s1)
        torch.cuda.current_stream().wait_stream(s2)
        b.record()
        torch.cuda.synchronize()
    ms = a.elapsed_time(b)
    print(f"{name}: {4 * n * (2 if both == 2 else 1) / ms / 1e6:.1f} GB/s total ({ms:.1f} ms)")
