"""Probe: e2e host-pipeline throughput vs chunk size / stream count (cfg3, 2^24 pairs)."""
import os
import sys

sys.path[:0] = [os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))]
import torch

import synth
from paper_2011_11134_b200.hostpipe import HostPipeline

dev = torch.device("cuda:0")
n = 1 << 24
b = synth.gen_config(3, n)
K = 4
x4h = torch.stack([torch.from_numpy(a.reshape(n, K)) for a in (b.p1.x, b.p1.y, b.p2.x, b.p2.y)]).pin_memory()
gh = torch.full((n,), -1.0 / n).pin_memory()
iouh = torch.empty(n).pin_memory()
g4h = torch.empty((4, n, K)).pin_memory()
for chunk in (1 << 18, 1 << 19, 1 << 20, 1 << 21):
    for ns in (2, 3, 4):
        pipe = HostPipeline(K, chunk=chunk, nstreams=ns, device=dev)
        pipe.run(x4h, gh, iouh, g4h)
        torch.cuda.synchronize()
        a, z = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(3):
            pipe.run(x4h, gh, iouh, g4h)
        z.record()
        torch.cuda.synchronize()
        ms = a.elapsed_time(z) / 3
        print(f"chunk 2^{chunk.bit_length() - 1} streams {ns}: {ms:.2f} ms  {n / ms / 1e6:.3f} G pairs/s", flush=True)
        del pipe
