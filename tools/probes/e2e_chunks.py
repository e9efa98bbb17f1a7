"""Probe: e2e host-buffer call (dgal_iou_paired_host) throughput vs chunk size
(cfg3, 2^24 pairs, pinned buffers, three library streams)."""
import os
import sys

sys.path[:0] = [os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))]
import torch

import paper_2011_11134_b200 as dgal
import synth

dev = torch.device("cuda:0")
n = 1 << 24
b = synth.gen_config(3, n)
K = 4
xh = [torch.from_numpy(a.reshape(n, K)).pin_memory() for a in (b.p1.x, b.p1.y, b.p2.x, b.p2.y)]
gh = torch.full((n,), -1.0 / n).pin_memory()
out = (torch.empty(n).pin_memory(), *(torch.empty((n, K)).pin_memory() for _ in range(4)))
for chunk in (1 << 18, 1 << 19, 1 << 20, 1 << 21, 1 << 22):
    dgal.iou_paired_host(*xh, gh, out=out, chunk=chunk, device=dev)
    torch.cuda.synchronize()
    a, z = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(3):
        dgal.iou_paired_host(*xh, gh, out=out, chunk=chunk, device=dev)
    z.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(z) / 3
    print(f"chunk 2^{chunk.bit_length() - 1}: {ms:.2f} ms  {n / ms / 1e6:.3f} G pairs/s", flush=True)
