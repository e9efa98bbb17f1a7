"""Probe: per-launch CUDA-event times of the cfg3 fused loss call (fused kernel + refine
pass), 40 launches, for the loaded build (DGAL_SO): mean, min, max, and the number of
pairs the refine queue took (RefineQueue count after one call)."""
import os
import sys

sys.path[:0] = [os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))]
import torch

import paper_2011_11134_b200 as dgal
import synth

dev = torch.device("cuda:0")
n = 1 << 24
bt = synth.gen_config(3, n)
X = [torch.from_numpy(a.reshape(n, 4)).to(dev) for a in (bt.p1.x, bt.p1.y, bt.p2.x, bt.p2.y)]
out = (torch.empty(n, device=dev), *(torch.empty((n, 4), device=dev) for _ in range(4)))
for _ in range(3):
    dgal.iou_paired_fused(*X, scale=-1.0 / n, out=out)
torch.cuda.synchronize()
ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(40)]
for a, b in ev:
    a.record()
    dgal.iou_paired_fused(*X, scale=-1.0 / n, out=out)
    b.record()
torch.cuda.synchronize()
t = sorted(a.elapsed_time(b) for a, b in ev)
print(os.environ.get("DGAL_SO", "libdgal.so"), f"mean {sum(t)/len(t):.4f} min {t[0]:.4f} med {t[20]:.4f} max {t[-1]:.4f}",
      flush=True)
