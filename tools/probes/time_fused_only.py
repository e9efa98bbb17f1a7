"""Probe: CUDA-event time of the paired fused kernel alone (+ its refine pass) on
cfg3 / cfg4, repeated 3 times (A/B of builds via DGAL_SO)."""
import os
import sys

sys.path[:0] = [os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))]
import torch

import paper_2011_11134_b200 as dgal
import synth

dev = torch.device("cuda:0")
label = sys.argv[1] if len(sys.argv) > 1 else "?"
res = {}
for cfg, n in ((3, 1 << 24), (4, 1 << 22)):
    b = synth.gen_config(cfg, n)
    K = b.p1.K
    X = [torch.from_numpy(a.reshape(n, K)).to(dev) for a in (b.p1.x, b.p1.y, b.p2.x, b.p2.y)]
    out = (torch.empty(n, device=dev), *(torch.empty((n, K), device=dev) for _ in range(4)))
    for _ in range(5):
        dgal.iou_paired_fused(*X, scale=-1.0 / n, out=out)
    ts = []
    for _ in range(3):
        a, z = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(40):
            dgal.iou_paired_fused(*X, scale=-1.0 / n, out=out)
        z.record()
        torch.cuda.synchronize()
        ts.append(round(a.elapsed_time(z) / 40, 4))
    res[f"cfg{cfg}"] = ts
print(label, res, flush=True)
