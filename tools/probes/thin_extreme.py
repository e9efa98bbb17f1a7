"""Probe: IoU of gen_thin_pairs at aspect 1e3 / 1e4 (split, fused) vs the oracle."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.getcwd())
import oracle  # noqa: E402
import paper_2011_11134_b200 as dgal  # noqa: E402
import synth  # noqa: E402

dev = torch.device("cuda:0")
N = 20000
for K, verts in ((4, 3), (4, 4), (8, 8), (8, 5)):
    for aspect in (1e3, 1e4):
        b = synth.gen_thin_pairs(N, K, verts, aspect)
        X = [torch.from_numpy(a.reshape(N, K)).to(dev) for a in (b.p1.x, b.p1.y, b.p2.x, b.p2.y)]
        un = lambda a: a.reshape(N, K)[:, :verts].astype(np.float64)  # noqa: E731
        ref = oracle.iou_paired_fwd((un(b.p1.x), un(b.p1.y)), (un(b.p2.x), un(b.p2.y)))["iou"]
        iou = dgal.iou_paired_fwd(*X)[0].cpu().numpy()
        f = dgal.iou_paired_fused(*X, scale=1.0)[0].cpu().numpy()
        e, ef = np.abs(iou - ref), np.abs(f - ref)
        print(K, verts, aspect, f"overlap {(ref > 0).mean():.2f} fwd max {e.max():.3e} n>1e-5 {(e > 1e-5).sum()}  "
              f"fused max {ef.max():.3e} n>1e-5 {(ef > 1e-5).sum()}", flush=True)
