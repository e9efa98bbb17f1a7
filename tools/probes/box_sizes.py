"""Probe: box IoU (2D / 3D, split and fused) vs the oracle with every length (sizes, centre
offsets from the scene origin, heights) scaled by s."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.getcwd())
import oracle  # noqa: E402
import paper_2011_11134_b200 as dgal  # noqa: E402
import synth  # noqa: E402

dev = torch.device("cuda:0")
for dims in (2, 3):
    lens = (0, 1, 2, 3) if dims == 2 else (0, 1, 2, 3, 4, 5)
    for s in (1e-4, 1e-2, 1e2, 1e4):
        b = synth.gen_box_pairs(1 << 15, dims, seed=31)
        for bb in (b.b1, b.b2):
            for r in lens:
                bb[r] *= np.float32(s)
        r1, r2 = b.rows64()
        ref = oracle.box_iou_paired(r1, r2, b.grad.astype(np.float64))
        B1, B2 = torch.from_numpy(b.b1).to(dev), torch.from_numpy(b.b2).to(dev)
        iou = dgal.box_iou_paired_fwd(B1, B2)[0].cpu().numpy()
        f = dgal.box_iou_paired_fused(B1, B2, grad=torch.from_numpy(b.grad).to(dev))[0].cpu().numpy()
        e = np.abs(iou.astype(np.float64) - ref["iou"])
        ef = np.abs(f.astype(np.float64) - ref["iou"])
        print(dims, s, f"fwd max {e.max():.3e} n>1e-5 {(e > 1e-5).sum()}  fused max {ef.max():.3e} n>1e-5 {(ef > 1e-5).sum()}",
              flush=True)
