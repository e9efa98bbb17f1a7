"""Probe: 3D box IoU vs the oracle with the vertical centres moved by a common offset (m)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.getcwd())
import oracle  # noqa: E402
import paper_2011_11134_b200 as dgal  # noqa: E402
import synth  # noqa: E402

dev = torch.device("cuda:0")
for off in (0.0, 1e2, 1e3, 1e4):
    b = synth.gen_box_pairs(1 << 15, 3, seed=21)
    b.b1[2] += np.float32(off)
    b.b2[2] += np.float32(off)
    r1, r2 = b.rows64()
    ref = oracle.box_iou_paired(r1, r2, b.grad.astype(np.float64))
    iou, nx, xf = dgal.box_iou_paired_fwd(torch.from_numpy(b.b1).to(dev), torch.from_numpy(b.b2).to(dev))
    e = np.abs(iou.cpu().numpy().astype(np.float64) - ref["iou"])
    f = dgal.box_iou_paired_fused(torch.from_numpy(b.b1).to(dev), torch.from_numpy(b.b2).to(dev),
                                  grad=torch.from_numpy(b.grad).to(dev))[0].cpu().numpy()
    ef = np.abs(f.astype(np.float64) - ref["iou"])
    print(off, f"fwd max {e.max():.3e} n>1e-5 {(e > 1e-5).sum()}  fused max {ef.max():.3e} n>1e-5 {(ef > 1e-5).sum()}",
          flush=True)
