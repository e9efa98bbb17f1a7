"""Probe: paired forward / fused IoU of cfg3 (K=4) and cfg4 (K=8) pairs scaled by s (float
inputs rounded after scaling) against the oracle: max |IoU - oracle|, count > 1e-5."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.getcwd())
import oracle  # noqa: E402
import paper_2011_11134_b200 as dgal  # noqa: E402
import synth  # noqa: E402

dev = torch.device("cuda:0")
for cfg in (3, 4):
    b = synth.gen_config(cfg, 1 << 15)
    K = b.p1.K
    for s in (1e-6, 1e-3, 1e3, 1e6):
        a = [(v.reshape(-1, K).astype(np.float64) * s).astype(np.float32) for v in (b.p1.x, b.p1.y, b.p2.x, b.p2.y)]
        X = [torch.from_numpy(np.ascontiguousarray(v)).to(dev) for v in a]
        iou, nx, xf = dgal.iou_paired_fwd(*X)
        iou_f = dgal.iou_paired_fused(*X, scale=1.0)[0]
        ref = oracle.iou_paired_fwd((a[0].astype(np.float64), a[1].astype(np.float64)),
                                    (a[2].astype(np.float64), a[3].astype(np.float64)))["iou"]
        e = np.abs(iou.cpu().numpy() - ref)
        ef = np.abs(iou_f.cpu().numpy() - ref)
        print(cfg, s, f"fwd max {e.max():.3e} n>1e-5 {(e > 1e-5).sum()}  fused max {ef.max():.3e} n>1e-5 {(ef > 1e-5).sum()}",
              flush=True)
