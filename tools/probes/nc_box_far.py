"""Probe: near-coincident box pairs (prediction ~ target) moved far from the origin and
with large angles: IoU vs the oracle on every pair, parameter gradients (split, fused) on
the pairs whose flags equal the oracle's."""
import math
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.getcwd())
sys.path.insert(0, os.path.join(os.getcwd(), "tests"))
import oracle  # noqa: E402
import paper_2011_11134_b200 as dgal  # noqa: E402
from test_gpu_paired import _near_coincident_boxes  # noqa: E402

dev = torch.device("cuda:0")
for scale in (1e-5, 1e-3):
    for off, dth in ((0.0, 0.0), (5e3, 0.0), (0.0, 100.0), (5e3, 100.0)):
        b1, b2 = _near_coincident_boxes(40_000, scale, seed=7)
        b1, b2 = b1.copy(), b2.copy()
        b1[0] += np.float32(off); b2[0] += np.float32(off)
        b1[1] -= np.float32(off); b2[1] -= np.float32(off)
        b1[4] += np.float32(dth); b2[4] += np.float32(dth)
        g = np.random.default_rng(6).uniform(-1, 1, b1.shape[1]).astype(np.float32)
        B1, B2 = torch.from_numpy(b1).to(dev), torch.from_numpy(b2).to(dev)
        iou, nx, xf = dgal.box_iou_paired_fwd(B1, B2)
        gg = torch.from_numpy(g).to(dev)
        g1, g2 = dgal.box_iou_paired_bwd(B1, B2, gg, nx, xf)
        fi, f1, f2 = dgal.box_iou_paired_fused(B1, B2, grad=gg)
        ref = oracle.box_iou_paired(b1.T.astype(np.float64), b2.T.astype(np.float64), g.astype(np.float64))
        nx, xf = nx.cpu().numpy(), xf.cpu().numpy()
        same = (nx == ref["nx"]) & np.all(xf == ref["xflags"], 1)
        def gerr(a, want):
            a = a.cpu().numpy().T.astype(np.float64)[same]
            e = np.abs(a - want[same])
            return int(((e > 1e-4) & (e > 1e-3 * np.abs(want[same]))).sum())
        ei = np.abs(iou.cpu().numpy() - ref["iou"]).max()
        ef = np.abs(fi.cpu().numpy() - ref["iou"]).max()
        print(scale, off, dth, f"iou {ei:.2e} fused {ef:.2e} same {same.mean():.3f} bad-grad split "
              f"{gerr(g1, ref['gb1']) + gerr(g2, ref['gb2'])} fused {gerr(f1, ref['gb1']) + gerr(f2, ref['gb2'])}", flush=True)
