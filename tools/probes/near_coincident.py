"""Probe: IoU error of the device path on near-identical box pairs (prediction ~
ground truth, the converged-training regime): b2 = b1 + small perturbations of
the centre / size / yaw.  Prints the max |IoU_gpu - IoU_oracle| per scale, for
the box path and for the polygon path on (oracle) corners."""
import os
import sys

sys.path[:0] = [os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))]
import numpy as np
import torch

import oracle
import paper_2011_11134_b200 as dgal

rng = np.random.default_rng(0)
n = 200_000
dev = torch.device("cuda:0")
for scale in [1e-7, 1e-6, 1e-5, 1e-4, 1e-3, 1e-2]:
    cx = rng.uniform(0, 70, n); cy = rng.uniform(-40, 40, n)
    w = rng.uniform(0.5, 5, n); h = rng.uniform(0.5, 2, n); th = rng.uniform(-np.pi, np.pi, n)
    b1 = np.stack([cx, cy, w, h, th]).astype(np.float32)
    pert = rng.normal(size=(5, n)) * scale * np.array([w, w, w, h, np.ones(n)])
    b2 = (b1.astype(np.float64) + pert).astype(np.float32)
    ref = oracle.box_iou_paired(b1.T.astype(np.float64), b2.T.astype(np.float64))["iou"]
    B1, B2 = torch.from_numpy(b1).to(dev), torch.from_numpy(b2).to(dev)
    iou = dgal.box_iou_paired_fwd(B1, B2)[0].cpu().numpy()
    e = np.abs(iou - ref)
    x1, y1 = oracle.box_corners(b1.T.astype(np.float64))
    x2, y2 = oracle.box_corners(b2.T.astype(np.float64))
    T = lambda a: torch.from_numpy(a.astype(np.float32)).to(dev)  # noqa: E731
    pi = dgal.iou_paired_fwd(T(x1), T(y1), T(x2), T(y2))[0].cpu().numpy()
    pref = oracle.iou_paired_fwd((x1.astype(np.float32), y1.astype(np.float32)),
                                 (x2.astype(np.float32), y2.astype(np.float32)))["iou"]
    ep = np.abs(pi - pref)
    print(f"scale {scale:.0e}: box max err {e.max():.2e} (>1e-5: {np.mean(e > 1e-5):.2e})  "
          f"poly max err {ep.max():.2e} (>1e-5: {np.mean(ep > 1e-5):.2e})  median iou {np.median(ref):.5f}",
          flush=True)
