"""Probe: box-parameter gradient error of the device box backward vs the oracle on
near-identical box pairs, per scale, on the pairs whose flags equal the oracle's."""
import os
import sys

sys.path[:0] = [os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))]
import numpy as np
import torch

import oracle
import paper_2011_11134_b200 as dgal

dev = torch.device("cuda:0")
n = 100_000
for scale in [1e-6, 1e-5, 1e-4, 1e-3, 1e-2, 1e-1]:
    rng = np.random.default_rng(int(-np.log10(scale)))
    cx = rng.uniform(0, 70, n); cy = rng.uniform(-40, 40, n)
    w = rng.uniform(0.5, 5, n); h = rng.uniform(0.5, 2, n); th = rng.uniform(-np.pi, np.pi, n)
    b1 = np.stack([cx, cy, w, h, th]).astype(np.float32)
    pert = rng.normal(size=(5, n)) * scale * np.array([w, w, w, h, np.ones(n)])
    b2 = (b1.astype(np.float64) + pert).astype(np.float32)
    g = rng.uniform(-1, 1, n).astype(np.float32)
    B1, B2 = torch.from_numpy(b1).to(dev), torch.from_numpy(b2).to(dev)
    iou, nx, xf = dgal.box_iou_paired_fwd(B1, B2)
    g1, g2 = dgal.box_iou_paired_bwd(B1, B2, torch.from_numpy(g).to(dev), nx, xf)
    ref = oracle.box_iou_paired(b1.T.astype(np.float64), b2.T.astype(np.float64), g.astype(np.float64))
    same = (nx.cpu().numpy() == ref["nx"]) & np.all(xf.cpu().numpy() == ref["xflags"], 1)
    G = np.concatenate([g1.cpu().numpy().T, g2.cpu().numpy().T], 1).astype(np.float64)
    R = np.concatenate([ref["gb1"], ref["gb2"]], 1)
    bad = (np.abs(G - R) > np.maximum(1e-4, 1e-3 * np.abs(R))).any(1)
    e = np.abs(G - R).max(1) / np.maximum(1.0, np.abs(R).max(1))
    print(f"scale {scale:.0e}: same flags {same.mean():.3f} out-of-tol {bad[same].mean():.2e} "
          f"p99 {np.quantile(e[same], 0.99):.1e} max {e[same].max():.1e}", flush=True)
