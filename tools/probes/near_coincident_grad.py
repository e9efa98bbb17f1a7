"""Probe: vertex-gradient error of the device backward (split fwd/bwd and fused)
vs the oracle on near-identical box pairs (prediction ~ target), per scale.
Error per pair = max |g_gpu - g_oracle| / max(1, max |g_oracle|) over its 16 entries."""
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
    x1, y1 = oracle.box_corners(b1.T.astype(np.float64))
    x2, y2 = oracle.box_corners(b2.T.astype(np.float64))
    x1, y1, x2, y2 = (a.astype(np.float32) for a in (x1, y1, x2, y2))
    g = rng.uniform(-1, 1, n).astype(np.float32)
    T = lambda a: torch.from_numpy(a).to(dev)  # noqa: E731
    X = (T(x1), T(y1), T(x2), T(y2))
    iou, nx, xf = dgal.iou_paired_fwd(*X)
    gs = dgal.iou_paired_bwd(*X, T(g), nx, xf)
    fu = dgal.iou_paired_fused(*X, grad=T(g))[1:]
    ref = oracle.iou_paired_bwd((x1, y1), (x2, y2), g)
    rf = oracle.iou_paired_fwd((x1, y1), (x2, y2))
    same = (nx.cpu().numpy() == rf["nx"]) & np.all(xf.cpu().numpy() == rf["xflags"], 1)
    R = np.concatenate(ref, 1)
    den = np.maximum(1.0, np.abs(R).max(1))
    for name, got in (("split", gs), ("fused", fu)):
        G = np.concatenate([t.cpu().numpy() for t in got], 1).astype(np.float64)
        e = np.abs(G - R).max(1) / den
        badm = (np.abs(G - R) > np.maximum(1e-4, 1e-3 * np.abs(R))).any(1)
        es = e[same]
        print(f"scale {scale:.0e} {name}: out-of-tol {badm.mean():.2e} | same flags {same.mean():.3f}: "
              f"p99 {np.quantile(es, 0.99):.1e} max {es.max():.1e} out-of-tol {badm[same].mean():.2e} | "
              f"other: out-of-tol {badm[~same].mean() if (~same).any() else 0:.2e}", flush=True)
