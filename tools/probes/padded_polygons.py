"""Probe: polygons with fewer than K vertices, padded by repeating their last vertex.
IoU vs the oracle on the padded input, and the vertex gradients summed over the copies
of the repeated vertex vs the oracle on the UNPADDED polygons (same m for both)."""
import os
import sys

sys.path[:0] = [os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))]
import numpy as np
import torch

import oracle
import paper_2011_11134_b200 as dgal

dev = torch.device("cuda:0")
rng = np.random.default_rng(0)


def convex(n, m):
    c = rng.uniform(-5, 5, (n, 2)); a = rng.uniform(1, 3, n); b = a * rng.uniform(0.5, 1, n)
    ang = np.sort(rng.uniform(0, 2 * np.pi, (n, m)), 1); phi = rng.uniform(-np.pi, np.pi, n)
    ex, ey = a[:, None] * np.cos(ang), b[:, None] * np.sin(ang)
    x = c[:, :1] + np.cos(phi)[:, None] * ex - np.sin(phi)[:, None] * ey
    y = c[:, 1:] + np.sin(phi)[:, None] * ex + np.cos(phi)[:, None] * ey
    return x.astype(np.float32), y.astype(np.float32)


def pad(x, K):
    m = x.shape[1]
    return np.ascontiguousarray(np.concatenate([x, np.repeat(x[:, -1:], K - m, 1)], 1) if m < K else x)


def fold(g, m):   # sum the copies of the repeated last vertex
    out = g[:, :m].copy()
    out[:, m - 1] += g[:, m:].sum(1)
    return out


n = 20000
for (m, K) in [(3, 4), (5, 8), (6, 8), (7, 8)]:
    x1, y1 = convex(n, m); x2, y2 = convex(n, m)
    x2 += (x1.mean(1, keepdims=True) - x2.mean(1, keepdims=True)) * 0.8
    y2 += (y1.mean(1, keepdims=True) - y2.mean(1, keepdims=True)) * 0.8
    X1, Y1, X2, Y2 = pad(x1, K), pad(y1, K), pad(x2, K), pad(y2, K)
    T = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)  # noqa: E731
    iou, nx, xf = dgal.iou_paired_fwd(T(X1), T(Y1), T(X2), T(Y2))
    g = [t.cpu().numpy().astype(np.float64) for t in
         dgal.iou_paired_bwd(T(X1), T(Y1), T(X2), T(Y2), torch.ones(n, device=dev), nx, xf)]
    ref = oracle.iou_paired_fwd((x1, y1), (x2, y2))
    rg = oracle.iou_paired_bwd((x1, y1), (x2, y2), np.ones(n))
    ok = oracle.margin_ok((x1, y1), (x2, y2))
    e = np.abs(iou.cpu().numpy() - ref["iou"])
    ge = max(np.abs(fold(a, m) - b)[ok].max() for a, b in zip(g, rg))
    print(f"m={m} padded to K={K}: max IoU err {e.max():.2e}; summed-copy gradient vs unpadded oracle "
          f"(margin pairs {ok.mean():.2f}): max err {ge:.2e}", flush=True)
