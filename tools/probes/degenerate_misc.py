"""Probe: degenerate but plausible pairs vs the oracle — identical polygons with a rotated
vertex order, zero-size boxes, point / segment polygons (padded), coincident edges."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.getcwd())
import oracle  # noqa: E402
import paper_2011_11134_b200 as dgal  # noqa: E402
import synth  # noqa: E402

dev = torch.device("cuda:0")


def run(name, x1, y1, x2, y2):
    X = [torch.from_numpy(np.ascontiguousarray(a.astype(np.float32))).to(dev) for a in (x1, y1, x2, y2)]
    iou, nx, xf = dgal.iou_paired_fwd(*X)
    f = dgal.iou_paired_fused(*X, scale=1.0)[0]
    p1 = (X[0].cpu().numpy().astype(np.float64), X[1].cpu().numpy().astype(np.float64))
    p2 = (X[2].cpu().numpy().astype(np.float64), X[3].cpu().numpy().astype(np.float64))
    ref = oracle.iou_paired_fwd(p1, p2)
    e = np.abs(iou.cpu().numpy() - ref["iou"])
    ef = np.abs(f.cpu().numpy() - ref["iou"])
    print(f"{name:28s} fwd max {e.max():.3e} n>1e-5 {(e > 1e-5).sum()}  fused max {ef.max():.3e} "
          f"n>1e-5 {(ef > 1e-5).sum()}  nx==ref {np.mean(nx.cpu().numpy() == ref['nx']):.3f}", flush=True)


for K in (4, 8):
    b = synth.gen_config(3 if K == 4 else 4, 8192)
    x, y = b.p1.x.reshape(-1, K), b.p1.y.reshape(-1, K)
    for r in range(1, K):
        run(f"K{K} identical, start +{r}", x, y, np.roll(x, r, 1), np.roll(y, r, 1))
    # p2 = p1 with one edge shared, the rest shrunk toward the shared edge's midpoint
    # (K = 4 only: for octagons the shrink makes 35 % of the p2 non-convex — invalid input)
    if K == 4:
        mx, my = 0.5 * (x[:, :1] + x[:, 1:2]), 0.5 * (y[:, :1] + y[:, 1:2])
        x2, y2 = x.copy(), y.copy()
        x2[:, 2:] = mx + 0.5 * (x[:, 2:] - mx)
        y2[:, 2:] = my + 0.5 * (y[:, 2:] - my)
        run(f"K{K} shared edge, inside", x, y, x2, y2)
    # zero-area p2: all vertices at p1's centroid / a segment along p1's edge
    cx, cy = x.mean(1, keepdims=True), y.mean(1, keepdims=True)
    run(f"K{K} point p2", x, y, np.repeat(cx, K, 1), np.repeat(cy, K, 1))
    run(f"K{K} point p1", np.repeat(cx, K, 1), np.repeat(cy, K, 1), x, y)
    sx = np.concatenate([np.repeat(x[:, :1], K // 2, 1), np.repeat(x[:, 1:2], K // 2, 1)], 1)
    sy = np.concatenate([np.repeat(y[:, :1], K // 2, 1), np.repeat(y[:, 1:2], K // 2, 1)], 1)
    run(f"K{K} segment p2 on edge", x, y, sx, sy)
