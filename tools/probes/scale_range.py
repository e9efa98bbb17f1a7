"""Probe: IoU / gradient parity at large coordinate scales (cfg1 pairs scaled by s):
the clip's sentinel values bound the usable range."""
import os
import sys

sys.path[:0] = [os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))),
                os.path.join(os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))), "tests")]
import numpy as np
import torch

import oracle
import paper_2011_11134_b200 as dgal
from helpers import margin_batch

dev = torch.device("cuda:0")
b = margin_batch(1, 20000)
for s in (1.0, 1e2, 1e3, 1e4, 3e4):
    X1, Y1 = (a * s for a in b.p1.xy64()); X2, Y2 = (a * s for a in b.p2.xy64())
    X1, Y1, X2, Y2 = (a.astype(np.float32) for a in (X1, Y1, X2, Y2))
    T = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)  # noqa: E731
    iou, nx, xf = dgal.iou_paired_fwd(T(X1), T(Y1), T(X2), T(Y2))
    g = dgal.iou_paired_bwd(T(X1), T(Y1), T(X2), T(Y2), torch.ones(X1.shape[0], device=dev), nx, xf)
    ref = oracle.iou_paired_fwd((X1, Y1), (X2, Y2))
    rg = oracle.iou_paired_bwd((X1, Y1), (X2, Y2), np.ones(X1.shape[0]))
    e = np.abs(iou.cpu().numpy() - ref["iou"]).max()
    fl = np.mean(nx.cpu().numpy() != ref["nx"])
    ge = max((np.abs(a.cpu().numpy() - r) / np.maximum(1e-30, np.abs(r).max(1, keepdims=True))).max()
             for a, r in zip(g, rg))
    print(f"scale {s:g}: max IoU err {e:.2e}, nx mismatch {fl:.2e}, max rel grad err {ge:.2e}", flush=True)
