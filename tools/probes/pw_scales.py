"""Probe: pairwise IoU (indexed and tiled) of a cfg2-like scene scaled by s and offset by o
(float vertices rounded after the transform) against the oracle: max |IoU - oracle|."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.getcwd())
import oracle  # noqa: E402
import paper_2011_11134_b200 as dgal  # noqa: E402
import synth  # noqa: E402

dev = torch.device("cuda:0")
sc = synth.gen_cfg2_scene(n_objects=20, per_object=25)
n = sc.polys.n
for s, o in ((1e-6, 0.0), (1e6, 0.0), (1.0, 2e4), (0.05, 1e4)):
    x = (sc.polys.x.reshape(n, 4).astype(np.float64) * s + o).astype(np.float32)
    y = (sc.polys.y.reshape(n, 4).astype(np.float64) * s - o).astype(np.float32)
    P = synth.Polys(np.ascontiguousarray(x.reshape(-1)), np.ascontiguousarray(y.reshape(-1)), 4)
    ref = oracle.iou_pairwise(P, P)
    X, Y = torch.from_numpy(x).to(dev), torch.from_numpy(y).to(dev)
    for indexed in (True, False):
        got = dgal.iou_pairwise(X, Y, X, Y, want_mask=False, indexed=indexed)[0].cpu().numpy()
        e = np.abs(got - ref)
        print(s, o, "indexed" if indexed else "tiled", f"max {e.max():.3e} n>1e-5 {(e > 1e-5).sum()} nnz {int((ref > 0).sum())}",
              flush=True)
