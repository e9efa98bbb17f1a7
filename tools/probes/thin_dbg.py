"""Probe: the pairs of gen_thin_pairs(aspect 1e4) whose IoU misses the oracle by > 1e-5:
GPU / oracle records, areas, and R^2 / A_u (the thin test's ratio)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.getcwd())
import oracle  # noqa: E402
import paper_2011_11134_b200 as dgal  # noqa: E402
import synth  # noqa: E402

dev = torch.device("cuda:0")
N = 20000
for K, verts in ((4, 3), (4, 4), (8, 5)):
    b = synth.gen_thin_pairs(N, K, verts, 1e4)
    X = [torch.from_numpy(a.reshape(N, K)).to(dev) for a in (b.p1.x, b.p1.y, b.p2.x, b.p2.y)]
    un = lambda a: a.reshape(N, K)[:, :verts].astype(np.float64)  # noqa: E731
    ref = oracle.iou_paired_fwd((un(b.p1.x), un(b.p1.y)), (un(b.p2.x), un(b.p2.y)))
    iou, nx, xf = dgal.iou_paired_fwd(*X)
    iou, nx, xf = iou.cpu().numpy(), nx.cpu().numpy(), xf.cpu().numpy()
    bad = np.nonzero(np.abs(iou - ref["iou"]) > 1e-5)[0]
    for k in bad[:4]:
        P = np.stack([un(b.p1.x)[k], un(b.p1.y)[k]], 1)
        Q = np.stack([un(b.p2.x)[k], un(b.p2.y)[k]], 1)
        o = P[0]
        R2 = max(np.max(np.sum((P - o) ** 2, 1)), np.max(np.sum((Q - o) ** 2, 1)))
        A = lambda V: 0.5 * np.sum(V[:, 0] * np.roll(V[:, 1], -1) - np.roll(V[:, 0], -1) * V[:, 1])  # noqa: E731
        Au = A(P - o) + A(Q - o) - ref["area_i"][k]
        print(K, verts, k, f"gpu {iou[k]:.6g} nx {nx[k]} {xf[k][:nx[k]].tolist()} | ora {ref['iou'][k]:.6g} nx {ref['nx'][k]} "
              f"{ref['xflags'][k][:ref['nx'][k]].tolist()} | R2/Au {R2 / (2 * Au):.3g}", flush=True)
