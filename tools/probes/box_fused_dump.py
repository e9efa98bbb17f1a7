"""Probe: the box pairs of tests/test_gpu_box.py::test_box_fused_near_coincident whose
fused gradients miss the oracle (same-flag pairs), dumped to gpurun_out/box_fused_dump.npz."""
import math
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]
import numpy as np
import torch

import oracle
import paper_2011_11134_b200 as dgal
from test_gpu_paired import _near_coincident_boxes

dev = torch.device("cuda:0")
out = {}
for dims in (2, 3):
    for scale in (1e-6, 1e-5, 1e-4, 1e-3, 1e-2):
        n = 40_000
        b1, b2 = _near_coincident_boxes(n, scale, seed=60 + dims + int(-math.log10(scale)))
        rng = np.random.default_rng(dims)
        if dims == 3:
            z = rng.normal(-1, 0.4, n); d = rng.uniform(1.4, 1.9, n)
            dz = scale * rng.normal(size=n) + 0.05 * rng.uniform(0.5, 1, n)
            b1 = np.concatenate([b1[:2], z[None], b1[2:4], d[None], b1[4:]]).astype(np.float32)
            b2 = np.concatenate([b2[:2], (z + dz)[None], b2[2:4], d[None], b2[4:]]).astype(np.float32)
        g = rng.uniform(-1, 1, n).astype(np.float32)
        B1, B2 = torch.from_numpy(np.ascontiguousarray(b1)).to(dev), torch.from_numpy(np.ascontiguousarray(b2)).to(dev)
        _, nx, xf = dgal.box_iou_paired_fwd(B1, B2)
        gs1, gs2 = dgal.box_iou_paired_bwd(B1, B2, torch.from_numpy(g).to(dev), nx, xf)
        iou, g1, g2 = dgal.box_iou_paired_fused(B1, B2, grad=torch.from_numpy(g).to(dev))
        ref = oracle.box_iou_paired(b1.T.astype(np.float64), b2.T.astype(np.float64), g.astype(np.float64))
        same = (nx.cpu().numpy() == ref["nx"]) & np.all(xf.cpu().numpy() == ref["xflags"], 1)
        G = np.concatenate([g1.cpu().numpy().T, g2.cpu().numpy().T], 1).astype(np.float64)
        S = np.concatenate([gs1.cpu().numpy().T, gs2.cpu().numpy().T], 1).astype(np.float64)
        R = np.concatenate([ref["gb1"], ref["gb2"]], 1)
        badf = ((np.abs(G - R) > 1e-4) & (np.abs(G - R) > 1e-3 * np.abs(R))).any(1) & same
        bads = ((np.abs(S - R) > 1e-4) & (np.abs(S - R) > 1e-3 * np.abs(R))).any(1) & same
        idx = np.nonzero(badf)[0]
        print(f"dims {dims} scale {scale:.0e}: fused bad {badf.sum()} split bad {bads.sum()} idx {idx[:8]}", flush=True)
        for k in idx[:3]:
            print("   ", k, "max err", np.abs(G[k] - R[k]).max(), "split err", np.abs(S[k] - R[k]).max(),
                  [hex(v) for v in xf[k].cpu().numpy()])
        key = f"d{dims}s{int(-math.log10(scale))}"
        out[key + "_b1"] = b1[:, idx]; out[key + "_b2"] = b2[:, idx]; out[key + "_g"] = g[idx]
        out[key + "_G"] = G[idx]; out[key + "_R"] = R[idx]; out[key + "_S"] = S[idx]
np.savez(os.path.join(ROOT, "gpurun_out", "box_fused_dump.npz"), **out)
