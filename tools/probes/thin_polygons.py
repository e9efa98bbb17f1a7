"""Probe: IoU / gradient error of the device paths vs the oracle on thin / sliver
polygons (synth.gen_thin_pairs: aspect 10..300, scene coordinates to +-354 m).
Per (K, verts, aspect): max |IoU - oracle| and the count above 1e-5 for the split
forward, the fused kernel and the pairwise diagonal; gradient out-of-tolerance
fraction (split, fused) on margin pairs."""
import os
import sys

sys.path[:0] = [os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))]
import numpy as np
import torch

import oracle
import paper_2011_11134_b200 as dgal
import synth

dev = torch.device("cuda:0")
n = int(os.environ.get("THIN_N", 20000))
for K, verts in ((4, 3), (4, 4), (8, 8), (8, 5)):
    for aspect in (10.0, 30.0, 100.0, 300.0):
        b = synth.gen_thin_pairs(n, K, verts, aspect)
        X = [torch.from_numpy(a.reshape(n, K)).to(dev) for a in (b.p1.x, b.p1.y, b.p2.x, b.p2.y)]
        iou, nx, xf = dgal.iou_paired_fwd(*X)
        g = torch.from_numpy(b.grad).to(dev)
        gs = dgal.iou_paired_bwd(*X, g, nx, xf)
        fu = dgal.iou_paired_fused(*X, grad=g)
        m = 2048
        pw = dgal.iou_pairwise(*[t[:m].contiguous() for t in X], want_mask=False)[0].diagonal()
        un = lambda a: a.reshape(n, K)[:, :verts].astype(np.float64)  # noqa: E731
        p1, p2 = (un(b.p1.x), un(b.p1.y)), (un(b.p2.x), un(b.p2.y))
        ref = oracle.iou_paired_fwd(p1, p2)
        ok = oracle.margin_ok(p1, p2)
        rg = oracle.iou_paired_bwd(p1, p2, b.grad)
        out = []
        for name, v in (("fwd", iou), ("fused", fu[0]), ("pw", pw)):
            v = v.cpu().numpy().astype(np.float64)
            e = np.abs(v - ref["iou"][:v.size])
            out.append(f"{name} max {e.max():.1e} >1e-5 {int((e > 1e-5).sum())}")
        for name, gr in (("split", gs), ("fused", fu[1:])):
            bad = np.zeros(n, bool)
            for got, want in zip(gr, rg):
                got = got.cpu().numpy().astype(np.float64)
                fold = got[:, :verts].copy()
                fold[:, verts - 1] += got[:, verts:].sum(1)
                bad |= ((np.abs(fold - want) > 1e-4) & (np.abs(fold - want) > 1e-3 * np.abs(want))).any(1)
            out.append(f"g{name} bad(margin) {int(bad[ok].sum())}/{int(ok.sum())}")
        nz = (ref["iou"] > 0).mean()
        print(f"K={K} verts={verts} aspect={aspect:>5.0f} overlap {nz:.2f} | " + " | ".join(out), flush=True)
