"""Probe: dump the thin-polygon pairs (synth.gen_thin_pairs) whose device IoU or
split-path gradient is out of tolerance, with the device's nx / xflags, to
gpurun_out/thin_dump.npz for offline study (tools/emu_clip.py)."""
import os
import sys

sys.path[:0] = [os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))]
import numpy as np
import torch

import oracle
import paper_2011_11134_b200 as dgal
import synth

dev = torch.device("cuda:0")
n = 20000
out = {}
for K, verts, aspect in ((4, 3, 100.0), (4, 3, 300.0), (4, 4, 100.0), (4, 4, 300.0)):
    b = synth.gen_thin_pairs(n, K, verts, aspect)
    X = [torch.from_numpy(a.reshape(n, K)).to(dev) for a in (b.p1.x, b.p1.y, b.p2.x, b.p2.y)]
    iou, nx, xf = dgal.iou_paired_fwd(*X)
    g = torch.from_numpy(b.grad).to(dev)
    gr = dgal.iou_paired_bwd(*X, g, nx, xf)
    un = lambda a: a.reshape(n, K)[:, :verts].astype(np.float64)  # noqa: E731
    p1, p2 = (un(b.p1.x), un(b.p1.y)), (un(b.p2.x), un(b.p2.y))
    ref = oracle.iou_paired_fwd(p1, p2)
    rg = oracle.iou_paired_bwd(p1, p2, b.grad)
    ok = oracle.margin_ok(p1, p2)
    e = np.abs(iou.cpu().numpy() - ref["iou"])
    bad = e > 1e-5
    gbad = np.zeros(n, bool)
    G = []
    for got, want in zip(gr, rg):
        got = got.cpu().numpy().astype(np.float64)
        f = got[:, :verts].copy()
        f[:, verts - 1] += got[:, verts:].sum(1)
        G.append(f)
        d = np.abs(f - want)
        gbad |= ((d > 1e-4) & (d > 1e-3 * np.abs(want))).any(1) & ok
    idx = np.nonzero(bad | gbad)[0]
    key = f"K{K}v{verts}a{int(aspect)}"
    print(key, "iou bad", np.nonzero(bad)[0][:10], "grad bad", np.nonzero(gbad)[0][:10])
    for k in idx[:10]:
        print("  ", k, "iou", iou[k].item(), ref["iou"][k], "nx", nx[k].item(), ref["nx"][k],
              [hex(v) for v in xf[k].cpu().numpy()], [hex(v) for v in ref["xflags"][k]], "margin", ok[k])
    out[key + "_idx"] = idx
    out[key + "_x"] = np.stack([a.reshape(n, K)[idx] for a in (b.p1.x, b.p1.y, b.p2.x, b.p2.y)])
    out[key + "_g"] = b.grad[idx]
    out[key + "_nx"] = nx.cpu().numpy()[idx]
    out[key + "_xf"] = xf.cpu().numpy()[idx]
    out[key + "_iou"] = iou.cpu().numpy()[idx]
    out[key + "_grad"] = np.stack([gg[idx] for gg in G])
os.makedirs("gpurun_out", exist_ok=True)
np.savez("gpurun_out/thin_dump.npz", **out)
