"""Alternating fwd + bwd steps (the bench's cfg3 / cfg4 step) of the loaded libdgal
(DGAL_SO selects a build): ms per step and the standalone kernel times beside it.
    python tools/probes/time_step.py [label]"""
import os
import sys

sys.path[:0] = [os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))]
import torch

import paper_2011_11134_b200 as dgal
import synth

label = sys.argv[1] if len(sys.argv) > 1 else os.environ.get("DGAL_SO", "libdgal.so")
dev = torch.device("cuda:0")
res = {}
for cfg, n in ((3, 1 << 24), (4, 1 << 22)):
    b = synth.gen_config(cfg, n)
    K = b.p1.K
    T = lambda a: torch.from_numpy(a.reshape(n, K)).to(dev)  # noqa: E731
    pl = (T(b.p1.x), T(b.p1.y), T(b.p2.x), T(b.p2.y))
    g = torch.full((n,), -1.0 / n, device=dev)
    fo = dgal.iou_paired_fwd(*pl)
    go = dgal.iou_paired_bwd(*pl, g, fo[1], fo[2])
    E = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731
    for _ in range(5):
        dgal.iou_paired_fwd(*pl, out=fo)
        dgal.iou_paired_bwd(*pl, g, fo[1], fo[2], out=go)
    a, z = E(), E()
    a.record()
    for _ in range(50):
        dgal.iou_paired_fwd(*pl, out=fo)
        dgal.iou_paired_bwd(*pl, g, fo[1], fo[2], out=go)
    z.record()
    torch.cuda.synchronize()
    res[f"cfg{cfg}_step"] = round(a.elapsed_time(z) / 50, 4)
for dims in (2, 3):
    bb = synth.gen_box_pairs(1 << 24, dims)
    n = bb.n
    B1, B2 = torch.from_numpy(bb.b1).to(dev), torch.from_numpy(bb.b2).to(dev)
    g = torch.full((n,), -1.0 / n, device=dev)
    fo = dgal.box_iou_paired_fwd(B1, B2)
    go = dgal.box_iou_paired_bwd(B1, B2, g, fo[1], fo[2])
    for _ in range(5):
        dgal.box_iou_paired_fwd(B1, B2, out=fo)
        dgal.box_iou_paired_bwd(B1, B2, g, fo[1], fo[2], out=go)
    a, z = E(), E()
    a.record()
    for _ in range(30):
        dgal.box_iou_paired_fwd(B1, B2, out=fo)
        dgal.box_iou_paired_bwd(B1, B2, g, fo[1], fo[2], out=go)
    z.record()
    torch.cuda.synchronize()
    res[f"box{dims}_step"] = round(a.elapsed_time(z) / 30, 4)
    del B1, B2, g, fo, go
print(label, res, flush=True)
