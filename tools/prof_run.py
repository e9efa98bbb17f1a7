#!/usr/bin/env python
"""One launch of every hot kernel at BASELINE sizes, for ncu captures:
cfg3 paired fwd+bwd (K=4, 2^24), cfg4 paired fwd+bwd (K=8, 2^22), box (2D and 3D
box fwd/bwd/fused, 2^24 pairs), cfg5 pairwise 100k x 100k (+ mask + lists) and
the NMS keep.  Each is run twice (the second
launch is the one to profile: -s skips the first), once with --once."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2011_11134_b200 as dgal  # noqa: E402
import synth  # noqa: E402


def main():
    dev = torch.device("cuda:0")
    args = sys.argv[1:]
    reps = 1 if "--once" in args else 2
    which = [a for a in args if a != "--once"] or ["cfg3", "cfg4", "box", "cfg5"]
    for cfg in (3, 4):
        if f"cfg{cfg}" not in which:
            continue
        b = synth.gen_config(cfg)
        n, K = b.n, b.p1.K
        T = lambda a: torch.from_numpy(a.reshape(n, K)).to(dev)  # noqa: E731
        x1, y1, x2, y2 = T(b.p1.x), T(b.p1.y), T(b.p2.x), T(b.p2.y)
        g = torch.full((n,), -1.0 / n, device=dev)
        for _ in range(reps):
            iou, nx, xf = dgal.iou_paired_fwd(x1, y1, x2, y2)
            dgal.iou_paired_bwd(x1, y1, x2, y2, g, nx, xf)
            dgal.iou_paired_fused(x1, y1, x2, y2, scale=-1.0 / n)
        torch.cuda.synchronize()
        del x1, y1, x2, y2, g, iou, nx, xf
    if "box" in which:
        for dims in (2, 3):
            b = synth.gen_box_pairs(1 << 24, dims)
            n = b.n
            B1, B2 = torch.from_numpy(b.b1).to(dev), torch.from_numpy(b.b2).to(dev)
            g = torch.full((n,), -1.0 / n, device=dev)
            for _ in range(reps):
                iou, nx, xf = dgal.box_iou_paired_fwd(B1, B2)
                dgal.box_iou_paired_bwd(B1, B2, g, nx, xf)
                dgal.box_iou_paired_fused(B1, B2, scale=-1.0 / n)
            torch.cuda.synchronize()
            del B1, B2, g, iou, nx, xf
    if "cfg5" in which:
        sc = synth.gen_cfg5_scene()
        n = sc.polys.n
        x = torch.from_numpy(sc.polys.x.reshape(n, 4)).to(dev)
        y = torch.from_numpy(sc.polys.y.reshape(n, 4)).to(dev)
        for _ in range(reps):
            iou, mask, cnt, idx = dgal.iou_pairwise(x, y, x, y, thr=sc.thr, nbr_cap=64)
            keep = dgal.nms_keep(mask, cnt, idx)
            torch.cuda.synchronize()
            del iou
        print("kept", int(keep.sum()))
    torch.cuda.synchronize()
    print("ok")


if __name__ == "__main__":
    main()
