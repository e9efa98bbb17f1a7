#!/usr/bin/env python
"""Small invocations of every kernel for compute-sanitizer (memcheck / racecheck /
synccheck / initcheck, one tool per run): ragged sizes so tails, bulk-copy tiles,
queues and the indexed pairwise grid are all exercised."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2011_11134_b200 as dgal  # noqa: E402
import synth  # noqa: E402


def main():
    dev = torch.device("cuda:0")
    for cfg, n in ((3, 256 * 9 + 37), (4, 256 * 5 + 3)):
        b = synth.gen_config(cfg, n)
        K = b.p1.K
        T = lambda a: torch.from_numpy(a.reshape(n, K)).to(dev)  # noqa: E731
        x1, y1, x2, y2 = T(b.p1.x), T(b.p1.y), T(b.p2.x), T(b.p2.y)
        g = torch.from_numpy(b.grad).to(dev)
        iou, nx, xf = dgal.iou_paired_fwd(x1, y1, x2, y2)
        dgal.iou_paired_bwd(x1, y1, x2, y2, g, nx, xf)
        gb = torch.empty(n + 1, device=dev)[1:]
        gb.copy_(g)
        dgal.iou_paired_bwd(x1, y1, x2, y2, gb, nx, xf)      # non-bulk path
        dgal.iou_paired_fused(x1, y1, x2, y2, grad=g)
    sc = synth.gen_cfg5_scene(n_objects=61, per_object=50, seed=3)
    n = sc.polys.n
    x = torch.from_numpy(sc.polys.x.reshape(n, 4)).to(dev)
    y = torch.from_numpy(sc.polys.y.reshape(n, 4)).to(dev)
    for indexed in (True, False):
        iou, mask, cnt, idx = dgal.iou_pairwise(x[5:], y[5:], x, y, row_offset=5, thr=0.5, nbr_cap=4,
                                                indexed=indexed)
    _, mask, cnt, idx = dgal.iou_pairwise(x, y, x, y, thr=0.5, nbr_cap=4)
    keep = dgal.nms_keep(mask, cnt, idx)
    st = torch.zeros(n, dtype=torch.uint8, device=dev)
    und = torch.zeros(1, dtype=torch.int32, device=dev)
    dgal.nms_round(n, 0, mask, cnt, idx, st, und)
    torch.cuda.synchronize()
    print("ok", int(keep.sum()))


if __name__ == "__main__":
    main()
