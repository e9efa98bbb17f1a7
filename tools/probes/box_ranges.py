"""Probe: box IoU vs the oracle under a common offset of the centres (m) and a common
scale of the sizes, 2^16 KITTI pairs each: max |IoU - oracle| and the count above 1e-5."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.getcwd())
import oracle  # noqa: E402
import paper_2011_11134_b200 as dgal  # noqa: E402
import synth  # noqa: E402

dev = torch.device("cuda:0")
for dims in (2, 3):
    for off in (0.0, 1e3, 1e4):
        for sc in (0.05, 1.0, 20.0):
            b = synth.gen_box_pairs(1 << 16, dims, seed=7)
            sz = (2, 3) if dims == 2 else (3, 4, 5)
            for bb in (b.b1, b.b2):
                bb[0] += np.float32(off)
                bb[1] -= np.float32(off)
                bb[0] = (bb[0] - np.float32(off)) * np.float32(sc) + np.float32(off) if sc != 1.0 else bb[0]
                bb[1] = (bb[1] + np.float32(off)) * np.float32(sc) - np.float32(off) if sc != 1.0 else bb[1]
                for r in sz:
                    bb[r] *= np.float32(sc)
                if dims == 3:
                    bb[2] *= np.float32(sc)
            r1, r2 = b.rows64()
            ref = oracle.box_iou_paired(r1, r2, b.grad.astype(np.float64))
            iou, nx, xf = dgal.box_iou_paired_fwd(torch.from_numpy(b.b1).to(dev), torch.from_numpy(b.b2).to(dev))
            e = np.abs(iou.cpu().numpy().astype(np.float64) - ref["iou"])
            print(dims, off, sc, f"max {e.max():.3e} n>1e-5 {(e > 1e-5).sum()}", flush=True)
