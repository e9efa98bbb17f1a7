"""Time the box kernels of the loaded libdgal (DGAL_SO selects a build) on the
2^24-pair KITTI box inputs (2D and 3D): python tools/probes/time_box.py [label]."""
import os
import sys

sys.path[:0] = [os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))]
import torch

import paper_2011_11134_b200 as dgal
import synth

label = sys.argv[1] if len(sys.argv) > 1 else os.environ.get("DGAL_SO", "libdgal.so")
dev = torch.device("cuda:0")
res = {}
for dims in (2, 3):
    b = synth.gen_box_pairs(1 << 24, dims)
    n = b.n
    B1, B2 = torch.from_numpy(b.b1).to(dev), torch.from_numpy(b.b2).to(dev)
    g = torch.full((n,), -1.0 / n, device=dev)
    fo = dgal.box_iou_paired_fwd(B1, B2)
    E = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731
    for name, fn in (("fwd", lambda: dgal.box_iou_paired_fwd(B1, B2)),
                     ("bwd", lambda: dgal.box_iou_paired_bwd(B1, B2, g, fo[1], fo[2])),
                     ("fused", lambda: dgal.box_iou_paired_fused(B1, B2, scale=-1.0 / n))):
        for _ in range(5):
            fn()
        a, z = E(), E()
        a.record()
        for _ in range(30):
            fn()
        z.record()
        torch.cuda.synchronize()
        res[f"box{dims}_{name}"] = round(a.elapsed_time(z) / 30, 4)
print(label, res, flush=True)
