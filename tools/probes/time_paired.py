"""Time the paired kernels of the loaded libdgal (DGAL_SO selects a build) on the
cfg3 / cfg4 inputs: python tools/probes/time_paired.py [label]."""
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
    try:
        uo = dgal.iou_paired_fused(*pl, scale=-1.0 / n)
    except Exception:   # a build with another fused ABI (A/B of older builds)
        uo = None
    E = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731
    for name, fn in (("fwd", lambda: dgal.iou_paired_fwd(*pl, out=fo)),
                     ("bwd", lambda: dgal.iou_paired_bwd(*pl, g, fo[1], fo[2], out=go)),
                     ("fused", lambda: dgal.iou_paired_fused(*pl, scale=-1.0 / n, out=uo))):
        if name == "fused" and uo is None:
            continue
        for _ in range(5):
            fn()
        a, z = E(), E()
        a.record()
        for _ in range(50):
            fn()
        z.record()
        torch.cuda.synchronize()
        res[f"cfg{cfg}_{name}"] = round(a.elapsed_time(z) / 50, 4)
print(label, res, flush=True)
