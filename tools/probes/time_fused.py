"""Probe: CUDA-event time of the fused loss kernels (+ refine pass) on the bench
workloads (cfg3 polygons 2^24, cfg4 octagons 2^22, boxes 2D/3D 2^24)."""
import os
import sys

sys.path[:0] = [os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))]
import torch

import paper_2011_11134_b200 as dgal
import synth

dev = torch.device("cuda:0")
reps = int(os.environ.get("REPS", 20))


def timeit(f):
    for _ in range(3):
        f()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        f()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


for cfg, n in ((3, 1 << 24), (4, 1 << 22)):
    bt = synth.gen_config(cfg, n)
    K = bt.p1.K
    X = [torch.from_numpy(a.reshape(n, K)).to(dev) for a in (bt.p1.x, bt.p1.y, bt.p2.x, bt.p2.y)]
    out = (torch.empty(n, device=dev), *(torch.empty((n, K), device=dev) for _ in range(4)))
    o2 = (torch.empty(n, device=dev), torch.empty(n, dtype=torch.uint8, device=dev),
          torch.empty((n, 2 * K), dtype=torch.uint8, device=dev))
    g = torch.full((n,), -1.0 / n, device=dev)
    print(f"cfg{cfg} fused {timeit(lambda: dgal.iou_paired_fused(*X, scale=-1.0 / n, out=out)):.4f} ms  "
          f"fwd {timeit(lambda: dgal.iou_paired_fwd(*X, out=o2)):.4f} ms  "
          f"bwd {timeit(lambda: dgal.iou_paired_bwd(*X, g, o2[1], o2[2], out=out[1:])):.4f} ms", flush=True)
    del X, out, o2
for dims in (2, 3):
    n = 1 << 24
    b = synth.gen_box_pairs(n, dims, seed=synth.seed_for(3) + 101 * dims)
    B1, B2 = torch.from_numpy(b.b1).to(dev), torch.from_numpy(b.b2).to(dev)
    uo = (torch.empty(n, device=dev), torch.empty_like(B1), torch.empty_like(B2))
    fo = (torch.empty(n, device=dev), torch.empty(n, dtype=torch.uint8, device=dev),
          torch.empty((n, 8), dtype=torch.uint8, device=dev))
    go = (torch.empty_like(B1), torch.empty_like(B2))
    g = torch.full((n,), -1.0 / n, device=dev)
    print(f"box{dims}d fused {timeit(lambda: dgal.box_iou_paired_fused(B1, B2, scale=-1.0 / n, out=uo)):.4f} ms  "
          f"fwd {timeit(lambda: dgal.box_iou_paired_fwd(B1, B2, out=fo)):.4f} ms  "
          f"bwd {timeit(lambda: dgal.box_iou_paired_bwd(B1, B2, g, fo[1], fo[2], out=go)):.4f} ms", flush=True)
