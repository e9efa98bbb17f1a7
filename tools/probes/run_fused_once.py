"""One warm-up + one profiled launch of the fused loss kernel (+ refine pass) on the
cfg3 batch (2^24 pairs), for ncu captures (-k regex -s 2 skips the warm-up)."""
import os
import sys

sys.path[:0] = [os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))]
import torch

import paper_2011_11134_b200 as dgal
import synth

dev = torch.device("cuda:0")
n = 1 << 24
b = synth.gen_config(3, n)
X = [torch.from_numpy(a.reshape(n, 4)).to(dev) for a in (b.p1.x, b.p1.y, b.p2.x, b.p2.y)]
for _ in range(2):
    dgal.iou_paired_fused(*X, scale=-1.0 / n)
torch.cuda.synchronize()
