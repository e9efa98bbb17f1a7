"""How the per-kernel split of the cfg3 step depends on the measuring method: the step loop
(two alternating input sets), events around each launch, the step loop again, and
back-to-back runs of one kernel over the alternating sets with per-set outputs.
python tools/probes/time_split.py"""
import os
import sys

sys.path[:0] = [os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))]
import torch

import paper_2011_11134_b200 as dgal
import synth

dev = torch.device("cuda:0")
n = 1 << 24
b = synth.gen_config(3, n)
T = lambda a: torch.from_numpy(a.reshape(n, 4)).to(dev)  # noqa: E731
sets = [(T(b.p1.x), T(b.p1.y), T(b.p2.x), T(b.p2.y))]
sets.append(tuple(t.clone() for t in sets[0]))
g = torch.full((n,), -1.0 / n, device=dev)
outs = [dgal.iou_paired_fwd(*s) for s in sets]
grads = [dgal.iou_paired_bwd(*s, g, o[1], o[2]) for s, o in zip(sets, outs)]
E = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731
S = 50


def loop(fn):
    for s in range(5):
        fn(s)
    torch.cuda.synchronize()
    a, z = E(), E()
    a.record()
    for s in range(S):
        fn(s)
    z.record()
    torch.cuda.synchronize()
    return a.elapsed_time(z) / S


def step(s):
    o = outs[s % 2]
    dgal.iou_paired_fwd(*sets[s % 2], out=o)
    dgal.iou_paired_bwd(*sets[s % 2], g, o[1], o[2], out=grads[s % 2])


res = {"step": loop(step)}
ev = [tuple(E() for _ in range(3)) for _ in range(S)]
for s in range(S):
    o = outs[s % 2]
    ev[s][0].record()
    dgal.iou_paired_fwd(*sets[s % 2], out=o)
    ev[s][1].record()
    dgal.iou_paired_bwd(*sets[s % 2], g, o[1], o[2], out=grads[s % 2])
    ev[s][2].record()
torch.cuda.synchronize()
res["bracket_fwd"] = sum(a.elapsed_time(b) for a, b, _ in ev) / S
res["bracket_bwd"] = sum(b.elapsed_time(c) for _, b, c in ev) / S
res["step_again"] = loop(step)
res["fwd_only"] = loop(lambda s: dgal.iou_paired_fwd(*sets[s % 2], out=outs[s % 2]))
res["bwd_only"] = loop(lambda s: dgal.iou_paired_bwd(*sets[s % 2], g, outs[s % 2][1], outs[s % 2][2],
                                                      out=grads[s % 2]))
res["fwd_same"] = loop(lambda s: dgal.iou_paired_fwd(*sets[0], out=outs[0]))
print({k: round(v, 4) for k, v in res.items()}, flush=True)
