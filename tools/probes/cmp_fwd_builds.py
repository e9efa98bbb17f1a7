"""Forward outputs (cfg3 prefix + box worked examples) of the loaded build (DGAL_SO) -> npz,
for bitwise A/B of two builds with tools/probes/cmp_fwd_npz.py."""
import os, sys, numpy as np, torch, math
sys.path.insert(0, os.getcwd())
import paper_2011_11134_b200 as dgal, synth
dev = torch.device("cuda:0")
out = {}
b = synth.gen_config(3, 1 << 16)
T = lambda a: torch.from_numpy(a.reshape(-1, 4)).to(dev)
iou, nx, xf = dgal.iou_paired_fwd(T(b.p1.x), T(b.p1.y), T(b.p2.x), T(b.p2.y))
out["iou"], out["nx"], out["xf"] = iou.cpu().numpy(), nx.cpu().numpy(), xf.cpu().numpy()
rows = np.array([[0, 0, 2, 2, 0], [3, -2, 4, 1.5, 0.4]], np.float32).T.copy()
rows2 = np.array([[0, 0, 2, 2, math.pi / 4], [3, -2, 4, 1.5, 0.4]], np.float32).T.copy()
bi, bn, bx = dgal.box_iou_paired_fwd(torch.from_numpy(rows).to(dev), torch.from_numpy(rows2).to(dev))
out["biou"], out["bnx"], out["bxf"] = bi.cpu().numpy(), bn.cpu().numpy(), bx.cpu().numpy()
np.savez(sys.argv[1], **out)
