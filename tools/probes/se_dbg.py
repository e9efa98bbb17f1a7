import os, sys, numpy as np, torch
sys.path.insert(0, os.getcwd())
import oracle, paper_2011_11134_b200 as dgal, synth
dev = torch.device("cuda:0")
K = 8
b = synth.gen_config(4, 8192)
x, y = b.p1.x.reshape(-1, K), b.p1.y.reshape(-1, K)
mx, my = 0.5 * (x[:, :1] + x[:, 1:2]), 0.5 * (y[:, :1] + y[:, 1:2])
x2, y2 = x.copy(), y.copy()
x2[:, 2:] = mx + 0.5 * (x[:, 2:] - mx); y2[:, 2:] = my + 0.5 * (y[:, 2:] - my)
X = [torch.from_numpy(np.ascontiguousarray(a.astype(np.float32))).to(dev) for a in (x, y, x2, y2)]
iou, nx, xf = dgal.iou_paired_fwd(*X)
p1 = (x.astype(np.float64), y.astype(np.float64)); p2 = (x2.astype(np.float64), y2.astype(np.float64))
ref = oracle.iou_paired_fwd(p1, p2)
sh = oracle.sh_intersect(p1, p2) if hasattr(oracle, 'sh_intersect') else None
A = lambda X_, Y_: 0.5 * np.sum(X_ * np.roll(Y_, -1, 1) - np.roll(X_, -1, 1) * Y_, 1)
A1, A2 = A(*p1), A(*p2)
g = iou.cpu().numpy(); e = np.abs(g - ref["iou"])
bad = np.nonzero(e > 1e-5)[0]
print("bad", bad.size, "A2/A1 vs gpu max", np.abs(A2/A1 - g).max(), "A2/A1 vs oracle max", np.abs(A2/A1 - ref["iou"]).max())
for k in bad[:3]:
    print(k, "gpu", g[k], nx[k].item(), xf[k][:nx[k]].tolist(), "ora", ref["iou"][k], ref["nx"][k], ref["xflags"][k][:ref["nx"][k]].tolist(), "A2/A1", A2[k]/A1[k])
    if sh is not None: print("   sh", {kk: (v[k] if hasattr(v,'__getitem__') else v) for kk, v in sh.items()} if isinstance(sh, dict) else sh)
