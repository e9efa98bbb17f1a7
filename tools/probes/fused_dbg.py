import os, sys
sys.path[:0] = ['/root/repo']
import numpy as np, torch, oracle, paper_2011_11134_b200 as dgal
dev = torch.device("cuda:0")
n = 20000; scale = 1e-4
rng = np.random.default_rng(4)
cx = rng.uniform(0, 70, n); cy = rng.uniform(-40, 40, n)
w = rng.uniform(0.5, 5, n); h = rng.uniform(0.5, 2, n); th = rng.uniform(-np.pi, np.pi, n)
b1 = np.stack([cx, cy, w, h, th]).astype(np.float32)
pert = rng.normal(size=(5, n)) * scale * np.array([w, w, w, h, np.ones(n)])
b2 = (b1.astype(np.float64) + pert).astype(np.float32)
x1, y1 = oracle.box_corners(b1.T.astype(np.float64)); x2, y2 = oracle.box_corners(b2.T.astype(np.float64))
x1, y1, x2, y2 = (a.astype(np.float32) for a in (x1, y1, x2, y2))
g = np.ones(n, np.float32)
T = lambda a: torch.from_numpy(a).to(dev)
X = (T(x1), T(y1), T(x2), T(y2))
iou, nx, xf = dgal.iou_paired_fwd(*X)
gs = [t.cpu().numpy() for t in dgal.iou_paired_bwd(*X, T(g), nx, xf)]
fu = dgal.iou_paired_fused(*X, grad=T(g))
fi = fu[0].cpu().numpy(); gf = [t.cpu().numpy() for t in fu[1:]]
ref = oracle.iou_paired_bwd((x1, y1), (x2, y2), g)
R = np.concatenate(ref, 1); S = np.concatenate(gs, 1); F = np.concatenate(gf, 1)
den = np.maximum(1, np.abs(R).max(1))
es = np.abs(S - R).max(1) / den; ef = np.abs(F - R).max(1) / den
rf = oracle.iou_paired_fwd((x1, y1), (x2, y2))
same = (nx.cpu().numpy() == rf["nx"]) & np.all(xf.cpu().numpy() == rf["xflags"], 1)
ef = np.where(same, ef, 0); es = np.where(same, es, 0)
k = int(np.argmax(ef))
np.set_printoptions(precision=6, linewidth=200, suppress=True)
print("worst fused pair", k, "ef", ef[k], "es", es[k], "iou", iou[k].item(), fi[k], "nx", nx[k].item(), [hex(b) for b in xf[k].cpu().numpy()])
print("oracle", R[k]); print("split ", S[k]); print("fused ", F[k])
print("P", np.stack([x1[k], y1[k]], 1).tolist()); print("Q", np.stack([x2[k], y2[k]], 1).tolist())
print("count ef>1e-4", (ef > 1e-4).sum(), "es>1e-4", (es > 1e-4).sum())
order = np.argsort(-ef)[:6]
for k in order:
    print(k, "ef", ef[k], "nx", nx[k].item(), [hex(b) for b in xf[k].cpu().numpy()[:nx[k].item()]], "iou", iou[k].item())
    print("   dF", (F[k]-R[k]).round(6))
