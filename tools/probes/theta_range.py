import sys, os, numpy as np, torch
sys.path.insert(0, os.getcwd())
import paper_2011_11134_b200 as dgal, synth, oracle
dev = torch.device("cuda:0")
for dims in (2, 3):
    for R in (math_r for math_r in (3.2, 10.0, 30.0, 100.0, 1000.0)):
        b = synth.gen_box_pairs(1 << 16, dims, seed=99)
        rng = np.random.default_rng(5)
        sh = rng.uniform(-R, R, b.n).astype(np.float32)
        th_i = 4 if dims == 2 else 6
        b.b1[th_i] += sh; b.b2[th_i] += sh
        r1, r2 = b.rows64()
        ref = oracle.box_iou_paired(r1, r2, b.grad.astype(np.float64))
        iou, nx, xf = dgal.box_iou_paired_fwd(torch.from_numpy(b.b1).to(dev), torch.from_numpy(b.b2).to(dev))
        e = np.abs(iou.cpu().numpy().astype(np.float64) - ref["iou"])
        print(dims, R, "max", e.max(), "n>1e-5", (e > 1e-5).sum(), flush=True)
