"""GPU parity on thin / sliver polygons (§V: "improve the numerical stability
... arbitrary shape input"; north_star tolerances): synth.gen_thin_pairs, aspect
30-1000, scene coordinates up to +-354 m, padded triangles / quads for K=4 and
octagon / pentagon slivers for K=8.  The float area sum of such pairs is
ill-conditioned (~eps R^2 against an area ~R^2 / aspect); the kernels detect them
(R^2 > kThinRatio A_u) and redo the record and its area in double (record_exact,
csrc/dgal_core.cuh; areas_exact, csrc/dgal_exact.cuh).  IoU is compared on EVERY pair (R18), flags and vertex
gradients on the margin pairs (R13); padded vertices' gradients are folded onto
the last real vertex (include/dgal.h)."""
import numpy as np
import pytest
import torch

import oracle
import paper_2011_11134_b200 as dgal
import synth
from gpu_util import assert_flags_exact, assert_grad_close, assert_iou_close, dev

pytestmark = pytest.mark.gpu

CASES = [(K, v, a) for K, v in ((4, 3), (4, 4), (8, 8), (8, 5)) for a in (30.0, 100.0, 300.0, 1000.0)]
N = 20000


def _case(K, verts, aspect):
    b = synth.gen_thin_pairs(N, K, verts, aspect)
    X = [torch.from_numpy(a.reshape(N, K)).to(dev()) for a in (b.p1.x, b.p1.y, b.p2.x, b.p2.y)]
    un = lambda a: a.reshape(N, K)[:, :verts].astype(np.float64)  # noqa: E731
    p1, p2 = (un(b.p1.x), un(b.p1.y)), (un(b.p2.x), un(b.p2.y))
    return b, X, p1, p2


def _fold(g, verts):
    g = g.cpu().numpy().astype(np.float64)
    f = g[:, :verts].copy()
    f[:, verts - 1] += g[:, verts:].sum(1)
    return f


@pytest.mark.parametrize("K,verts,aspect", CASES)
def test_thin_split_path(K, verts, aspect):
    b, X, p1, p2 = _case(K, verts, aspect)
    iou, nx, xf = dgal.iou_paired_fwd(*X)
    g = torch.from_numpy(b.grad).to(dev())
    gr = dgal.iou_paired_bwd(*X, g, nx, xf)
    ref = oracle.iou_paired_fwd(p1, p2)
    assert (ref["iou"] > 0).mean() > 0.85             # the workload does overlap
    assert_iou_close(iou.cpu().numpy(), ref["iou"])
    ok = oracle.margin_ok(p1, p2)
    assert ok.mean() > (0.5 if aspect < 1000 else 0.3)   # enough margin pairs to compare flags / gradients
    # flags of the padded polygons: indices of the real vertices / edges are the same
    # (the repeated vertex's zero-length edge never carries a crossing)
    nxk = nx.cpu().numpy()
    xfk = xf.cpu().numpy()
    if verts == K:
        assert_flags_exact(nxk[ok], xfk[ok], {"nx": ref["nx"][ok], "xflags": ref["xflags"][ok]})
    rg = oracle.iou_paired_bwd(p1, p2, b.grad)
    for got, want in zip(gr, rg):
        assert_grad_close(_fold(got, verts)[ok], want[ok])


@pytest.mark.parametrize("K,verts,aspect", CASES)
def test_thin_fused(K, verts, aspect):
    b, X, p1, p2 = _case(K, verts, aspect)
    g = torch.from_numpy(b.grad).to(dev())
    iou, *gr = dgal.iou_paired_fused(*X, grad=g)
    ref = oracle.iou_paired_fwd(p1, p2)
    assert_iou_close(iou.cpu().numpy(), ref["iou"])
    ok = oracle.margin_ok(p1, p2)
    rg = oracle.iou_paired_bwd(p1, p2, b.grad)
    for got, want in zip(gr, rg):
        assert_grad_close(_fold(got, verts)[ok], want[ok])


@pytest.mark.parametrize("K,verts,aspect", [(4, 3, 300.0), (4, 4, 300.0), (8, 8, 300.0), (8, 5, 300.0),
                                            (4, 3, 100.0), (8, 5, 100.0)])
@pytest.mark.parametrize("indexed", [True, False])
def test_thin_pairwise(K, verts, aspect, indexed):
    """The pairwise evaluators (grid-indexed and tiled): rows = the thin p1 of 1024
    pairs, columns = their p2 — the full 1024 x 1024 matrix against the oracle at
    1e-5 (thin candidates recomputed from the recorded intersection in double)."""
    b, X, p1, p2 = _case(K, verts, aspect)
    m = 1024
    x1, y1, x2, y2 = (t[:m].contiguous() for t in X)
    got = dgal.iou_pairwise(x1, y1, x2, y2, want_mask=False, indexed=indexed)[0].cpu().numpy()
    # the oracle on the padded polygons (a repeated vertex is a zero-length edge: same polygon)
    P = synth.Polys(np.ascontiguousarray(b.p1.x.reshape(N, K)[:m].reshape(-1)),
                    np.ascontiguousarray(b.p1.y.reshape(N, K)[:m].reshape(-1)), K)
    Q = synth.Polys(np.ascontiguousarray(b.p2.x.reshape(N, K)[:m].reshape(-1)),
                    np.ascontiguousarray(b.p2.y.reshape(N, K)[:m].reshape(-1)), K)
    ref = oracle.iou_pairwise(P, Q)
    assert (np.diag(ref) > 0).mean() > 0.85
    assert np.abs(got - ref).max() <= 1e-5
