"""GPU parity of the paired forward/backward (dgal_iou_paired_fwd/bwd)
against the CPU oracle, through the C ABI.  Tolerances are the north_star's:
nx/xflags bit-exact on margin inputs, IoU <= 1e-5 abs, vertex gradients <=
1e-4 abs or <= 1e-3 rel."""
import math

import numpy as np
import pytest
import torch

import oracle
import paper_2011_11134_b200 as dgal
import synth
from gpu_util import (assert_flags_exact, assert_grad_close, assert_iou_close,
                      check_paired_against_oracle, dev, gpu_paired, to_dev)
from helpers import box, margin_batch, regular

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("cfg,n", [(1, 1024), (3, 40_000), (4, 20_000)])
def test_paired_margin_inputs_full_compare(cfg, n):
    """Every output element of a margin-filtered batch of the config."""
    check_paired_against_oracle(margin_batch(cfg, n))


def test_general_quads_all_walk_states():
    """Non-rectangular convex quads (synth.gen_quad_pairs): containment both ways,
    runs of up to 3 FromP2 bytes after an exit, up to 8 crossings — the states of
    the K=4 forward's walk tables beyond what box pairs reach.
    Full compare on margin inputs, and the workload must actually reach them."""
    from helpers import margin_filter
    b = margin_filter(synth.gen_quad_pairs(12_000), 8192)
    ref = oracle.iou_paired_fwd(b.p1, b.p2)
    nx, xf = ref["nx"], ref["xflags"].reshape(b.n, 8)
    assert set(np.unique(nx)) >= {0, 3, 4, 5, 6, 7, 8}
    tags = xf >> 6
    runs3 = ((tags[:, :-2] == 2) & (tags[:, 1:-1] == 2) & (tags[:, 2:] == 2)).any(1)
    assert runs3.sum() > 10                                    # 3 FromP2 in a row
    assert ((tags[:, :4] == 2).all(1) & (nx == 4)).sum() > 10  # p2 inside p1
    assert ((tags[:, :4] == 1).all(1) & (nx == 4)).sum() > 10  # p1 inside p2
    check_paired_against_oracle(b)


@pytest.mark.parametrize("n", [1, 2, 31, 255, 257, 1000, 4097])
def test_ragged_sizes(n):
    check_paired_against_oracle(margin_batch(1, n))


@pytest.mark.parametrize("cfg,n", [(3, 127), (3, 1023), (3, 1025), (3, 8193), (4, 1), (4, 129), (4, 511),
                                   (4, 513), (4, 2049)])
def test_ragged_around_cta_chunks(cfg, n):
    """Sizes around the kernels' CTA chunks (forward: 128 threads x 8 tiles for K=4,
    x 4 tiles for K=8, with the cp.async ring; backward: 128-pair tiles x 8 (K=4) or
    the 128-pair producer tiles (K=8)) — the partial last tile and the partial chunk."""
    check_paired_against_oracle(margin_batch(cfg, n))


def _pairs(P_list, Q_list, K):
    P = np.stack(P_list).astype(np.float32)
    Q = np.stack(Q_list).astype(np.float32)
    mk = lambda A: synth.Polys(np.ascontiguousarray(A[..., 0].reshape(-1)),  # noqa: E731
                               np.ascontiguousarray(A[..., 1].reshape(-1)), K)
    g = np.linspace(-1, 1, len(P_list)).astype(np.float32)
    return synth.PairBatch(mk(P), mk(Q), g)


def test_degenerate_zoo():
    """identical (IoU exactly 1), disjoint, touching edge / corner (empty),
    strict subset / superset, offset squares."""
    sq = np.array([[0, 0], [1, 0], [1, 1], [0, 1]], float)
    cases = [(sq, sq), (sq, sq + 5), (sq, sq + [1.0, 0]), (sq, sq + [1.0, 1.0]),
             (sq * 0.5 + 0.25, sq), (sq, sq * 0.5 + 0.25), (sq, sq + 0.5)]
    rng = np.random.default_rng(0)
    for _ in range(200):   # random identical pairs at scene coordinates
        b = box(*rng.uniform(-300, 300, 2), *rng.uniform(0.3, 12, 2), rng.uniform(-4, 4))
        cases.append((b, b.copy()))
    b = _pairs([c[0] for c in cases], [c[1] for c in cases], 4)
    iou, nx, xf, gr = gpu_paired(b)
    assert np.all(iou[7:] == 1.0) and iou[0] == 1.0
    assert list(xf[0][:4]) == [0x40, 0x41, 0x42, 0x43] and nx[0] == 4
    assert iou[1] == 0 and iou[2] == 0 and iou[3] == 0 and np.all(nx[1:4] == 0)
    assert np.all(xf[1:4] == 0)
    for k in (1, 2, 3):
        assert all(np.all(g.reshape(-1, 4)[k] == 0) for g in gr)
    assert list(xf[4][:4]) == [0x40, 0x41, 0x42, 0x43]
    assert list(xf[5][:4]) == [0x80, 0x81, 0x82, 0x83]
    assert list(xf[6][:4]) == [0xC8, 0x42, 0xD3, 0x80]
    assert abs(iou[6] - 1 / 7) < 1e-6
    ref = oracle.iou_paired_fwd(b.p1, b.p2)
    assert_iou_close(iou, ref["iou"])


@pytest.mark.parametrize("K", [4, 8])
def test_regular_ngons_max_vertices(K):
    """Regular K-gons with equal apothem rotated by pi/K: IoU = cos(pi/K), nx = 2K
    (the capacity bound; 16 vertices for K=8), all Cross."""
    rng = np.random.default_rng(K)
    P_list, Q_list = [], []
    for _ in range(256):
        a = rng.uniform(0.5, 3)
        R = a / math.cos(math.pi / K)
        ph = rng.uniform(0, 6.3)
        c = rng.uniform(-50, 50, 2)
        P_list.append(regular(K, R, ph, c))
        Q_list.append(regular(K, R, ph + math.pi / K, c))
    b = _pairs(P_list, Q_list, K)
    ok = oracle.margin_ok(b.p1, b.p2)
    iou, nx, xf, gr = gpu_paired(b)
    # the float32 vertices are a rounding of the exact n-gons: against the closed form
    # within that rounding, against the oracle (same float inputs) at the north_star 1e-5
    assert np.all(np.abs(iou - math.cos(math.pi / K)) < 2e-5)
    assert_iou_close(iou, oracle.iou_paired_fwd(b.p1, b.p2)["iou"])
    assert np.all(nx[ok] == 2 * K)
    ref = oracle.iou_paired_fwd(b.p1, b.p2)
    assert_flags_exact(nx[ok], xf[ok], {"nx": ref["nx"][ok], "xflags": ref["xflags"][ok]})
    rg = oracle.iou_paired_bwd(b.p1, b.p2, b.grad)
    for got, want in zip(gr, rg):
        assert_grad_close(got.reshape(want.shape)[ok], want[ok])


def test_bitwise_linearity_and_determinism():
    b = margin_batch(3, 20_000)
    x1, y1 = to_dev(b.p1)
    x2, y2 = to_dev(b.p2)
    g = torch.from_numpy(b.grad).to(dev())
    iou, nx, xf = dgal.iou_paired_fwd(x1, y1, x2, y2)
    iou2, nx2, xf2 = dgal.iou_paired_fwd(x1, y1, x2, y2)
    assert torch.equal(iou, iou2) and torch.equal(nx, nx2) and torch.equal(xf, xf2)
    r1 = dgal.iou_paired_bwd(x1, y1, x2, y2, g, nx, xf)
    r2 = dgal.iou_paired_bwd(x1, y1, x2, y2, 2 * g, nx, xf)
    r3 = dgal.iou_paired_bwd(x1, y1, x2, y2, -g, nx, xf)
    for a, bb, c in zip(r1, r2, r3):
        assert torch.equal(bb, 2 * a) and torch.equal(c, -a)
    # a prefix of the batch gives bitwise the same per-pair results
    m = 777
    i3, n3, f3 = dgal.iou_paired_fwd(x1[:m].contiguous(), y1[:m].contiguous(), x2[:m].contiguous(),
                                     y2[:m].contiguous())
    assert torch.equal(i3, iou[:m]) and torch.equal(f3, xf[:m])


@pytest.mark.parametrize("cfg", [3, 4])
def test_full_size_sampled(cfg):
    """BASELINE size, the launch configuration bench.py times (raw inputs, one
    launch over all pairs); sampled outputs checked one by one against the oracle.
    IoU is checked on every sampled pair, nx/xflags/gradients on the sampled
    pairs that are a margin away from degeneracy."""
    b = synth.gen_config(cfg)
    iou, nx, xf, gr = gpu_paired(b)
    rng = np.random.default_rng(cfg)
    idx = np.sort(rng.choice(b.n, size=1_000_000 if cfg == 3 else 400_000, replace=False))
    s = b.take(idx)
    ref = oracle.iou_paired_fwd(s.p1, s.p2)
    assert_iou_close(iou[idx], ref["iou"])
    ok = oracle.margin_ok(s.p1, s.p2)
    assert ok.mean() > 0.85
    assert_flags_exact(nx[idx][ok], xf[idx][ok], {"nx": ref["nx"][ok], "xflags": ref["xflags"][ok]})
    K = b.p1.K
    rg = oracle.iou_paired_bwd(s.p1, s.p2, s.grad)
    for got, want in zip(gr, rg):
        assert_grad_close(got.reshape(-1, K)[idx][ok], want[ok])
    # invariants that hold for every pair
    assert np.all((iou >= 0) & (iou <= 1))
    assert np.all((nx == 0) | ((nx >= 3) & (nx <= 2 * K)))
    assert np.all(iou[nx == 0] == 0)


def test_autograd_function_matches_bwd():
    b = margin_batch(1, 512)
    x1, y1 = to_dev(b.p1)
    x2, y2 = to_dev(b.p2)
    for t in (x1, y1, x2, y2):
        t.requires_grad_(True)
    iou = dgal.PolyIoU.apply(x1, y1, x2, y2)
    g = torch.from_numpy(b.grad).to(dev())
    (iou * g).sum().backward()
    _, nx, xf = dgal.iou_paired_fwd(x1.detach(), y1.detach(), x2.detach(), y2.detach())
    r = dgal.iou_paired_bwd(x1.detach(), y1.detach(), x2.detach(), y2.detach(), g, nx, xf)
    for t, want in zip((x1, y1, x2, y2), r):
        assert torch.equal(t.grad, want)


def test_empty_batch_is_noop():
    z = torch.empty((0, 4), dtype=torch.float32, device=dev())
    iou, nx, xf = dgal.iou_paired_fwd(z, z, z, z)
    assert iou.numel() == 0
    with pytest.raises(dgal.DgalError):
        bad = torch.zeros((8, 5), dtype=torch.float32, device=dev())
        dgal.iou_paired_fwd(bad, bad, bad, bad)


def test_backward_unaligned_side_inputs():
    """grad / nx / xflags not 16-byte aligned: the kernel loads tiles directly
    instead of by bulk copy; results are bitwise those of the aligned call."""
    b = margin_batch(3, 5000)
    x1, y1 = to_dev(b.p1)
    x2, y2 = to_dev(b.p2)
    g = torch.from_numpy(b.grad).to(dev())
    iou, nx, xf = dgal.iou_paired_fwd(x1, y1, x2, y2)
    ref = dgal.iou_paired_bwd(x1, y1, x2, y2, g, nx, xf)
    gb = torch.empty(g.numel() + 1, device=dev())[1:]
    gb.copy_(g)
    nb = torch.empty(nx.numel() + 3, dtype=torch.uint8, device=dev())[3:]
    nb.copy_(nx)
    got = dgal.iou_paired_bwd(x1, y1, x2, y2, gb, nb, xf)
    for a, c in zip(ref, got):
        assert torch.equal(a, c)


# ---------------------------------------------------------------------------
# fused loss forward + backward
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("cfg,n", [(1, 1024), (3, 40_000), (4, 20_000)])
def test_fused_matches_oracle(cfg, n):
    b = margin_batch(cfg, n)
    x1, y1 = to_dev(b.p1)
    x2, y2 = to_dev(b.p2)
    g = torch.from_numpy(b.grad).to(dev())
    iou, *gr = dgal.iou_paired_fused(x1, y1, x2, y2, grad=g)
    torch.cuda.synchronize()
    ref = oracle.iou_paired_fwd(b.p1, b.p2)
    assert_iou_close(iou.cpu().numpy(), ref["iou"])
    rg = oracle.iou_paired_bwd(b.p1, b.p2, b.grad)
    for got, want in zip(gr, rg):
        assert_grad_close(got.cpu().numpy().reshape(want.shape), want)


@pytest.mark.parametrize("cfg,n", [(3, 1), (3, 127), (3, 1023), (3, 1025), (3, 8193), (4, 129), (4, 1023),
                                   (4, 1025), (4, 4097)])
def test_fused_ragged_around_cta_chunks(cfg, n):
    """The fused kernel's CTA chunk is 128 threads x 8 tiles with the cp.async ring
    (both K): partial last tile and partial chunk, per-pair and scalar dL/dIoU."""
    b = margin_batch(cfg, n)
    x1, y1 = to_dev(b.p1)
    x2, y2 = to_dev(b.p2)
    g = torch.from_numpy(b.grad).to(dev())
    iou, *gr = dgal.iou_paired_fused(x1, y1, x2, y2, grad=g)
    torch.cuda.synchronize()
    assert_iou_close(iou.cpu().numpy(), oracle.iou_paired_fwd(b.p1, b.p2)["iou"])
    for got, want in zip(gr, oracle.iou_paired_bwd(b.p1, b.p2, b.grad)):
        assert_grad_close(got.cpu().numpy().reshape(want.shape), want)
    _, *ga = dgal.iou_paired_fused(x1, y1, x2, y2, scale=0.5)
    _, *gb = dgal.iou_paired_fused(x1, y1, x2, y2, grad=torch.full_like(g, 0.5))
    for a_, c_ in zip(ga, gb):
        assert torch.equal(a_, c_)


def test_fused_consistent_with_split_and_pairwise():
    b = margin_batch(3, 20_000)
    x1, y1 = to_dev(b.p1)
    x2, y2 = to_dev(b.p2)
    g = torch.from_numpy(b.grad).to(dev())
    iou_f, *gf = dgal.iou_paired_fused(x1, y1, x2, y2, grad=g)
    iou_s, nx, xf = dgal.iou_paired_fwd(x1, y1, x2, y2)
    gs = dgal.iou_paired_bwd(x1, y1, x2, y2, g, nx, xf)
    assert torch.allclose(iou_f, iou_s, atol=2e-6, rtol=0)
    for a, c in zip(gf, gs):
        assert torch.allclose(a, c, atol=1e-4, rtol=1e-3)
    # the fused IoU is bitwise the pairwise (flag-free) IoU of the same pairs, except on
    # the pairs the refine pass redid with the split forward (include/dgal.h)
    m = 256
    pw, _, _, _ = dgal.iou_pairwise(x1[:m].contiguous(), y1[:m].contiguous(), x2[:m].contiguous(),
                                    y2[:m].contiguous(), want_mask=False)
    d = pw.diagonal() != iou_f[:m]
    assert int(d.sum()) <= m // 10
    assert torch.allclose(pw.diagonal(), iou_f[:m], atol=2e-6, rtol=0)
    assert torch.equal(iou_f[:m][d], iou_s[:m][d])
    # scalar mode == constant array; bitwise linearity in dL/dIoU
    s = -1.0 / 4096
    _, *ga = dgal.iou_paired_fused(x1, y1, x2, y2, scale=s)
    _, *gb = dgal.iou_paired_fused(x1, y1, x2, y2, grad=torch.full_like(g, s))
    _, *gc = dgal.iou_paired_fused(x1, y1, x2, y2, scale=2 * s)
    for a, c, d in zip(ga, gb, gc):
        assert torch.equal(a, c) and torch.equal(d, 2 * a)


def test_fused_loss_autograd():
    b = margin_batch(1, 1000)
    x1, y1 = to_dev(b.p1)
    x2, y2 = to_dev(b.p2)
    ts = [t.clone().requires_grad_(True) for t in (x1, y1, x2, y2)]
    loss = dgal.PolyIoULoss.apply(*ts)
    loss.backward()
    iou = oracle.iou_paired_fwd(b.p1, b.p2)["iou"]
    assert abs(loss.item() - float(np.mean(1 - iou))) < 1e-5
    rg = oracle.iou_paired_bwd(b.p1, b.p2, np.full(b.n, -1.0 / b.n))
    for t, want in zip(ts, rg):
        assert_grad_close(t.grad.cpu().numpy().reshape(want.shape), want)


def _near_coincident_boxes(n, scale, seed):
    """Box pairs b2 = b1 + perturbation of relative size `scale` on a random subset of
    the parameters (prediction ~ target: nearly coincident edges, shared vertices)."""
    rng = np.random.default_rng(seed)
    cx = rng.uniform(0, 70, n); cy = rng.uniform(-40, 40, n)
    w = rng.uniform(0.5, 5, n); h = rng.uniform(0.5, 2, n); th = rng.uniform(-np.pi, np.pi, n)
    b1 = np.stack([cx, cy, w, h, th]).astype(np.float32)
    pert = rng.normal(size=(5, n)) * scale * np.array([w, w, w, h, np.ones(n)])
    pert *= rng.uniform(size=(5, n)) < 0.6
    b2 = (b1.astype(np.float64) + pert).astype(np.float32)
    return b1, b2


@pytest.mark.parametrize("scale", [1e-7, 1e-6, 1e-5, 1e-4, 1e-3, 1e-2])
def test_near_coincident_polygons_iou(scale):
    """The converged-training regime: IoU within 1e-5 of the oracle on every pair
    (closure of the clip), not only on margin inputs."""
    b1, b2 = _near_coincident_boxes(100_000, scale, seed=int(-math.log10(scale)))
    x1, y1 = oracle.box_corners(b1.T.astype(np.float64))
    x2, y2 = oracle.box_corners(b2.T.astype(np.float64))
    x1, y1, x2, y2 = (a.astype(np.float32) for a in (x1, y1, x2, y2))
    T = lambda a: torch.from_numpy(a).to(dev())  # noqa: E731
    iou, nx, xf = dgal.iou_paired_fwd(T(x1), T(y1), T(x2), T(y2))
    ref = oracle.iou_paired_fwd((x1, y1), (x2, y2))
    assert_iou_close(iou.cpu().numpy(), ref["iou"])
    nxc = nx.cpu().numpy()
    assert np.all((nxc >= 3) & (nxc <= 8))          # always a valid record for the backward


def test_integer_grid_rectangles_on_device():
    """Exact shared edges / touching / containment: the axis-aligned closed form."""
    rng = np.random.default_rng(12)
    g = rng.integers(0, 4, size=(50_000, 8)).astype(np.float32)
    x0, y0, a, b = g[:, 0], g[:, 1], 1 + g[:, 2], 1 + g[:, 3]
    u0, v0, c, d = g[:, 4], g[:, 5], 1 + g[:, 6], 1 + g[:, 7]
    P = [np.stack([x0, x0 + a, x0 + a, x0], 1), np.stack([y0, y0, y0 + b, y0 + b], 1)]
    Q = [np.stack([u0, u0 + c, u0 + c, u0], 1), np.stack([v0, v0, v0 + d, v0 + d], 1)]
    T = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev())  # noqa: E731
    iou = dgal.iou_paired_fwd(T(P[0]), T(P[1]), T(Q[0]), T(Q[1]))[0].cpu().numpy()
    ox = np.clip(np.minimum(x0 + a, u0 + c) - np.maximum(x0, u0), 0, None)
    oy = np.clip(np.minimum(y0 + b, v0 + d) - np.maximum(y0, v0), 0, None)
    ai = ox * oy
    want = ai / (a * b + c * d - ai)
    assert np.max(np.abs(iou - want)) <= 1e-6


@pytest.mark.parametrize("scale", [1e-6, 1e-5, 1e-4, 1e-3, 1e-2])
def test_near_coincident_gradients(scale):
    """Backward on prediction ~ target pairs: wherever the device's nx/xflags equal the
    oracle's (same piece of the piecewise-smooth IoU), the vertex gradients match the
    oracle at the north_star tolerance — the crossing parameters of nearly parallel
    edges are refined in double.  Pairs whose flags differ sit within
    rounding of a flag change, where the gradient is discontinuous."""
    b1, b2 = _near_coincident_boxes(50_000, scale, seed=20 + int(-math.log10(scale)))
    x1, y1 = oracle.box_corners(b1.T.astype(np.float64))
    x2, y2 = oracle.box_corners(b2.T.astype(np.float64))
    x1, y1, x2, y2 = (a.astype(np.float32) for a in (x1, y1, x2, y2))
    g = np.random.default_rng(5).uniform(-1, 1, x1.shape[0]).astype(np.float32)
    T = lambda a: torch.from_numpy(a).to(dev())  # noqa: E731
    X = (T(x1), T(y1), T(x2), T(y2))
    iou, nx, xf = dgal.iou_paired_fwd(*X)
    gr = dgal.iou_paired_bwd(*X, T(g), nx, xf)
    rf = oracle.iou_paired_fwd((x1, y1), (x2, y2))
    same = (nx.cpu().numpy() == rf["nx"]) & np.all(xf.cpu().numpy() == rf["xflags"], 1)
    assert same.mean() > 0.8
    ref = oracle.iou_paired_bwd((x1, y1), (x2, y2), g)
    for got, want in zip(gr, ref):
        assert_grad_close(got.cpu().numpy()[same], want[same])


@pytest.mark.parametrize("scale", [1e-7, 1e-5, 1e-3, 1e-2])
def test_near_coincident_octagons_iou(scale):
    """K = 8: convex octagons (ellipse-inscribed, as cfg4) and a copy with every vertex
    moved by ~scale x size (still convex at these scales): IoU within 1e-5 on every pair,
    and a valid record (3 <= nx <= 16)."""
    rng = np.random.default_rng(30 + int(-math.log10(scale)))
    n = 50_000
    c = rng.uniform(-10, 10, (n, 2))
    a = rng.uniform(1, 3, n)
    b = a * rng.uniform(0.6, 1.0, n)
    phi = rng.uniform(-np.pi, np.pi, n)
    ang = (np.arange(8)[None, :] + rng.uniform(-0.3, 0.3, (n, 8))) * np.pi / 4
    ex, ey = a[:, None] * np.cos(ang), b[:, None] * np.sin(ang)
    x1 = c[:, :1] + np.cos(phi)[:, None] * ex - np.sin(phi)[:, None] * ey
    y1 = c[:, 1:] + np.sin(phi)[:, None] * ex + np.cos(phi)[:, None] * ey
    x2 = x1 + rng.normal(size=x1.shape) * scale * a[:, None] * (rng.uniform(size=x1.shape) < 0.6)
    y2 = y1 + rng.normal(size=y1.shape) * scale * a[:, None] * (rng.uniform(size=y1.shape) < 0.6)
    x1, y1, x2, y2 = (v.astype(np.float32) for v in (x1, y1, x2, y2))
    T = lambda v: torch.from_numpy(np.ascontiguousarray(v)).to(dev())  # noqa: E731
    iou, nx, xf = dgal.iou_paired_fwd(T(x1), T(y1), T(x2), T(y2))
    ref = oracle.iou_paired_fwd((x1, y1), (x2, y2))
    assert_iou_close(iou.cpu().numpy(), ref["iou"])
    nxc = nx.cpu().numpy()
    assert np.all((nxc >= 3) & (nxc <= 16))


@pytest.mark.parametrize("m,K", [(3, 4), (5, 8), (6, 8), (7, 8)])
def test_padded_polygons(m, K):
    """Polygons with m < K vertices, padded by repeating the last vertex (include/dgal.h):
    IoU and the gradient of each real vertex (summed over its copies) equal the oracle on
    the unpadded polygons (margin inputs)."""
    rng = np.random.default_rng(50 + m)
    n = 20000
    def convex():
        c = rng.uniform(-5, 5, (n, 2)); a = rng.uniform(1, 3, n); b = a * rng.uniform(0.5, 1, n)
        # vertex angles uniform on the ellipse, no minimum gap: slivers and near-zero-length
        # edges included (thin pairs are redone in double, DESIGN.md §4.1 Conditioning)
        gaps = rng.uniform(0.0, 1.0, (n, m))
        gaps = gaps / gaps.sum(1, keepdims=True) * (2 * np.pi)
        ang = rng.uniform(0, 2 * np.pi, (n, 1)) + np.cumsum(gaps, 1) - gaps[:, :1]
        phi = rng.uniform(-np.pi, np.pi, n)
        ex, ey = a[:, None] * np.cos(ang), b[:, None] * np.sin(ang)
        return ((c[:, :1] + np.cos(phi)[:, None] * ex - np.sin(phi)[:, None] * ey).astype(np.float32),
                (c[:, 1:] + np.sin(phi)[:, None] * ex + np.cos(phi)[:, None] * ey).astype(np.float32))
    x1, y1 = convex()
    x2, y2 = convex()
    x2 += (x1.mean(1, keepdims=True) - x2.mean(1, keepdims=True)) * 0.8
    y2 += (y1.mean(1, keepdims=True) - y2.mean(1, keepdims=True)) * 0.8
    ok = oracle.margin_ok((x1, y1), (x2, y2))
    x1, y1, x2, y2 = (v[ok] for v in (x1, y1, x2, y2))
    pad = lambda v: np.ascontiguousarray(np.concatenate([v, np.repeat(v[:, -1:], K - m, 1)], 1))  # noqa: E731
    T = lambda v: torch.from_numpy(pad(v)).to(dev())  # noqa: E731
    X = (T(x1), T(y1), T(x2), T(y2))
    g = np.random.default_rng(1).uniform(-1, 1, x1.shape[0]).astype(np.float32)
    iou, nx, xf = dgal.iou_paired_fwd(*X)
    gr = dgal.iou_paired_bwd(*X, torch.from_numpy(g).to(dev()), nx, xf)
    ref = oracle.iou_paired_fwd((x1, y1), (x2, y2))
    assert_iou_close(iou.cpu().numpy(), ref["iou"])
    rg = oracle.iou_paired_bwd((x1, y1), (x2, y2), g)
    for got, want in zip(gr, rg):
        got = got.cpu().numpy()
        folded = got[:, :m].copy()
        folded[:, m - 1] += got[:, m:].sum(1)
        assert_grad_close(folded, want)


def _near_octagons(n, scale, seed):
    """Convex octagons (ellipse-inscribed, as cfg4) and a copy with EVERY vertex moved by
    ~scale x size (convex at these scales; no exactly shared vertex, so the flags are
    those of nearly parallel crossings, not of exact ties)."""
    rng = np.random.default_rng(seed)
    c = rng.uniform(-10, 10, (n, 2))
    a = rng.uniform(1, 3, n)
    b = a * rng.uniform(0.6, 1.0, n)
    phi = rng.uniform(-np.pi, np.pi, n)
    ang = (np.arange(8)[None, :] + rng.uniform(-0.3, 0.3, (n, 8))) * np.pi / 4
    ex, ey = a[:, None] * np.cos(ang), b[:, None] * np.sin(ang)
    x1 = c[:, :1] + np.cos(phi)[:, None] * ex - np.sin(phi)[:, None] * ey
    y1 = c[:, 1:] + np.sin(phi)[:, None] * ex + np.cos(phi)[:, None] * ey
    x2 = x1 + rng.normal(size=x1.shape) * scale * a[:, None]
    y2 = y1 + rng.normal(size=y1.shape) * scale * a[:, None]
    return tuple(np.ascontiguousarray(v.astype(np.float32)) for v in (x1, y1, x2, y2))


@pytest.mark.parametrize("K", [4, 8])
@pytest.mark.parametrize("scale", [1e-6, 1e-5, 1e-4, 1e-3, 1e-2])
def test_fused_near_coincident_gradients(K, scale):
    """The fused loss kernel on prediction ~ target pairs (the regime an IoU loss ends
    training in): IoU within 1e-5 on every pair, and wherever the split forward's flags
    equal the oracle's, the fused vertex gradients match the oracle at the north_star
    tolerance — nearly parallel edge pairs are marked and redone by the refine pass with
    the split path's exact crossings (include/dgal.h)."""
    seed = 40 + int(-math.log10(scale)) + K
    if K == 4:
        b1, b2 = _near_coincident_boxes(50_000, scale, seed=seed)
        x1, y1 = oracle.box_corners(b1.T.astype(np.float64))
        x2, y2 = oracle.box_corners(b2.T.astype(np.float64))
        x1, y1, x2, y2 = (np.ascontiguousarray(a.astype(np.float32)) for a in (x1, y1, x2, y2))
    else:
        x1, y1, x2, y2 = _near_octagons(30_000, scale, seed)
    n = x1.shape[0]
    g = np.random.default_rng(seed).uniform(-1, 1, n).astype(np.float32)
    T = lambda a: torch.from_numpy(a).to(dev())  # noqa: E731
    X = (T(x1), T(y1), T(x2), T(y2))
    _, nx, xf = dgal.iou_paired_fwd(*X)
    iou_f, *gf = dgal.iou_paired_fused(*X, grad=T(g))
    rf = oracle.iou_paired_fwd((x1, y1), (x2, y2))
    assert_iou_close(iou_f.cpu().numpy(), rf["iou"])
    same = (nx.cpu().numpy() == rf["nx"]) & np.all(xf.cpu().numpy() == rf["xflags"], 1)
    assert same.mean() > 0.8
    ref = oracle.iou_paired_bwd((x1, y1), (x2, y2), g)
    for got, want in zip(gf, ref):
        assert_grad_close(got.cpu().numpy()[same], want[same])


def test_fused_workspace_stays_zero_and_reusable():
    """The refine queue is left all-zero by every call (include/dgal.h), so one workspace
    serves consecutive calls; results are bitwise repeatable."""
    b1, b2 = _near_coincident_boxes(20_000, 1e-4, seed=7)
    x1, y1 = oracle.box_corners(b1.T.astype(np.float64))
    x2, y2 = oracle.box_corners(b2.T.astype(np.float64))
    X = [torch.from_numpy(np.ascontiguousarray(a.astype(np.float32))).to(dev()) for a in (x1, y1, x2, y2)]
    ws = torch.zeros(dgal.lib().dgal_fused_workspace_bytes(20_000), dtype=torch.uint8, device=dev())
    r1 = dgal.iou_paired_fused(*X, scale=0.25, workspace=ws)
    assert int(ws[:8].count_nonzero()) == 0          # count and done reset by the refine kernel
    r2 = dgal.iou_paired_fused(*X, scale=0.25, workspace=ws)
    for a_, b_ in zip(r1, r2):
        assert torch.equal(a_, b_)


@pytest.mark.parametrize("K,offset", [(4, 1e3), (4, 5e3), (8, 5e3), (4, 2e4), (8, 2e4)])
def test_far_from_origin_scene_coordinates(K, offset):
    """Pairs placed at scene coordinates up to +-offset metres (float32 inputs rounded
    once there: the ulp of the coordinates grows to ~5e-4 m): every result is that of
    the rounded float polygons, so the oracle runs on exactly the device's inputs.
    The kernels re-centre on p1's vertex 0 (exact subtraction) before any arithmetic:
    IoU <= 1e-5 on every pair, flags and gradients on the margin pairs; the same for the
    fused loss kernel."""
    cfg = 3 if K == 4 else 4
    n = 20000
    b = synth.gen_config(cfg, n)
    rng = np.random.default_rng(int(offset) + K)
    ox = rng.uniform(-offset, offset, (n, 1))
    oy = rng.uniform(-offset, offset, (n, 1))
    sh = lambda a, o: (a.reshape(n, K).astype(np.float64) + o).astype(np.float32)  # noqa: E731
    x1, y1, x2, y2 = sh(b.p1.x, ox), sh(b.p1.y, oy), sh(b.p2.x, ox), sh(b.p2.y, oy)
    X = [torch.from_numpy(np.ascontiguousarray(a)).to(dev()) for a in (x1, y1, x2, y2)]
    g = torch.from_numpy(b.grad).to(dev())
    iou, nx, xf = dgal.iou_paired_fwd(*X)
    gr = dgal.iou_paired_bwd(*X, g, nx, xf)
    p1 = (x1.astype(np.float64), y1.astype(np.float64))
    p2 = (x2.astype(np.float64), y2.astype(np.float64))
    ref = oracle.iou_paired_fwd(p1, p2)
    assert_iou_close(iou.cpu().numpy(), ref["iou"])
    ok = oracle.margin_ok(p1, p2)
    assert ok.mean() > 0.5
    assert_flags_exact(nx.cpu().numpy()[ok], xf.cpu().numpy()[ok],
                       {"nx": ref["nx"][ok], "xflags": ref["xflags"][ok]})
    rg = oracle.iou_paired_bwd(p1, p2, b.grad)
    for got, want in zip(gr, rg):
        assert_grad_close(got.cpu().numpy().astype(np.float64)[ok], want[ok])
    # the fused loss kernel (and its refine pass) on the same far-away pairs
    iou_f, *gf = dgal.iou_paired_fused(*X, grad=g)
    assert_iou_close(iou_f.cpu().numpy(), ref["iou"])
    for got, want in zip(gf, rg):
        assert_grad_close(got.cpu().numpy().astype(np.float64)[ok], want[ok])


@pytest.mark.parametrize("K,scale", [(4, 1e-6), (4, 1e6), (8, 1e-6), (8, 1e6)])
def test_scale_extremes(K, scale):
    """cfg3 / cfg4 pairs scaled by 1e-6 and 1e6 (float inputs rounded after scaling): the
    decisions, areas and thin test are relative, so IoU of every pair (split and fused)
    stays within 1e-5 of the oracle, flags bit-exact on the margin pairs."""
    b = synth.gen_config(3 if K == 4 else 4, 8192)
    a = [(v.reshape(-1, K).astype(np.float64) * scale).astype(np.float32) for v in (b.p1.x, b.p1.y, b.p2.x, b.p2.y)]
    X = [torch.from_numpy(np.ascontiguousarray(v)).to(dev()) for v in a]
    iou, nx, xf = dgal.iou_paired_fwd(*X)
    iou_f = dgal.iou_paired_fused(*X, scale=1.0)[0]
    p1 = (a[0].astype(np.float64), a[1].astype(np.float64))
    p2 = (a[2].astype(np.float64), a[3].astype(np.float64))
    ref = oracle.iou_paired_fwd(p1, p2)
    assert_iou_close(iou.cpu().numpy(), ref["iou"])
    assert_iou_close(iou_f.cpu().numpy(), ref["iou"])
    ok = oracle.margin_ok(p1, p2)
    assert_flags_exact(nx.cpu().numpy()[ok], xf.cpu().numpy()[ok], {"nx": ref["nx"][ok], "xflags": ref["xflags"][ok]})


@pytest.mark.parametrize("K", [4, 8])
def test_zero_area_polygons(K):
    """Degenerate inputs of zero area (S:396 range, set inclusion): a point polygon inside
    the other, in both roles, and a segment along an edge — IoU within 1e-5 of the
    oracle's 0 (split and fused); identical polygons with a rotated vertex order give 1."""
    b = synth.gen_config(3 if K == 4 else 4, 4096)
    x, y = b.p1.x.reshape(-1, K), b.p1.y.reshape(-1, K)
    cx, cy = np.repeat(x.mean(1, keepdims=True), K, 1), np.repeat(y.mean(1, keepdims=True), K, 1)
    sx = np.concatenate([np.repeat(x[:, :1], K // 2, 1), np.repeat(x[:, 1:2], K // 2, 1)], 1)
    sy = np.concatenate([np.repeat(y[:, :1], K // 2, 1), np.repeat(y[:, 1:2], K // 2, 1)], 1)
    cases = [(x, y, cx, cy), (cx, cy, x, y), (x, y, sx, sy), (x, y, np.roll(x, 1, 1), np.roll(y, 1, 1))]
    for a in cases:
        X = [torch.from_numpy(np.ascontiguousarray(v.astype(np.float32))).to(dev()) for v in a]
        ref = oracle.iou_paired_fwd(*[(X[i].cpu().numpy().astype(np.float64), X[i + 1].cpu().numpy().astype(np.float64))
                                      for i in (0, 2)])
        assert_iou_close(dgal.iou_paired_fwd(*X)[0].cpu().numpy(), ref["iou"])
        assert_iou_close(dgal.iou_paired_fused(*X, scale=1.0)[0].cpu().numpy(), ref["iou"])
