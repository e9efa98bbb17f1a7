"""GPU parity of the rotated-box front end (dgal_box_iou_paired_fwd/bwd/fused;
SURVEY §8(f) f1 2D boxes and f3 yaw-only 3D boxes) against the oracle, through
the C ABI.  Same tolerances as the polygon path: nx/xflags bit-exact on margin
inputs, IoU <= 1e-5 abs, parameter gradients <= 1e-4 abs or <= 1e-3 rel."""
import math

import numpy as np
import pytest
import torch

import oracle
import paper_2011_11134_b200 as dgal
import synth
from gpu_util import assert_flags_exact, assert_grad_close, assert_iou_close, dev
from helpers import box_margin_batch, box_margin_ok

pytestmark = pytest.mark.gpu


def gpu_box(b, layout="planes", grad=None):
    """BoxPairBatch -> (iou, nx, xf, gb1 [P, n], gb2 [P, n]) through fwd + bwd."""
    if layout == "planes":
        b1, b2 = torch.from_numpy(b.b1).to(dev()), torch.from_numpy(b.b2).to(dev())
    else:
        b1 = torch.from_numpy(np.ascontiguousarray(b.b1.T)).to(dev())
        b2 = torch.from_numpy(np.ascontiguousarray(b.b2.T)).to(dev())
    iou, nx, xf = dgal.box_iou_paired_fwd(b1, b2, layout)
    g = torch.from_numpy(b.grad if grad is None else grad).to(dev())
    g1, g2 = dgal.box_iou_paired_bwd(b1, b2, g, nx, xf, layout)
    torch.cuda.synchronize()
    g1, g2 = g1.cpu().numpy(), g2.cpu().numpy()
    if layout == "rows":
        g1, g2 = g1.T, g2.T
    return iou.cpu().numpy(), nx.cpu().numpy(), xf.cpu().numpy(), g1, g2


def check_box_against_oracle(b, flags=True, layout="planes"):
    iou, nx, xf, g1, g2 = gpu_box(b, layout)
    r1, r2 = b.rows64()
    ref = oracle.box_iou_paired(r1, r2, b.grad.astype(np.float64))
    assert_iou_close(iou, ref["iou"])
    if flags:
        assert_flags_exact(nx, xf, ref)
    assert_grad_close(g1.T, ref["gb1"])
    assert_grad_close(g2.T, ref["gb2"])
    return iou, nx, xf, g1, g2, ref


def _batch(rows1, rows2, grad=None):
    r1 = np.asarray(rows1, np.float32)
    r2 = np.asarray(rows2, np.float32)
    g = np.ones(len(r1), np.float32) if grad is None else np.asarray(grad, np.float32)
    return synth.BoxPairBatch(np.ascontiguousarray(r1.T), np.ascontiguousarray(r2.T), g)


@pytest.mark.parametrize("dims", [2, 3])
@pytest.mark.parametrize("n", [1, 31, 257, 4097, 40_000])
def test_box_margin_inputs_full_compare(dims, n):
    check_box_against_oracle(box_margin_batch(dims, n))


@pytest.mark.parametrize("dims", [2, 3])
def test_rows_layout_is_bitwise_planes(dims):
    b = box_margin_batch(dims, 3000)
    a = gpu_box(b, "planes")
    r = gpu_box(b, "rows")
    for x, y in zip(a, r):
        assert np.array_equal(x, y)
    check_box_against_oracle(b, layout="rows")


def test_box_equals_polygon_path_on_its_corners():
    """The box forward is the polygon forward on box_to_polygon's corners: IoU
    within rounding of the two corner computations, flags identical."""
    b = box_margin_batch(2, 5000)
    iou, nx, xf, _, _ = gpu_box(b)
    r1, r2 = b.rows64()
    x1, y1 = oracle.box_corners(r1)
    x2, y2 = oracle.box_corners(r2)
    T = lambda a: torch.from_numpy(a.astype(np.float32)).to(dev())  # noqa: E731
    pi, pn, pf = dgal.iou_paired_fwd(T(x1), T(y1), T(x2), T(y2))
    assert np.max(np.abs(pi.cpu().numpy() - iou)) <= 2e-5
    assert np.array_equal(pn.cpu().numpy(), nx) and np.array_equal(pf.cpu().numpy(), xf)


def test_box_worked_examples():
    """S:370-372, S:390-392 on the device."""
    rows2 = [[0, 0, 2, 2, 0], [3, -2, 4, 1.5, 0.4], [0, 0, 2, 2, 0.3]]
    rows2b = [[0, 0, 2, 2, math.pi / 4], [3, -2, 4, 1.5, 0.4], [10, 0, 2, 2, 1.1]]
    iou, nx, xf, g1, g2 = gpu_box(_batch(rows2, rows2b))
    assert abs(iou[0] - 1 / math.sqrt(2)) < 2e-6 and nx[0] == 8          # octagon
    assert iou[1] == 1.0                                                 # identical
    assert abs(g1[0, 1]) < 1e-5 and abs(g1[1, 1]) < 1e-5                 # stationary
    assert iou[2] == 0.0 and nx[2] == 0 and np.all(g1[:, 2] == 0)        # disjoint
    rows3 = [[0, 0, 0, 1, 1, 1, 0], [0, 0, 0, 1, 1, 1, 0], [0, 0, 0, 1, 1, 1, 0.2], [0, 0, 0, 1, 1, 1, 0]]
    rows3b = [[0, 0, 0, 1, 1, 1, 0], [0.5, 0.5, 0.5, 1, 1, 1, 0], [0.1, 0, 1.0, 1, 1, 1, 0], [0, 0, 0.3, 1, 1, 1, 0]]
    iou, nx, xf, g1, g2 = gpu_box(_batch(rows3, rows3b))
    assert iou[0] == 1.0
    assert abs(iou[1] - 1 / 15) < 1e-6
    assert iou[2] == 0.0 and nx[2] == 0 and np.all(g1[:, 2] == 0) and np.all(g2[:, 2] == 0)
    assert abs(g2[2, 3] + 2 / 1.3 ** 2) < 1e-5                           # dz closed form


def test_3d_reduces_to_2d_on_device():
    b3 = box_margin_batch(3, 4000)
    b3.b2[2] = b3.b1[2]
    b3.b2[5] = b3.b1[5]
    i3 = gpu_box(b3)[0]
    b2 = synth.BoxPairBatch(np.ascontiguousarray(b3.b1[[0, 1, 3, 4, 6]]),
                            np.ascontiguousarray(b3.b2[[0, 1, 3, 4, 6]]), b3.grad)
    i2 = gpu_box(b2)[0]
    assert np.max(np.abs(i3 - i2)) <= 2e-6


@pytest.mark.parametrize("dims", [2, 3])
def test_box_fused_matches_oracle_and_split(dims):
    b = box_margin_batch(dims, 20_000)
    B1, B2 = torch.from_numpy(b.b1).to(dev()), torch.from_numpy(b.b2).to(dev())
    g = torch.from_numpy(b.grad).to(dev())
    iou, g1, g2 = dgal.box_iou_paired_fused(B1, B2, grad=g)
    torch.cuda.synchronize()
    r1, r2 = b.rows64()
    ref = oracle.box_iou_paired(r1, r2, b.grad.astype(np.float64))
    assert_iou_close(iou.cpu().numpy(), ref["iou"])
    assert_grad_close(g1.cpu().numpy().T, ref["gb1"])
    assert_grad_close(g2.cpu().numpy().T, ref["gb2"])
    # scalar-gradient form == per-pair form with a constant vector, bitwise
    _, h1, _ = dgal.box_iou_paired_fused(B1, B2, scale=-0.25, want_iou=False)
    _, k1, _ = dgal.box_iou_paired_fused(B1, B2, grad=torch.full_like(g, -0.25))
    assert torch.equal(h1, k1)


@pytest.mark.parametrize("dims", [2, 3])
@pytest.mark.parametrize("n", [127, 1023, 1025, 8193])
def test_box_ragged_around_cta_chunks(dims, n):
    """Forward and fused box kernels: 128 threads x 8 tiles per CTA with the
    parameter prefetch ring — partial last tile and partial chunk."""
    b = box_margin_batch(dims, n)
    check_box_against_oracle(b)
    B1, B2 = torch.from_numpy(b.b1).to(dev()), torch.from_numpy(b.b2).to(dev())
    g = torch.from_numpy(b.grad).to(dev())
    iou, g1, g2 = dgal.box_iou_paired_fused(B1, B2, grad=g)
    torch.cuda.synchronize()
    r1, r2 = b.rows64()
    ref = oracle.box_iou_paired(r1, r2, b.grad.astype(np.float64))
    assert_iou_close(iou.cpu().numpy(), ref["iou"])
    assert_grad_close(g1.cpu().numpy().T, ref["gb1"])
    assert_grad_close(g2.cpu().numpy().T, ref["gb2"])


def test_box_autograd_and_loss():
    b = box_margin_batch(3, 2000)
    B1 = torch.from_numpy(b.b1).to(dev()).requires_grad_(True)
    B2 = torch.from_numpy(b.b2).to(dev()).requires_grad_(True)
    iou = dgal.BoxIoU.apply(B1, B2, "planes")
    (iou * torch.from_numpy(b.grad).to(dev())).sum().backward()
    r1, r2 = b.rows64()
    ref = oracle.box_iou_paired(r1, r2, b.grad.astype(np.float64))
    assert_grad_close(B1.grad.cpu().numpy().T, ref["gb1"])
    assert_grad_close(B2.grad.cpu().numpy().T, ref["gb2"])
    B1.grad = None
    B2.grad = None
    loss = dgal.BoxIoULoss.apply(B1, B2, "planes")
    loss.backward()
    ref = oracle.box_iou_paired(r1, r2, np.full(b.n, -1.0 / b.n))
    assert abs(loss.item() - (1 - ref["iou"]).mean()) < 1e-5
    assert_grad_close(B1.grad.cpu().numpy().T, ref["gb1"])


def test_box_empty_batch_is_noop():
    z = torch.empty(5, 0, device=dev())
    iou, nx, xf = dgal.box_iou_paired_fwd(z, z)
    assert iou.numel() == 0


@pytest.mark.parametrize("dims", [2, 3])
def test_box_full_size_sampled(dims):
    """bench.py's box workload (2^24 pairs, one launch each); sampled pairs vs the
    oracle, flags / gradients on the margin-passing ones; invariants on all."""
    b = synth.gen_box_pairs(1 << 24, dims)
    iou, nx, xf, g1, g2 = gpu_box(b)
    rng = np.random.default_rng(dims)
    idx = np.sort(rng.choice(b.n, size=50_000, replace=False))
    s = b.take(idx)
    r1, r2 = s.rows64()
    ref = oracle.box_iou_paired(r1, r2, s.grad.astype(np.float64))
    assert_iou_close(iou[idx], ref["iou"])
    ok = box_margin_ok(r1, r2)
    assert ok.mean() > 0.8
    assert_flags_exact(nx[idx][ok], xf[idx][ok], {"nx": ref["nx"][ok], "xflags": ref["xflags"][ok]})
    assert_grad_close(g1[:, idx].T[ok], ref["gb1"][ok])
    assert_grad_close(g2[:, idx].T[ok], ref["gb2"][ok])
    assert np.all((iou >= 0) & (iou <= 1))
    assert np.all(iou[nx == 0] == 0)


@pytest.mark.parametrize("scale", [1e-7, 1e-6, 1e-5, 1e-4, 1e-3, 1e-2])
def test_near_coincident_boxes_iou(scale):
    """Prediction ~ target box pairs (nearly coincident edges): IoU within 1e-5 on
    every pair, 2D and 3D."""
    from test_gpu_paired import _near_coincident_boxes
    b1, b2 = _near_coincident_boxes(100_000, scale, seed=7 + int(-math.log10(scale)))
    g = np.ones(b1.shape[1], np.float32)
    iou = gpu_box(synth.BoxPairBatch(b1, b2, g))[0]
    ref = oracle.box_iou_paired(b1.T.astype(np.float64), b2.T.astype(np.float64))["iou"]
    assert_iou_close(iou, ref)
    rng = np.random.default_rng(3)
    z = rng.normal(-1, 0.4, b1.shape[1]); d = rng.uniform(1.4, 1.9, b1.shape[1])
    b13 = np.concatenate([b1[:2], z[None], b1[2:4], d[None], b1[4:]]).astype(np.float32)
    b23 = np.concatenate([b2[:2], (z + scale * rng.normal(size=z.size))[None], b2[2:4], d[None], b2[4:]]).astype(np.float32)
    iou3 = gpu_box(synth.BoxPairBatch(b13, b23, g))[0]
    ref3 = oracle.box_iou_paired(b13.T.astype(np.float64), b23.T.astype(np.float64))["iou"]
    assert_iou_close(iou3, ref3)


@pytest.mark.parametrize("scale", [1e-6, 1e-5, 1e-4, 1e-3, 1e-2])
def test_near_coincident_box_gradients(scale):
    """Prediction ~ target boxes: on the pairs whose flags equal the oracle's, the box
    parameter gradients match it (the ill-conditioned crossings, |sin| < 2^-7, are
    refined on corners rebuilt in double from the parameters)."""
    from test_gpu_paired import _near_coincident_boxes
    b1, b2 = _near_coincident_boxes(50_000, scale, seed=40 + int(-math.log10(scale)))
    g = np.random.default_rng(6).uniform(-1, 1, b1.shape[1]).astype(np.float32)
    iou, nx, xf, g1, g2 = gpu_box(synth.BoxPairBatch(b1, b2, g))
    ref = oracle.box_iou_paired(b1.T.astype(np.float64), b2.T.astype(np.float64), g.astype(np.float64))
    same = (nx == ref["nx"]) & np.all(xf == ref["xflags"], 1)
    assert same.mean() > 0.8          # the rest sit within rounding of a flag change (exact ties at 1e-6)
    assert_grad_close(g1.T[same], ref["gb1"][same])
    assert_grad_close(g2.T[same], ref["gb2"][same])


@pytest.mark.parametrize("dims", [2, 3])
@pytest.mark.parametrize("scale", [1e-6, 1e-5, 1e-4, 1e-3, 1e-2])
def test_box_fused_near_coincident(dims, scale):
    """The fused box loss kernel on prediction ~ target pairs: IoU within 1e-5 on every
    pair, parameter gradients at the north_star tolerance wherever the split forward's
    flags equal the oracle's (nearly parallel edge pairs are redone by the refine pass
    with the box split path's exact crossings, include/dgal.h)."""
    from test_gpu_paired import _near_coincident_boxes
    n = 40_000
    b1, b2 = _near_coincident_boxes(n, scale, seed=60 + dims + int(-math.log10(scale)))
    rng = np.random.default_rng(dims)
    if dims == 3:
        z = rng.normal(-1, 0.4, n); d = rng.uniform(1.4, 1.9, n)
        dz = scale * rng.normal(size=n) + 0.05 * rng.uniform(0.5, 1, n)   # z extents away from ties
        b1 = np.concatenate([b1[:2], z[None], b1[2:4], d[None], b1[4:]]).astype(np.float32)
        b2 = np.concatenate([b2[:2], (z + dz)[None], b2[2:4], d[None], b2[4:]]).astype(np.float32)
    g = rng.uniform(-1, 1, n).astype(np.float32)
    B1, B2 = torch.from_numpy(np.ascontiguousarray(b1)).to(dev()), torch.from_numpy(np.ascontiguousarray(b2)).to(dev())
    _, nx, xf = dgal.box_iou_paired_fwd(B1, B2)
    iou, g1, g2 = dgal.box_iou_paired_fused(B1, B2, grad=torch.from_numpy(g).to(dev()))
    ref = oracle.box_iou_paired(b1.T.astype(np.float64), b2.T.astype(np.float64), g.astype(np.float64))
    assert_iou_close(iou.cpu().numpy(), ref["iou"])
    same = (nx.cpu().numpy() == ref["nx"]) & np.all(xf.cpu().numpy() == ref["xflags"], 1)
    assert same.mean() > 0.8
    assert_grad_close(g1.cpu().numpy().T[same], ref["gb1"][same])
    assert_grad_close(g2.cpu().numpy().T[same], ref["gb2"][same])


@pytest.mark.parametrize("dims", [2, 3])
def test_boxes_far_from_origin(dims):
    """Box pairs with centres at scene coordinates up to +-5 km (float32 centres,
    rounded once there): the kernels build both boxes' corners relative to box 1's
    centre, so IoU (every pair), flags and parameter gradients (margin pairs) match
    the oracle on the same float parameters."""
    n = 20000
    b = synth.gen_box_pairs(n, dims)
    rng = np.random.default_rng(dims + 77)
    off = rng.uniform(-5e3, 5e3, (2, n))
    b1, b2 = b.b1.copy(), b.b2.copy()
    for p in range(2):   # cx, cy planes
        b1[p] = (b1[p].astype(np.float64) + off[p]).astype(np.float32)
        b2[p] = (b2[p].astype(np.float64) + off[p]).astype(np.float32)
    s = synth.BoxPairBatch(np.ascontiguousarray(b1), np.ascontiguousarray(b2), b.grad)
    iou, nx, xf, g1, g2 = gpu_box(s)
    r1, r2 = s.rows64()
    ref = oracle.box_iou_paired(r1, r2, s.grad.astype(np.float64))
    assert_iou_close(iou, ref["iou"])
    ok = box_margin_ok(r1, r2)
    assert ok.mean() > 0.8
    assert_flags_exact(nx[ok], xf[ok], {"nx": ref["nx"][ok], "xflags": ref["xflags"][ok]})
    assert_grad_close(g1.T[ok], ref["gb1"][ok])
    assert_grad_close(g2.T[ok], ref["gb2"][ok])


@pytest.mark.parametrize("dims", [2, 3])
def test_box_thin_pairs_interleaved(dims):
    """Thin box pairs (aspect 100-300, nearly aligned, up to 300 m from the origin) on every
    7th slot of a KITTI batch, so most CTAs of the box forward hold a few: a thread's thin
    pass (areas of the recorded intersection in double, after its own tile loop) runs while
    other warps of its CTA are still in theirs.  IoU of EVERY pair (split forward and
    fused kernel) against the oracle at 1e-5 (R18); the thin pairs do overlap.  Their
    areas come from corners rebuilt in double (float corners of a 60 m x 0.2 m box at
    300 m alone put 1.4e-5 on the IoU)."""
    n = 1 << 16
    b = synth.gen_box_pairs(n, dims, seed=4242 + dims)
    rng = np.random.default_rng(77 + dims)
    idx = np.arange(0, n, 7)
    m = idx.size
    length = rng.uniform(20.0, 60.0, m)
    width = length / rng.uniform(100.0, 300.0, m)
    cx, cy = rng.uniform(-300.0, 300.0, m), rng.uniform(-300.0, 300.0, m)
    th = rng.uniform(-math.pi, math.pi, m)
    along, across = rng.uniform(-0.3, 0.3, m) * length, rng.uniform(-0.5, 0.5, m) * width
    cx2 = cx + np.cos(th) * along - np.sin(th) * across
    cy2 = cy + np.sin(th) * along + np.cos(th) * across
    th2 = th + rng.normal(0.0, 1e-3, m)
    w2 = width * rng.uniform(0.8, 1.2, m)
    if dims == 2:
        b.b1[:, idx] = np.stack([cx, cy, length, width, th]).astype(np.float32)
        b.b2[:, idx] = np.stack([cx2, cy2, length, w2, th2]).astype(np.float32)
    else:
        cz, d = rng.normal(-1.0, 0.4, m), rng.uniform(1.4, 1.8, m)
        b.b1[:, idx] = np.stack([cx, cy, cz, length, width, d, th]).astype(np.float32)
        b.b2[:, idx] = np.stack([cx2, cy2, cz + 0.1 * d, length, w2, d, th2]).astype(np.float32)
    r1, r2 = b.rows64()
    ref = oracle.box_iou_paired(r1, r2, b.grad.astype(np.float64))
    assert (ref["iou"][idx] > 0).mean() > 0.9
    B1, B2 = torch.from_numpy(b.b1).to(dev()), torch.from_numpy(b.b2).to(dev())
    iou, nx, xf = dgal.box_iou_paired_fwd(B1, B2)
    assert_iou_close(iou.cpu().numpy(), ref["iou"])
    # the fused kernel queues the thin pairs; its refine pass redoes them with the same
    # double-precision corners
    iou_f, g1, g2 = dgal.box_iou_paired_fused(B1, B2, grad=torch.from_numpy(b.grad).to(dev()))
    assert_iou_close(iou_f.cpu().numpy(), ref["iou"])


@pytest.mark.parametrize("dims", [2, 3])
def test_box_thin_crossing_gradients(dims):
    """Thin boxes (aspect 100-300, 20-60 m long, up to 300 m from the origin) crossing at
    2-6 degrees — thin pairs (R^2 >> A_u) whose crossings are well conditioned: IoU of
    every pair at 1e-5, and on the margin pairs (R13) flags bit-exact and the parameter
    gradients (split backward and fused kernel) within 1e-4 abs or 1e-3 rel."""
    n = 4096
    rng = np.random.default_rng(91 + dims)
    length = rng.uniform(20.0, 60.0, n)
    width = length / rng.uniform(100.0, 300.0, n)
    cx, cy = rng.uniform(-300.0, 300.0, n), rng.uniform(-300.0, 300.0, n)
    th = rng.uniform(-math.pi, math.pi, n)
    along, across = rng.uniform(-0.3, 0.3, n) * length, rng.uniform(-0.5, 0.5, n) * width
    cx2 = cx + np.cos(th) * along - np.sin(th) * across
    cy2 = cy + np.sin(th) * along + np.cos(th) * across
    th2 = th + rng.choice([-1.0, 1.0], n) * rng.uniform(0.035, 0.1, n)
    w2 = width * rng.uniform(0.8, 1.2, n)
    if dims == 2:
        r1 = np.stack([cx, cy, length, width, th], 1)
        r2 = np.stack([cx2, cy2, length, w2, th2], 1)
    else:
        cz, d = rng.normal(-1.0, 0.4, n), rng.uniform(1.4, 1.8, n)
        r1 = np.stack([cx, cy, cz, length, width, d, th], 1)
        r2 = np.stack([cx2, cy2, cz + 0.1 * d, length, w2, d, th2], 1)
    b = _batch(r1, r2, rng.uniform(-1, 1, n))
    q1, q2 = b.rows64()
    ref = oracle.box_iou_paired(q1, q2, b.grad.astype(np.float64))
    assert (ref["iou"] > 0).mean() > 0.9
    iou, nx, xf, g1, g2 = gpu_box(b)
    assert_iou_close(iou, ref["iou"])
    ok = box_margin_ok(q1, q2)
    assert ok.mean() > 0.5
    assert_flags_exact(nx[ok], xf[ok], {"nx": ref["nx"][ok], "xflags": ref["xflags"][ok]})
    assert_grad_close(g1.T[ok], ref["gb1"][ok])
    assert_grad_close(g2.T[ok], ref["gb2"][ok])
    B1, B2 = torch.from_numpy(b.b1).to(dev()), torch.from_numpy(b.b2).to(dev())
    iou_f, f1, f2 = dgal.box_iou_paired_fused(B1, B2, grad=torch.from_numpy(b.grad).to(dev()))
    assert_iou_close(iou_f.cpu().numpy(), ref["iou"])
    assert_grad_close(f1.cpu().numpy().T[ok], ref["gb1"][ok])
    assert_grad_close(f2.cpu().numpy().T[ok], ref["gb2"][ok])


@pytest.mark.parametrize("dims", [2, 3])
def test_box_unbounded_theta(dims):
    """theta is accepted unbounded: KITTI pairs with both angles shifted by a
    common U(-1000, 1000) rad — IoU of every pair at 1e-5 against the oracle (cos / sin
    of the float theta in double), flags bit-exact on the margin pairs.  (A float
    theta * (1/pi) alone put 9e-5 on the IoU at |theta| ~ 1000.)"""
    b = synth.gen_box_pairs(1 << 15, dims, seed=99)
    rng = np.random.default_rng(5)
    sh = rng.uniform(-1000.0, 1000.0, b.n).astype(np.float32)
    ti = 4 if dims == 2 else 6
    b.b1[ti] += sh
    b.b2[ti] += sh
    iou, nx, xf, g1, g2 = gpu_box(b)
    r1, r2 = b.rows64()
    ref = oracle.box_iou_paired(r1, r2, b.grad.astype(np.float64))
    assert_iou_close(iou, ref["iou"])
    ok = box_margin_ok(r1, r2)
    assert_flags_exact(nx[ok], xf[ok], {"nx": ref["nx"][ok], "xflags": ref["xflags"][ok]})
    assert_grad_close(g1.T[ok], ref["gb1"][ok])
    assert_grad_close(g2.T[ok], ref["gb2"][ok])


@pytest.mark.parametrize("dims", [2, 3])
def test_box_small_far_from_origin(dims):
    """KITTI pairs shrunk to 5 % (~20 x 8 cm boxes, centres within 3.5 m) and moved 10 km
    from the origin (float parameters): IoU of every pair at 1e-5 and flags on the margin
    pairs against the oracle (both work about the pair, not the origin)."""
    b = synth.gen_box_pairs(1 << 15, dims, seed=7)
    sz = (2, 3) if dims == 2 else (2, 3, 4, 5)
    for bb in (b.b1, b.b2):
        bb[0] = bb[0] * np.float32(0.05) + np.float32(1e4)
        bb[1] = bb[1] * np.float32(0.05) - np.float32(1e4)
        for r in sz:
            bb[r] *= np.float32(0.05)
    iou, nx, xf, g1, g2 = gpu_box(b)
    r1, r2 = b.rows64()
    ref = oracle.box_iou_paired(r1, r2, b.grad.astype(np.float64))
    assert (ref["iou"] > 0).mean() > 0.8
    assert_iou_close(iou, ref["iou"])
    ok = box_margin_ok(r1, r2)
    assert_flags_exact(nx[ok], xf[ok], {"nx": ref["nx"][ok], "xflags": ref["xflags"][ok]})
    assert_grad_close(g1.T[ok], ref["gb1"][ok])
    assert_grad_close(g2.T[ok], ref["gb2"][ok])


@pytest.mark.parametrize("cz", [1e3, 1e4])
def test_box3d_high_centres(cz):
    """3D KITTI pairs lifted by a common cz (global-frame heights): V_i / V_u is invariant
    under a vertical shift, and the z overlap is taken relative to box 1's centre — IoU of
    every pair (split and fused) at 1e-5, flags and gradients on the margin pairs."""
    b = synth.gen_box_pairs(1 << 14, 3, seed=21)
    b.b1[2] += np.float32(cz)
    b.b2[2] += np.float32(cz)
    iou, nx, xf, g1, g2 = gpu_box(b)
    r1, r2 = b.rows64()
    ref = oracle.box_iou_paired(r1, r2, b.grad.astype(np.float64))
    assert_iou_close(iou, ref["iou"])
    ok = box_margin_ok(r1, r2)
    assert_flags_exact(nx[ok], xf[ok], {"nx": ref["nx"][ok], "xflags": ref["xflags"][ok]})
    assert_grad_close(g1.T[ok], ref["gb1"][ok])
    assert_grad_close(g2.T[ok], ref["gb2"][ok])
    B1, B2 = torch.from_numpy(b.b1).to(dev()), torch.from_numpy(b.b2).to(dev())
    iou_f, f1, f2 = dgal.box_iou_paired_fused(B1, B2, grad=torch.from_numpy(b.grad).to(dev()))
    assert_iou_close(iou_f.cpu().numpy(), ref["iou"])
    assert_grad_close(f1.cpu().numpy().T[ok], ref["gb1"][ok])
    assert_grad_close(f2.cpu().numpy().T[ok], ref["gb2"][ok])
