"""T0 (CPU): the oracle's iou_grad pinned to central finite differences, the
invariances IoU has, and closed forms (SURVEY §8(c) "Gradients")."""
import json
import math
import os

import numpy as np
import pytest

import oracle
from helpers import as_pairs, box, bwd1, decode, margin_batch, regular

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_worked_examples.json")))
SQ = np.array([[0, 0], [1, 0], [1, 1], [0, 1]], float)


def _fd_check(b, h_rel=1e-7):
    """Central FD of the oracle IoU w.r.t. all 4K coordinates, on the
    pairs whose nx/flags are unchanged under every +-h perturbation.  Each pair is
    first translated near the origin (IoU and its gradient are translation
    invariant) so the FD rounding error is set by the polygon size, not by the
    scene coordinates; h = 1e-7 x that size balances truncation and rounding."""
    K, n = b.p1.K, b.n
    X1, Y1 = b.p1.xy64()
    X2, Y2 = b.p2.xy64()
    ox, oy = X1.mean(1, keepdims=True), Y1.mean(1, keepdims=True)
    X1, X2, Y1, Y2 = X1 - ox, X2 - ox, Y1 - oy, Y2 - oy
    base = np.stack([X1, Y1, X2, Y2], 1)            # (n, 4, K)
    scale = np.abs(base).max(axis=(1, 2)) + 1.0
    h = h_rel * scale
    f0 = oracle.iou_paired_fwd((X1, Y1), (X2, Y2))
    pert = np.repeat(base[:, None], 8 * K, axis=1)   # (n, 8K, 4, K)
    for c in range(4 * K):
        plane, v = divmod(c, K)
        pert[:, 2 * c, plane, v] += h
        pert[:, 2 * c + 1, plane, v] -= h
    P = pert.reshape(-1, 4, K)
    fp = oracle.iou_paired_fwd((P[:, 0], P[:, 1]), (P[:, 2], P[:, 3]))
    iou = fp["iou"].reshape(n, 4 * K, 2)
    fd = (iou[..., 0] - iou[..., 1]) / (2 * h[:, None])   # (n, 4K)
    stable = np.ones(n, bool)
    nxp = fp["nx"].reshape(n, 8 * K)
    xfp = fp["xflags"].reshape(n, 8 * K, -1)
    stable &= np.all(nxp == f0["nx"][:, None], axis=1)
    stable &= np.all(xfp == f0["xflags"][:, None, :], axis=(1, 2))
    gx1, gy1, gx2, gy2 = oracle.iou_paired_bwd((X1, Y1), (X2, Y2), np.ones(n))
    an = np.concatenate([gx1, gy1, gx2, gy2], 1)        # (n, 4K), same order as fd
    return an, fd, stable


@pytest.mark.parametrize("cfg", [1, 3, 4])
def test_grad_vs_central_fd(cfg):
    b = margin_batch(cfg, 300)
    an, fd, stable = _fd_check(b)
    assert stable.mean() > 0.9                         # exclusions < 10%
    a, d = an[stable], fd[stable]
    err = np.abs(a - d)
    tol = 1e-6 * np.maximum(1.0, np.abs(d)).max(axis=1, keepdims=True)
    assert np.all(err <= tol), err.max()


@pytest.mark.parametrize("cfg", [1, 3, 4])
def test_grad_invariances(cfg):
    """IoU is invariant under translation, rotation and scaling of both polygons:
    sum g = 0, sum v x g = 0, sum v . g = 0 (exact identities of the true gradient)."""
    b = margin_batch(cfg, 500)
    X1, Y1 = b.p1.xy64()
    X2, Y2 = b.p2.xy64()
    gx1, gy1, gx2, gy2 = oracle.iou_paired_bwd((X1, Y1), (X2, Y2), np.ones(b.n))
    X = np.concatenate([X1, X2], 1)
    Y = np.concatenate([Y1, Y2], 1)
    GX = np.concatenate([gx1, gx2], 1)
    GY = np.concatenate([gy1, gy2], 1)
    mag = np.abs(GX).sum(1) + np.abs(GY).sum(1) + 1e-300
    L = np.abs(X).max(1) + np.abs(Y).max(1)
    assert np.all(np.abs(GX.sum(1)) <= 1e-12 * mag)
    assert np.all(np.abs(GY.sum(1)) <= 1e-12 * mag)
    assert np.all(np.abs((X * GY - Y * GX).sum(1)) <= 1e-12 * mag * L)
    assert np.all(np.abs((X * GX + Y * GY).sum(1)) <= 1e-12 * mag * L)


def _area_grad(P):
    """Closed form dA/dv_k = ((y_{k+1}-y_{k-1})/2, (x_{k-1}-x_{k+1})/2) — S:268."""
    nxt, prv = np.roll(P, -1, 0), np.roll(P, 1, 0)
    return np.stack([(nxt[:, 1] - prv[:, 1]) / 2, (prv[:, 0] - nxt[:, 0]) / 2], 1)


def test_area_grad_worked_example_via_subset():
    """p1 = unit square strictly inside p2 => grad_p1 = dA1/A2 (subset closed form),
    so dIoU/dx_0 * A2 must equal the SPEC's dA/dx_0 = -0.5."""
    Q = np.array([[-10, -10], [10, -10], [10, 10], [-10, 10]], float)
    g1, g2 = bwd1(SQ, Q)
    assert abs(g1[0, 0] * 400.0 - GOLD["area_grad_unit_square_v0"]["dA_dx0"]) < 1e-14


def test_identical_closed_form():
    """Identical polygons (all FromP1; the P1 ⊂ P2 piece, R9): IoU = A1/A2 so
    grad_p1 = g dA/A, grad_p2 = -g dA/A."""
    rng = np.random.default_rng(3)
    for _ in range(50):
        K = int(rng.integers(4, 9))
        P = regular(K, rng.uniform(1, 3), rng.uniform(0, 6)) * [1.0, rng.uniform(0.5, 1)]
        g = rng.uniform(-2, 2)
        g1, g2 = bwd1(P, P.copy(), g)
        A = 0.5 * np.sum(P[:, 0] * np.roll(P[:, 1], -1) - np.roll(P[:, 0], -1) * P[:, 1])
        want = g * _area_grad(P) / A
        np.testing.assert_allclose(g1, want, rtol=1e-13, atol=1e-15)
        np.testing.assert_allclose(g2, -want, rtol=1e-13, atol=1e-15)


def test_subset_closed_form():
    rng = np.random.default_rng(4)
    for _ in range(50):
        K = int(rng.integers(4, 9))
        Q = regular(K, rng.uniform(2, 4), rng.uniform(0, 6))
        P = Q * rng.uniform(0.2, 0.8) + rng.uniform(-0.05, 0.05, 2)
        g1, g2 = bwd1(P, Q)
        A1 = 0.5 * np.sum(P[:, 0] * np.roll(P[:, 1], -1) - np.roll(P[:, 0], -1) * P[:, 1])
        A2 = 0.5 * np.sum(Q[:, 0] * np.roll(Q[:, 1], -1) - np.roll(Q[:, 0], -1) * Q[:, 1])
        np.testing.assert_allclose(g1, _area_grad(P) / A2, rtol=1e-12, atol=1e-15)
        np.testing.assert_allclose(g2, -A1 * _area_grad(Q) / A2 ** 2, rtol=1e-12, atol=1e-15)


def test_axis_aligned_xmax_derivative():
    """Sum of g_x over p1's two right-edge vertices = d/dx1max of the rectangle
    closed form IoU = Ix Iy / (A1 + A2 - Ix Iy) (x1max binding, x2max not)."""
    rng = np.random.default_rng(8)
    for _ in range(100):
        x0, y0 = rng.uniform(-1, 1, 2)
        x1, y1 = x0 + rng.uniform(1, 3), y0 + rng.uniform(1, 3)
        u0, v0 = x0 + rng.uniform(0.1, 0.8), y0 + rng.uniform(-0.8, 0.8)
        u1, v1 = x1 + rng.uniform(0.1, 2), v0 + rng.uniform(1, 3)
        P = np.array([[x0, y0], [x1, y0], [x1, y1], [x0, y1]])
        Q = np.array([[u0, v0], [u1, v0], [u1, v1], [u0, v1]])
        ix, iy = x1 - u0, min(y1, v1) - max(y0, v0)
        A1, A2, I = (x1 - x0) * (y1 - y0), (u1 - u0) * (v1 - v0), ix * iy
        U = A1 + A2 - I
        dI, dA1 = iy, (y1 - y0)
        want = (dI * U - I * (dA1 - dI)) / U ** 2
        g1, _ = bwd1(P, Q)
        assert abs(g1[1, 0] + g1[2, 0] - want) < 1e-13


def test_offset_squares_dIoU_dAi():
    g = GOLD["offset_squares"]
    P, Q = np.array(g["p1"], float), np.array(g["p2"], float)
    g1, g2 = bwd1(P, Q)
    # vertex 2 of p1 = (1,1): dIoU/dx2 = cu dA1/dx2 + ci dAi/dx2.
    # dA1/dx2 = (y3 - y1)/2 = 0.5.  Moving v2 to (1+d, 1) tilts p1's right
    # edge to x = 1 + d*y, so Ai(d) = int_{0.5}^{1} (0.5 + d*y) dy = 0.25 + 0.375 d:
    # dAi/dx2 = 0.375 (same for y by the diagonal symmetry).
    ci = g["dIoU_dAi"]
    cu = -g["area_i"] / g["area_u"] ** 2
    want = cu * 0.5 + ci * 0.375
    assert abs(g1[2, 0] - want) < 1e-7 and abs(g1[2, 1] - want) < 1e-7


def test_bitwise_linearity():
    b = margin_batch(1, 1000)
    X1, Y1 = b.p1.xy64()
    X2, Y2 = b.p2.xy64()
    g = b.grad.astype(np.float64)
    r1 = oracle.iou_paired_bwd((X1, Y1), (X2, Y2), g)
    r2 = oracle.iou_paired_bwd((X1, Y1), (X2, Y2), 2 * g)
    r3 = oracle.iou_paired_bwd((X1, Y1), (X2, Y2), -g)
    for a, b2, c in zip(r1, r2, r3):
        assert np.array_equal(b2, 2 * a)
        assert np.array_equal(c, -a)


def test_disjoint_zero_grad():
    g1, g2 = bwd1(SQ, SQ + 5.0, 3.0)
    assert np.all(g1 == 0) and np.all(g2 == 0)
    g1, g2 = bwd1(SQ, SQ + [1.0, 0.0], 3.0)             # touching edge: empty
    assert np.all(g1 == 0) and np.all(g2 == 0)


def test_ascent_step_increases_iou():
    P, Q = SQ, SQ + 0.5
    g1, g2 = bwd1(P, Q)
    from helpers import fwd1
    i0 = fwd1(P, Q)[0]
    i1 = fwd1(P, Q + 1e-3 * g2)[0]
    assert i1 > i0
