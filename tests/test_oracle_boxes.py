"""T0 (CPU): the rotated-box front end of the oracle (SPEC
metrics-boxes S:336-418) pinned to the worked examples, closed forms, invariants,
central finite differences and a Monte-Carlo volume estimate that shares no
code with the clipping path (point-in-box tests only)."""
import math

import numpy as np
import pytest

import oracle
import synth
from helpers import box_margin_batch, footprint

PI = math.pi


def biou(b1, b2, grad=None):
    return oracle.box_iou_paired(np.atleast_2d(b1), np.atleast_2d(b2), grad)


# --- box_to_polygon --------------------------------------------
def test_corners_axis_square():
    x, y = oracle.box_corners([[0, 0, 2, 2, 0]])
    assert np.allclose(np.stack([x[0], y[0]], 1), [[-1, -1], [1, -1], [1, 1], [-1, 1]], atol=1e-15)


def test_corners_rotated_square_is_vertex_rotation():
    x, y = oracle.box_corners([[0, 0, 2, 2, PI / 2]])
    got = np.stack([x[0], y[0]], 1)
    ref = np.array([[-1, -1], [1, -1], [1, 1], [-1, 1]], float)
    assert any(np.allclose(got, np.roll(ref, s, 0), atol=1e-12) for s in range(4))


def test_corners_rotated_rectangle():
    x, y = oracle.box_corners([[1, 1, 2, 4, PI / 2]])
    got = np.stack([x[0], y[0]], 1)
    assert np.allclose(got, [[3, 0], [3, 2], [-1, 2], [-1, 0]], atol=1e-12)
    # CCW: positive shoelace area = w h
    assert math.isclose(oracle.area(x, y)[0], 8.0, rel_tol=1e-14)


# --- box_to_polygon_grad ----------------------------------------
def test_corner_vjp_translation_channel():
    rng = np.random.default_rng(0)
    b = np.array([[rng.normal(), rng.normal(), 2.0, 3.0, 0.7]])
    g = oracle.box_corners_vjp(b, np.ones((1, 4)), np.zeros((1, 4)))
    assert math.isclose(g[0, 0], 4.0) and abs(g[0, 1]) < 1e-15


def test_corner_vjp_readoff_at_theta0():
    gx = np.zeros((1, 4)); gx[0, 2] = 1.0                        # corner (+w/2, +h/2) is #2
    g = oracle.box_corners_vjp(np.array([[0.3, -0.2, 2.0, 3.0, 0.0]]), gx, np.zeros((1, 4)))
    assert math.isclose(g[0, 2], 0.5) and abs(g[0, 3]) < 1e-15
    assert math.isclose(g[0, 0], 1.0) and abs(g[0, 1]) < 1e-15
    # d/dtheta at theta=0 of x-corner (w/2 c - h/2 s) = -h/2
    assert math.isclose(g[0, 4], -1.5)


def test_corner_vjp_zero_cotangent():
    g = oracle.box_corners_vjp(np.array([[1, 2, 3, 4, 5.0]]), np.zeros((1, 4)), np.zeros((1, 4)))
    assert np.all(g == 0)


def test_corner_vjp_matches_fd():                                 # S:357 (Jacobian)
    rng = np.random.default_rng(1)
    b = np.column_stack([rng.normal(size=20), rng.normal(size=20), rng.uniform(0.5, 4, 20),
                         rng.uniform(0.5, 4, 20), rng.uniform(-4, 4, 20)])
    gx, gy = rng.normal(size=(20, 4)), rng.normal(size=(20, 4))
    an = oracle.box_corners_vjp(b, gx, gy)
    h = 1e-6
    for p in range(5):
        bp, bm = b.copy(), b.copy()
        bp[:, p] += h; bm[:, p] -= h
        xp, yp = oracle.box_corners(bp)
        xm, ym = oracle.box_corners(bm)
        fd = ((xp - xm) * gx + (yp - ym) * gy).sum(1) / (2 * h)
        assert np.allclose(an[:, p], fd, atol=1e-8), p


# --- box_iou_2d --------------------------------------------------
def test_identical_boxes_iou_one():
    r = biou([3, -2, 4, 1.5, 0.4], [3, -2, 4, 1.5, 0.4])
    assert r["iou"][0] == 1.0


def test_square_vs_45deg_octagon():
    r = biou([0, 0, 2, 2, 0], [0, 0, 2, 2, PI / 4])
    ai = 8 * (math.sqrt(2) - 1)
    assert r["nx"][0] == 8
    assert math.isclose(r["iou"][0], ai / (8 - ai), rel_tol=1e-12)
    assert math.isclose(r["iou"][0], 1 / math.sqrt(2), rel_tol=1e-12)


def test_disjoint_boxes():
    r = biou([0, 0, 2, 2, 0.3], [10, 0, 2, 2, 1.1], grad=[1.0])
    assert r["iou"][0] == 0.0 and r["nx"][0] == 0
    assert np.all(r["gb1"] == 0) and np.all(r["gb2"] == 0)


# --- box_iou_2d_grad ---------------------------------------------
def test_identical_boxes_stationary_translation():
    r = biou([3, -2, 4, 1.5, 0.4], [3, -2, 4, 1.5, 0.4], grad=[1.0])
    assert abs(r["gb1"][0, 0]) < 1e-9 and abs(r["gb1"][0, 1]) < 1e-9
    assert abs(r["gb2"][0, 0]) < 1e-9 and abs(r["gb2"][0, 1]) < 1e-9


def test_zero_grad_gives_zero():
    b = box_margin_batch(2, 50)
    r1, r2 = b.rows64()
    r = oracle.box_iou_paired(r1, r2, np.zeros(b.n))
    assert np.all(r["gb1"] == 0) and np.all(r["gb2"] == 0)


def _fd_boxes(r1, r2, h_rel=1e-7):
    """Central FD of IoU w.r.t. all 2P box parameters, stable pairs only.
    Pairs are translated to the origin first (IoU is translation invariant)."""
    r1, r2 = r1.copy(), r2.copy()
    r2[:, 0] -= r1[:, 0]; r2[:, 1] -= r1[:, 1]
    r1[:, 0] = 0.0; r1[:, 1] = 0.0
    n, P = r1.shape
    base = np.concatenate([r1, r2], 1)
    h = h_rel * (np.abs(base).max(1) + 1.0)
    f0 = oracle.box_iou_paired(r1, r2)
    pert = np.repeat(base[:, None], 4 * P, axis=1)
    for c in range(2 * P):
        pert[:, 2 * c, c] += h
        pert[:, 2 * c + 1, c] -= h
    Q = pert.reshape(-1, 2 * P)
    fp = oracle.box_iou_paired(Q[:, :P], Q[:, P:])
    iou = fp["iou"].reshape(n, 2 * P, 2)
    fd = (iou[..., 0] - iou[..., 1]) / (2 * h[:, None])
    stable = np.all(fp["nx"].reshape(n, 4 * P) == f0["nx"][:, None], 1)
    stable &= np.all(fp["xflags"].reshape(n, 4 * P, 8) == f0["xflags"][:, None], axis=(1, 2))
    g = oracle.box_iou_paired(r1, r2, np.ones(n))
    an = np.concatenate([g["gb1"], g["gb2"]], 1)
    return an, fd, stable & (f0["iou"] > 0)


@pytest.mark.parametrize("dims", [2, 3])
def test_box_grad_vs_central_fd(dims):
    b = box_margin_batch(dims, 300)
    r1, r2 = b.rows64()
    an, fd, stable = _fd_boxes(r1, r2)
    assert stable.mean() > 0.85
    a, d = an[stable], fd[stable]
    err = np.abs(a - d)
    tol = 1e-6 * np.maximum(1.0, np.abs(d).max(axis=1, keepdims=True))   # S:381 asks < 1e-4
    assert np.all(err <= tol), err.max()


# --- invariants ---------------------------------------------------
def test_symmetry_range_periodicity_rigid():
    b = box_margin_batch(2, 200)
    r1, r2 = b.rows64()
    i12 = oracle.box_iou_paired(r1, r2)["iou"]
    i21 = oracle.box_iou_paired(r2, r1)["iou"]
    assert np.max(np.abs(i12 - i21)) < 1e-9
    assert np.all((i12 >= 0) & (i12 <= 1))
    s1 = r1.copy(); s1[:, 4] += 2 * PI
    assert np.max(np.abs(oracle.box_iou_paired(s1, r2)["iou"] - i12)) < 1e-9
    # common rigid motion about the first centre
    a = 0.7
    c, s = math.cos(a), math.sin(a)
    def move(r):
        q = r.copy()
        dx, dy = r[:, 0] - r1[:, 0], r[:, 1] - r1[:, 1]
        q[:, 0] = r1[:, 0] + c * dx - s * dy + 3.0
        q[:, 1] = r1[:, 1] + s * dx + c * dy - 1.0
        q[:, 4] += a
        return q
    assert np.max(np.abs(oracle.box_iou_paired(move(r1), move(r2))["iou"] - i12)) < 1e-7


# --- box_iou_3d --------------------------------------------
def test_3d_identical_unit_cubes():
    r = biou([0, 0, 0, 1, 1, 1, 0], [0, 0, 0, 1, 1, 1, 0])
    assert r["iou"][0] == 1.0


def test_3d_offset_unit_cubes():
    r = biou([0, 0, 0, 1, 1, 1, 0], [0.5, 0.5, 0.5, 1, 1, 1, 0])
    assert math.isclose(r["iou"][0], 1 / 15, rel_tol=1e-12)


def test_3d_stacked_cubes_zero_and_zero_grad():
    r = biou([0, 0, 0, 1, 1, 1, 0.2], [0.1, 0, 1.0, 1, 1, 1, 0.0], grad=[1.0])
    assert r["iou"][0] == 0.0
    assert np.all(r["gb1"] == 0) and np.all(r["gb2"] == 0)


def test_3d_reduces_to_2d():
    b = box_margin_batch(3, 200)
    r1, r2 = b.rows64()
    r2 = r2.copy(); r2[:, 2] = r1[:, 2]; r2[:, 5] = r1[:, 5]
    i3 = oracle.box_iou_paired(r1, r2)["iou"]
    i2 = oracle.box_iou_paired(footprint(r1), footprint(r2))["iou"]
    assert np.max(np.abs(i3 - i2)) < 1e-12


def test_3d_dz_gradient_closed_form():                            # S:387 (product rule through dz)
    # axis-aligned unit cubes, box 2 shifted by z0 in z only: IoU = (1-z0)/(1+z0)
    z0 = 0.3
    r = biou([0, 0, 0, 1, 1, 1, 0], [0, 0, z0, 1, 1, 1, 0], grad=[1.0])
    assert math.isclose(r["iou"][0], (1 - z0) / (1 + z0), rel_tol=1e-12)
    assert math.isclose(r["gb2"][0, 2], -2 / (1 + z0) ** 2, rel_tol=1e-12)
    assert math.isclose(r["gb1"][0, 2], 2 / (1 + z0) ** 2, rel_tol=1e-12)


def _point_in_box(px, py, b):
    """Point-in-rotated-rectangle by local coordinates (no polygon clipping)."""
    c, s = math.cos(b[-1]), math.sin(b[-1])
    dx, dy = px - b[0], py - b[1]
    u, v = c * dx + s * dy, -s * dx + c * dy
    w, h = (b[3], b[4]) if len(b) == 7 else (b[2], b[3])
    return (np.abs(u) <= w / 2) & (np.abs(v) <= h / 2)


@pytest.mark.parametrize("dims", [2, 3])
def test_monte_carlo_volume(dims):                                # S:391 cross-check
    b = box_margin_batch(dims, 40, seed=77)
    r1, r2 = b.rows64()
    ref = oracle.box_iou_paired(r1, r2)["iou"]
    rng = np.random.default_rng(5)
    Nmc = 200_000
    for k in range(b.n):
        a, c = r1[k], r2[k]
        R = max(math.hypot(*footprint(a[None])[0, 2:4]), math.hypot(*footprint(c[None])[0, 2:4])) / 2
        lo = np.minimum(a[:2], c[:2]) - R
        hi = np.maximum(a[:2], c[:2]) + R
        px = rng.uniform(lo[0], hi[0], Nmc)
        py = rng.uniform(lo[1], hi[1], Nmc)
        vol = (hi[0] - lo[0]) * (hi[1] - lo[1])
        in1, in2 = _point_in_box(px, py, a), _point_in_box(px, py, c)
        if dims == 3:
            zl = min(a[2] - a[5] / 2, c[2] - c[5] / 2)
            zh = max(a[2] + a[5] / 2, c[2] + c[5] / 2)
            pz = rng.uniform(zl, zh, Nmc)
            vol *= zh - zl
            in1 &= np.abs(pz - a[2]) <= a[5] / 2
            in2 &= np.abs(pz - c[2]) <= c[5] / 2
        p_i, p_u = np.mean(in1 & in2), np.mean(in1 | in2)
        est = p_i / p_u if p_u > 0 else 0.0
        # ratio estimator sd ~ sqrt(p_i (1 - p_i / p_u) / N) / p_u
        sd = math.sqrt(max(p_i * (1 - est), 1e-12) / Nmc) / max(p_u, 1e-12)
        assert abs(est - ref[k]) <= 5 * sd + 1e-4, (k, est, ref[k], sd)


def test_translation_invariance_far_from_origin():
    """S:397 rigid invariance at 10 km: KITTI box pairs shrunk to 5 % (~20 x 8 cm) and
    translated by (1e4, -1e4) exactly give the same 2D / 3D IoU within 1e-9."""
    for dims in (2, 3):
        b = synth.gen_box_pairs(4000, dims, seed=11)
        r1, r2 = b.rows64()
        sz = [2, 3] if dims == 2 else [2, 3, 4, 5]
        for r in (r1, r2):
            r[:, 0] *= 0.05
            r[:, 1] *= 0.05
            r[:, sz] *= 0.05
        i0 = oracle.box_iou_paired(r1, r2)["iou"]
        f1, f2 = r1.copy(), r2.copy()
        for r in (f1, f2):
            r[:, 0] += 1e4
            r[:, 1] -= 1e4
        assert (i0 > 0).mean() > 0.8
        assert np.max(np.abs(oracle.box_iou_paired(f1, f2)["iou"] - i0)) < 1e-9
