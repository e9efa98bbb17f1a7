"""T0 (CPU): the forward oracle pinned to the paper / SPEC worked examples, closed
forms, exact rational brute force, rasterisation and invariants — never to itself.
Citations: P:n = PAPER.md line n, S:n = SPEC.md line n (golden file holds the values)."""
import json
import math
import os
from fractions import Fraction

import numpy as np
import pytest

import oracle
import synth
from helpers import as_pairs, box, bwd1, decode, fwd1, margin_batch, regular

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_worked_examples.json")))
SQ = np.array([[0, 0], [1, 0], [1, 1], [0, 1]], float)


def test_area_worked_examples():
    g = GOLD["area_unit_square"]
    P = np.array(g["poly"], float)
    assert oracle.area(P[None, :, 0], P[None, :, 1])[0] == g["area"]
    g = GOLD["area_triangle"]
    P = np.array(g["poly"], float)
    assert oracle.area(P[None, :, 0], P[None, :, 1])[0] == g["area"]


def test_identical_squares():
    g = GOLD["identical_squares"]
    iou, nx, fl, _ = fwd1(np.array(g["p1"], float), np.array(g["p2"], float))
    assert iou == g["iou"] and nx == g["nx"] and fl == g["xflags"]


def test_offset_squares():
    g = GOLD["offset_squares"]
    P, Q = np.array(g["p1"], float), np.array(g["p2"], float)
    iou, nx, fl, ai = fwd1(P, Q)
    assert abs(iou - 1 / 7) < 1e-15 and abs(iou - g["iou"]) < 1e-15
    assert ai == g["area_i"] and nx == g["nx"]
    assert fl == g["xflags"]
    # same cyclic sequence as the SPEC's hand construction, rotated (R3)
    sh = g["flags_sh_order"]
    assert any(fl == sh[r:] + sh[:r] for r in range(4))
    verts, flags, (A1, A2, Ai) = oracle.intersect_one(P, Q)
    got = {tuple(v) for v in np.round(verts, 12)}
    assert got == {tuple(v) for v in g["vertices_up_to_rotation"]}
    assert abs((A1 + A2 - Ai) - g["area_u"]) < 1e-15


def test_disjoint_squares():
    iou, nx, fl, ai = fwd1(SQ, SQ + 5.0)
    assert iou == 0.0 and nx == 0 and fl == [] and ai == 0.0


def test_square_vs_45deg():
    g = GOLD["square_vs_45deg"]
    iou, nx, fl, ai = fwd1(box(*g["box1"]), box(*g["box2"]))
    assert abs(ai - 8 * (math.sqrt(2) - 1)) < 1e-12
    assert abs(iou - g["iou"]) < 1e-12 and nx == g["nx"]
    assert all(decode(b)[0] == 3 for b in fl)


@pytest.mark.parametrize("n", [4, 8])
def test_regular_ngons_rotated(n):
    """Two regular n-gons, same centre and apothem, rotated by pi/n intersect in a
    regular 2n-gon: IoU = cos(pi/n) (derived in DESIGN.md §3.5); nx = 2n, all Cross,
    each p1 edge crossed exactly twice."""
    a = 1.7
    R = a / math.cos(math.pi / n)
    P = regular(n, R, 0.3)
    Q = regular(n, R, 0.3 + math.pi / n)
    iou, nx, fl, _ = fwd1(P, Q)
    assert abs(iou - math.cos(math.pi / n)) < 1e-12
    assert nx == 2 * n
    tags = [decode(b) for b in fl]
    assert all(t == 3 for t, _, _ in tags)
    for i in range(n):
        assert sum(1 for _, ii, _ in tags if ii == i) == 2


def test_subset_and_superset():
    rng = np.random.default_rng(5)
    for _ in range(50):
        K = int(rng.integers(4, 9))
        Q = regular(K, rng.uniform(2, 4), rng.uniform(0, 6)) + rng.uniform(-5, 5, 2)
        c = Q.mean(0)
        P = c + (Q - c) * rng.uniform(0.2, 0.8)
        P = P + rng.uniform(-0.05, 0.05, 2)
        iou, nx, fl, ai = fwd1(P, Q)
        A1 = oracle.area(P[None, :, 0], P[None, :, 1])[0]
        A2 = oracle.area(Q[None, :, 0], Q[None, :, 1])[0]
        assert abs(iou - A1 / A2) < 1e-12
        assert nx == K and fl == [0x40 | k for k in range(K)]
        iou, nx, fl, ai = fwd1(Q, P)                  # p2 strictly inside p1
        assert abs(iou - A1 / A2) < 1e-12
        assert nx == K and fl == [0x80 | k for k in range(K)]


def test_axis_aligned_closed_form():
    rng = np.random.default_rng(7)
    P_list, Q_list, want = [], [], []
    for _ in range(300):
        x0, y0 = rng.uniform(-3, 3, 2)
        x1, y1 = x0 + rng.uniform(0.3, 4), y0 + rng.uniform(0.3, 4)
        u0, v0 = rng.uniform(-3, 3, 2)
        u1, v1 = u0 + rng.uniform(0.3, 4), v0 + rng.uniform(0.3, 4)
        ix = max(0.0, min(x1, u1) - max(x0, u0))
        iy = max(0.0, min(y1, v1) - max(y0, v0))
        I = ix * iy
        want.append(I / ((x1 - x0) * (y1 - y0) + (u1 - u0) * (v1 - v0) - I))
        P_list.append(np.array([[x0, y0], [x1, y0], [x1, y1], [x0, y1]]))
        Q_list.append(np.array([[u0, v0], [u1, v0], [u1, v1], [u0, v1]]))
    p1, p2 = as_pairs(P_list, Q_list)
    got = oracle.iou_paired_fwd(p1, p2)["iou"]
    np.testing.assert_allclose(got, want, rtol=0, atol=1e-13)


def _relabel_swap(flags):
    out = []
    for b in flags:
        t, i, j = decode(b)
        out.append({1: 0x80 | j, 2: 0x40 | j, 3: 0xC0 | (j << 3) | i}[t])
    return out


def _canon(seq):
    if not seq:
        return seq
    s = seq.index(min(seq))
    return seq[s:] + seq[:s]


def test_symmetry_and_role_swap():
    b = synth.gen_cfg1_pairs(2000)
    f = oracle.iou_paired_fwd(b.p1, b.p2)
    r = oracle.iou_paired_fwd(b.p2, b.p1)
    np.testing.assert_allclose(f["iou"], r["iou"], rtol=0, atol=1e-12)
    ok = oracle.margin_ok(b.p1, b.p2)
    for k in np.nonzero(ok)[0][:500]:
        n1, n2 = f["nx"][k], r["nx"][k]
        assert n1 == n2
        a = [int(x) for x in f["xflags"][k][:n1]]
        bb = [int(x) for x in r["xflags"][k][:n2]]
        assert _canon(_relabel_swap(bb)) == _canon(a)


@pytest.mark.parametrize("cfg", [1, 3, 4])
def test_bounds_and_nx_range(cfg):
    b = synth.gen_config(cfg, 4000)
    f = oracle.iou_paired_fwd(b.p1, b.p2)
    assert np.all(f["iou"] >= 0) and np.all(f["iou"] <= 1)
    A1 = oracle.area(*b.p1.xy64())
    A2 = oracle.area(*b.p2.xy64())
    assert np.all(f["area_i"] <= np.minimum(A1, A2) * (1 + 1e-12))
    ne = f["nx"] > 0
    K = b.p1.K
    assert np.all(f["nx"][ne] >= 3) and np.all(f["nx"][ne] <= 2 * K)
    assert np.all(f["status"] == 0)
    if K == 4:
        g = GOLD["rectangles_nx_range"]
        assert f["nx"][ne].min() >= g["min"] and f["nx"][ne].max() <= g["max"]
    # padding bytes are 0x00, valid bytes never are
    for k in range(200):
        n = f["nx"][k]
        assert np.all(f["xflags"][k][n:] == 0) and np.all(f["xflags"][k][:n] != 0)


# ---------------------------------------------------------------------------
# exact rational brute force on lattice polygons
# ---------------------------------------------------------------------------
def _hull(points):
    pts = sorted(set(points))
    if len(pts) < 3:
        return pts

    def cr(o, a, b):
        return (a[0] - o[0]) * (b[1] - o[1]) - (a[1] - o[1]) * (b[0] - o[0])
    lo, hi = [], []
    for p in pts:
        while len(lo) >= 2 and cr(lo[-2], lo[-1], p) <= 0:
            lo.pop()
        lo.append(p)
    for p in reversed(pts):
        while len(hi) >= 2 and cr(hi[-2], hi[-1], p) <= 0:
            hi.pop()
        hi.append(p)
    return lo[:-1] + hi[:-1]


def _exact_clip_area(P, Q):
    """Exact (Fraction) half-plane clipping of P by every edge of Q, then shoelace."""
    poly = [(Fraction(x), Fraction(y)) for x, y in P]
    K = len(Q)
    for j in range(K):
        ax, ay = Q[j]
        bx, by = Q[(j + 1) % K]
        def s(p):
            return (bx - ax) * (p[1] - ay) - (by - ay) * (p[0] - ax)
        out = []
        n = len(poly)
        for k in range(n):
            cur, prv = poly[k], poly[k - 1]
            sc, sp = s(cur), s(prv)
            if sc >= 0:
                if sp < 0:
                    t = sp / (sp - sc)
                    out.append((prv[0] + t * (cur[0] - prv[0]), prv[1] + t * (cur[1] - prv[1])))
                out.append(cur)
            elif sp >= 0:
                t = sp / (sp - sc)
                out.append((prv[0] + t * (cur[0] - prv[0]), prv[1] + t * (cur[1] - prv[1])))
        poly = out
        if not poly:
            return Fraction(0)
    a = Fraction(0)
    for k in range(len(poly)):
        x0, y0 = poly[k]
        x1, y1 = poly[(k + 1) % len(poly)]
        a += x0 * y1 - x1 * y0
    return a / 2


@pytest.mark.parametrize("K", [4, 6, 8])
def test_lattice_exact(K):
    rng = np.random.default_rng(100 + K)
    done = 0
    P_list, Q_list, want = [], [], []
    while done < 150:
        hs = []
        for _ in range(2):
            while True:
                pts = [tuple(int(v) for v in rng.integers(0, 9, 2)) for _ in range(3 * K)]
                h = _hull(pts)
                if len(h) == K:
                    break
            hs.append(h)
        P, Q = hs
        want.append(float(_exact_clip_area(P, Q)))
        P_list.append(np.array(P, float))
        Q_list.append(np.array(Q, float))
        done += 1
    p1, p2 = as_pairs(P_list, Q_list)
    got = oracle.iou_paired_fwd(p1, p2)["area_i"]
    np.testing.assert_allclose(got, want, rtol=0, atol=1e-12)


# ---------------------------------------------------------------------------
# raster IoU
# ---------------------------------------------------------------------------
def _inside(P, X, Y):
    K = len(P)
    m = np.ones_like(X, dtype=bool)
    for k in range(K):
        ax, ay = P[k]
        bx, by = P[(k + 1) % K]
        m &= (bx - ax) * (Y - ay) - (by - ay) * (X - ax) >= 0
    return m


def test_raster_iou():
    b = synth.gen_cfg1_pairs(60, seed=99)
    f = oracle.iou_paired_fwd(b.p1, b.p2)
    x1, y1 = b.p1.xy64()
    x2, y2 = b.p2.xy64()
    res = 1024
    for k in range(b.n):
        P = np.stack([x1[k], y1[k]], 1)
        Q = np.stack([x2[k], y2[k]], 1)
        lo = np.minimum(P.min(0), Q.min(0))
        hi = np.maximum(P.max(0), Q.max(0))
        xs = lo[0] + (np.arange(res) + 0.5) * (hi[0] - lo[0]) / res
        ys = lo[1] + (np.arange(res) + 0.5) * (hi[1] - lo[1]) / res
        X, Y = np.meshgrid(xs, ys)
        a, c = _inside(P, X, Y), _inside(Q, X, Y)
        r = (a & c).sum() / max(1, (a | c).sum())
        assert abs(r - f["iou"][k]) < 3e-3, (k, r, f["iou"][k])


# ---------------------------------------------------------------------------
# flags: faithfulness and agreement with a literal SH clip
# ---------------------------------------------------------------------------
def _line_cross(P, Q, R, S):
    e, f = Q - P, S - R
    t = ((R - P)[0] * f[1] - (R - P)[1] * f[0]) / (e[0] * f[1] - e[1] * f[0])
    return P + t * e


@pytest.mark.parametrize("cfg", [1, 3, 4])
def test_flag_faithfulness(cfg):
    b = margin_batch(cfg, 300)
    x1, y1 = b.p1.xy64()
    x2, y2 = b.p2.xy64()
    K = b.p1.K
    for k in range(b.n):
        P = np.stack([x1[k], y1[k]], 1)
        Q = np.stack([x2[k], y2[k]], 1)
        verts, flags, _ = oracle.intersect_one(P, Q)
        for v, fl in zip(verts, flags):
            t, i, j = decode(fl)
            if t == 1:
                w = P[j]
            elif t == 2:
                w = Q[j]
            else:
                w = _line_cross(P[i], P[(i + 1) % K], Q[j], Q[(j + 1) % K])
            assert np.max(np.abs(w - v)) < 1e-9


@pytest.mark.parametrize("cfg", [1, 3, 4])
def test_sh_secondary_oracle_agrees(cfg):
    b = margin_batch(cfg, 3000)
    f = oracle.iou_paired_fwd(b.p1, b.p2)
    s = oracle.sh_intersect(b.p1, b.p2)
    np.testing.assert_array_equal(f["nx"], s["nx"])
    np.testing.assert_array_equal(f["xflags"], s["xflags"])
    np.testing.assert_allclose(f["area_i"], s["area_i"], rtol=1e-11, atol=1e-12)


def test_sh_degenerate_zoo_matches_definition():
    """identical, subset, shared edge, touching edge/corner, vertex on edge."""
    cases = [
        (SQ, SQ),                                       # identical
        (SQ * 0.5 + 0.25, SQ),                          # strict subset
        (SQ, SQ + [1.0, 0.0]),                          # touching edge -> empty
        (SQ, SQ + [1.0, 1.0]),                          # touching corner -> empty
        (SQ, np.array([[0, 0], [2, 0], [2, 1], [0, 1]], float)),   # shared edges, subset
    ]
    for P, Q in cases:
        iou, nx, fl, ai = fwd1(P, Q)
        p1, p2 = as_pairs([P], [Q])
        s = oracle.sh_intersect(p1, p2)
        assert int(s["nx"][0]) == nx
        assert [int(x) for x in s["xflags"][0][:nx]] == fl
        assert abs(s["area_i"][0] - ai) < 1e-15
    assert fwd1(SQ, SQ + [1.0, 0.0])[0] == 0.0
    assert fwd1(SQ, SQ + [1.0, 1.0])[0] == 0.0


def _p1_key(P, v, b):
    """position along p1's boundary from v0 (reading R3): FromP1(i) -> i,
    Cross(i, j) -> i + t; FromP2 -> None (not on p1's boundary)."""
    t, i, j = decode(b)
    K = len(P)
    if t == 1:
        return float(j)
    if t == 3:
        a, e = P[i], P[(i + 1) % K] - P[i]
        return i + float(np.dot(v - a, e) / np.dot(e, e))
    return None


@pytest.mark.parametrize("cfg", [1, 3, 4])
def test_canonical_start_convention(cfg):
    """R3: xflags start at the vertex met first walking p1's boundary CCW from v0
    (the smallest byte when no vertex lies on p1's boundary), and the sequence is
    CCW (positive signed area of the listed vertices)."""
    b = margin_batch(cfg, 400)
    x1, y1 = b.p1.xy64()
    x2, y2 = b.p2.xy64()
    for k in range(b.n):
        P = np.stack([x1[k], y1[k]], 1)
        Q = np.stack([x2[k], y2[k]], 1)
        verts, flags, _ = oracle.intersect_one(P, Q)
        if not flags:
            continue
        keys = [_p1_key(P, v, f) for v, f in zip(verts, flags)]
        on = [x for x in keys if x is not None]
        if on:
            assert keys[0] == min(on)
        else:
            assert flags[0] == min(flags)
        a = 0.5 * np.sum(verts[:, 0] * np.roll(verts[:, 1], -1) - np.roll(verts[:, 0], -1) * verts[:, 1])
        assert a > 0


CANON = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "canonical_start.json")))


@pytest.mark.parametrize("case", CANON["cases"], ids=lambda c: c["name"])
def test_canonical_start_hand_derived(case):
    """R3 pinned to hand-derived sequences (tests/golden/canonical_start.json): the
    start is the smallest position i + t along p1's boundary, with t measured on
    p1's edge (case 1 would start elsewhere with t taken on p2's edge), not the
    smallest byte (cases 2, 3), wrapping through p1's closing edge (case 3)."""
    P, Q = np.array(case["p1"], float), np.array(case["p2"], float)
    iou, nx, fl, ai = fwd1(P, Q)
    assert nx == case["nx"] and fl == case["xflags"]
    assert abs(ai - case["area_i"][0] / case["area_i"][1]) < 1e-14
    assert abs(iou - case["iou"][0] / case["iou"][1]) < 1e-14


# --- degenerate geometry pinned to closed forms (R5 boundary-inclusive) --------
def test_nested_collinear_boxes_closed_form():
    """Same centre, height and yaw, widths w and w(1 - delta): p2 inside p1 with two
    collinear edge pairs; IoU = A2/A1 = 1 - delta exactly (by definition)."""
    rng = np.random.default_rng(11)
    n = 400
    w = rng.uniform(0.5, 5, n); h = rng.uniform(0.5, 2, n); th = rng.uniform(-4, 4, n)
    cx = rng.uniform(0, 70, n); cy = rng.uniform(-40, 40, n)
    delta = rng.choice([1e-7, 1e-6, 1e-4, 1e-2, 0.3], n)
    b1 = np.stack([cx, cy, w, h, th], 1)
    b2 = np.stack([cx, cy, w * (1 - delta), h, th], 1)
    r = oracle.box_iou_paired(b1, b2)
    assert np.max(np.abs(r["iou"] - (1 - delta))) < 1e-9


def test_integer_grid_rectangles_closed_form():
    """Axis-aligned rectangles on an integer grid (exact shared edges, touching,
    containment): IoU from the interval-overlap closed form."""
    rng = np.random.default_rng(12)
    g = rng.integers(0, 4, size=(3000, 8)).astype(float)
    x0, y0, a, b = g[:, 0], g[:, 1], 1 + g[:, 2], 1 + g[:, 3]
    u0, v0, c, d = g[:, 4], g[:, 5], 1 + g[:, 6], 1 + g[:, 7]
    P = [np.stack([x0, x0 + a, x0 + a, x0], 1), np.stack([y0, y0, y0 + b, y0 + b], 1)]
    Q = [np.stack([u0, u0 + c, u0 + c, u0], 1), np.stack([v0, v0, v0 + d, v0 + d], 1)]
    r = oracle.iou_paired_fwd(tuple(P), tuple(Q))
    ox = np.clip(np.minimum(x0 + a, u0 + c) - np.maximum(x0, u0), 0, None)
    oy = np.clip(np.minimum(y0 + b, v0 + d) - np.maximum(y0, v0), 0, None)
    ai = ox * oy
    want = ai / (a * b + c * d - ai)
    assert np.max(np.abs(r["iou"] - want)) < 1e-12


def test_translation_invariance_far_from_origin():
    """S:397 rigid invariance, at 10 km: small polygons (~5-50 cm) translated by
    (1e4, -1e4) exactly (double inputs) give the same IoU within 1e-9 and the same flags
    and vertex gradients.  (An oracle computing in absolute coordinates fails this by
    ~1e-4: the shoelace products and a dedupe tolerance proportional to |coordinate|.)"""
    b = synth.gen_config(1, 2000)
    sc = 0.01
    p1 = (b.p1.x.reshape(-1, 4).astype(np.float64) * sc, b.p1.y.reshape(-1, 4).astype(np.float64) * sc)
    p2 = (b.p2.x.reshape(-1, 4).astype(np.float64) * sc, b.p2.y.reshape(-1, 4).astype(np.float64) * sc)
    far = lambda p: (p[0] + 1e4, p[1] - 1e4)  # noqa: E731  (exact in double)
    r0 = oracle.iou_paired_fwd(p1, p2)
    r1 = oracle.iou_paired_fwd(far(p1), far(p2))
    assert (r0["iou"] > 0).mean() > 0.8
    assert np.max(np.abs(r0["iou"] - r1["iou"])) < 1e-9
    assert np.array_equal(r0["nx"], r1["nx"]) and np.array_equal(r0["xflags"], r1["xflags"])
    g = np.random.default_rng(3).uniform(-1, 1, b.n)
    g0 = oracle.iou_paired_bwd(p1, p2, g)
    g1 = oracle.iou_paired_bwd(far(p1), far(p2), g)
    for a, c in zip(g0, g1):
        assert np.max(np.abs(a - c)) <= 1e-9 * max(1.0, np.max(np.abs(a)))


def test_zero_area_polygons_give_zero():
    """S:396 (0 <= IoU <= 1 always) and set inclusion (|P1 n P2| <= min(|P1|, |P2|)): a
    polygon of zero area — all vertices at one point inside the other, or on a segment
    along its edge — intersects in nothing: IoU 0, nx 0, both argument orders."""
    P = SQ * 2.0
    pt = np.full((4, 2), 0.7)
    seg = np.array([[0.0, 0.0], [0.0, 0.0], [2.0, 0.0], [2.0, 0.0]])
    for Z in (pt, seg):
        for a, b in ((P, Z), (Z, P)):
            iou, nx, fl, ai = fwd1(a, b)
            assert iou == 0.0 and nx == 0 and ai == 0.0
