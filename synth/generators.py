"""Seeded generators for the five BASELINE.json configurations.

Every generator draws float64 box / polygon parameters from numpy's PCG64 and
rounds the resulting vertex coordinates ONCE to float32.  That float32
structure-of-arrays buffer is the single source of truth: the CUDA path reads
it as-is and the oracle converts it exactly to float64.

Layout (SoA, matching include/dgal.h): polygon n, vertex k is
(x[n*K + k], y[n*K + k]); vertices counter-clockwise (§III
"stored in counter-clockwise order").

Draws are done in fixed-size chunks (CHUNK pairs, each chunk from its own
SeedSequence child), so the first m pairs of a batch of n >= m pairs are the
same for every n ("prefix stable") — the parity tests at small n sample the
very workload the bench times at full n.

This module holds no arithmetic of the method (no clipping, area or IoU).
"""
from __future__ import annotations

import math
import os
from dataclasses import dataclass

import numpy as np

CHUNK = 1 << 16
BASE_SEED = 1134000

#: BASELINE.json configs (index = cfg number)
CONFIGS = {
    1: dict(kind="paired", K=4, n=1024,
            desc="paired IoU fwd+bwd, 1,024 random rotated rectangles (SPEC generator)"),
    2: dict(kind="pairwise", K=4, n=2000,
            desc="pairwise 2,000x2,000 KITTI-scale BEV boxes, forward"),
    3: dict(kind="paired", K=4, n=1 << 24,
            desc="paired IoU loss fwd+bwd, 16M KITTI-like rotated-box pairs"),
    4: dict(kind="paired", K=8, n=1 << 22,
            desc="paired IoU fwd+bwd, 4M convex octagon pairs (K=8)"),
    5: dict(kind="pairwise", K=4, n=100_000,
            desc="pairwise 100k x 100k nuScenes-like boxes + rotated-NMS keep"),
}


def seed_for(cfg: int, rank: int = 0) -> int:
    """Seed of config `cfg` (1134000 + cfg); rank r of a weak-scaling
    run draws its own shard from seed + 7919*r."""
    return BASE_SEED + cfg + 7919 * rank


@dataclass
class Polys:
    """A batch of n convex CCW polygons with exactly K vertices, SoA float32."""
    x: np.ndarray  # float32 [n*K]
    y: np.ndarray  # float32 [n*K]
    K: int

    @property
    def n(self) -> int:
        return self.x.size // self.K

    def take(self, idx) -> "Polys":
        idx = np.asarray(idx)
        X = self.x.reshape(-1, self.K)[idx].reshape(-1)
        Y = self.y.reshape(-1, self.K)[idx].reshape(-1)
        return Polys(np.ascontiguousarray(X), np.ascontiguousarray(Y), self.K)

    def xy64(self):
        """(n, K) float64 views of the float32 coordinates (exact conversion)."""
        return (self.x.astype(np.float64).reshape(-1, self.K),
                self.y.astype(np.float64).reshape(-1, self.K))


@dataclass
class PairBatch:
    p1: Polys
    p2: Polys
    grad: np.ndarray  # float32 [n], dL/dIoU ~ U(-1, 1)

    @property
    def n(self) -> int:
        return self.p1.n

    def take(self, idx) -> "PairBatch":
        idx = np.asarray(idx)
        return PairBatch(self.p1.take(idx), self.p2.take(idx),
                         np.ascontiguousarray(self.grad[idx]))


@dataclass
class Scene:
    """Detections sorted by descending score (NMS order)."""
    polys: Polys
    scores: np.ndarray  # float32 [n], descending
    thr: float


# ----------------------------------------------------------------------------
# box parameters -> rectangle corners
# ----------------------------------------------------------------------------
_SX = np.array([-0.5, 0.5, 0.5, -0.5])
_SY = np.array([-0.5, -0.5, 0.5, 0.5])


def boxes_to_polys(cx, cy, length, width, theta) -> Polys:
    """Rectangles c + R(theta)(+-l/2, +-w/2), CCW, starting at (-l/2, -w/2)
    (SPEC.md l.347).  float64 in, float32 out (one rounding)."""
    cx, cy, length, width, theta = (np.asarray(a, dtype=np.float64)
                                    for a in (cx, cy, length, width, theta))
    c, s = np.cos(theta)[:, None], np.sin(theta)[:, None]
    lx = length[:, None] * _SX[None, :]
    wy = width[:, None] * _SY[None, :]
    x = cx[:, None] + c * lx - s * wy
    y = cy[:, None] + s * lx + c * wy
    return Polys(np.ascontiguousarray(x.astype(np.float32).reshape(-1)),
                 np.ascontiguousarray(y.astype(np.float32).reshape(-1)), 4)


def _chunked(n, seed, draw_chunk):
    """Call draw_chunk(rng, CHUNK) for ceil(n/CHUNK) chunks (each with its own
    SeedSequence child, drawn in a thread pool — the result does not depend on
    the scheduling), concat, truncate."""
    nch = max(1, -(-n // CHUNK))
    ss = np.random.SeedSequence(seed)
    children = ss.spawn(nch)
    job = lambda c: draw_chunk(np.random.Generator(np.random.PCG64(c)), CHUNK)  # noqa: E731
    if nch >= 8:
        from concurrent.futures import ThreadPoolExecutor
        with ThreadPoolExecutor(max_workers=min(32, os.cpu_count() or 4)) as ex:
            parts = list(ex.map(job, children))
    else:
        parts = [job(c) for c in children]
    return [np.concatenate(fields)[:n] for fields in zip(*parts)]


# ----------------------------------------------------------------------------
# cfg1: SPEC.md generate_pairs
# ----------------------------------------------------------------------------
def _cfg1_chunk(rng, m):
    c1 = rng.uniform(-10, 10, size=(m, 2))
    e1 = rng.uniform(0.5, 5, size=(m, 2))
    t1 = rng.uniform(-math.pi, math.pi, size=m)
    c2 = c1 + rng.uniform(-2, 2, size=(m, 2))
    e2 = rng.uniform(0.5, 5, size=(m, 2))
    t2 = rng.uniform(-math.pi, math.pi, size=m)
    g = rng.uniform(-1, 1, size=m)
    return (c1[:, 0], c1[:, 1], e1[:, 0], e1[:, 1], t1,
            c2[:, 0], c2[:, 1], e2[:, 0], e2[:, 1], t2, g)


def gen_cfg1_pairs(n: int = 1024, seed: int | None = None) -> PairBatch:
    seed = seed_for(1) if seed is None else seed
    a = _chunked(n, seed, _cfg1_chunk)
    return PairBatch(boxes_to_polys(*a[0:5]), boxes_to_polys(*a[5:10]),
                     a[10].astype(np.float32))


# ----------------------------------------------------------------------------
# KITTI-like objects (cfg2, cfg3)
# ----------------------------------------------------------------------------
# (share, length mean, length sd, width mean, width sd)
_KITTI = np.array([
    (0.75, 3.89, 0.43, 1.62, 0.10),   # car
    (0.15, 0.84, 0.23, 0.66, 0.14),   # pedestrian
    (0.10, 1.76, 0.18, 0.60, 0.12),   # cyclist
])


def _kitti_objects(rng, m):
    cls = rng.choice(len(_KITTI), size=m, p=_KITTI[:, 0])
    row = _KITTI[cls]
    length = np.maximum(rng.normal(row[:, 1], row[:, 2]), 0.25 * row[:, 1])
    width = np.maximum(rng.normal(row[:, 3], row[:, 4]), 0.25 * row[:, 3])
    cx = rng.uniform(0.0, 70.4, size=m)
    cy = rng.uniform(-40.0, 40.0, size=m)
    th = rng.uniform(-math.pi, math.pi, size=m)
    return cx, cy, length, width, th


def _jitter(rng, cx, cy, length, width, th, s_c, s_logsize, s_th, flip=0.0):
    diag = np.hypot(length, width)
    m = cx.size
    jx = cx + rng.normal(0, 1, size=m) * s_c * diag
    jy = cy + rng.normal(0, 1, size=m) * s_c * diag
    jl = length * np.exp(rng.normal(0, s_logsize, size=m))
    jw = width * np.exp(rng.normal(0, s_logsize, size=m))
    jt = th + rng.normal(0, 1, size=m) * s_th
    if flip:
        jt = jt + math.pi * (rng.uniform(size=m) < flip)
    return jx, jy, jl, jw, jt


def _cfg3_chunk(rng, m):
    gt = _kitti_objects(rng, m)
    good = _jitter(rng, *gt, 0.1, 0.1, 0.1)
    poor = _jitter(rng, *gt, 0.5, 0.3, math.pi / 2)
    is_poor = rng.uniform(size=m) < 0.10
    pred = tuple(np.where(is_poor, p, g) for g, p in zip(good, poor))
    g = rng.uniform(-1, 1, size=m)
    return (*pred, *gt, g)


def gen_cfg3_pairs(n: int = 1 << 24, seed: int | None = None) -> PairBatch:
    """KITTI paired training batch: p1 = prediction, p2 = ground truth;
    90% matched (centre sd 0.1 diag, log-size sd 0.1, yaw sd 0.1 rad),
    10% poor (0.5 diag, 0.3, pi/2)."""
    seed = seed_for(3) if seed is None else seed
    a = _chunked(n, seed, _cfg3_chunk)
    return PairBatch(boxes_to_polys(*a[0:5]), boxes_to_polys(*a[5:10]),
                     a[10].astype(np.float32))


# ----------------------------------------------------------------------------
# rotated-box parameter batches: the cfg3 distribution
# kept as box parameters instead of corners
# ----------------------------------------------------------------------------
# KITTI vertical extent (mean, sd) per class and the LiDAR-frame centre height
_KITTI_D = np.array([(1.53, 0.14), (1.76, 0.11), (1.74, 0.09)])
_KITTI_CZ = (-1.0, 0.4)


@dataclass
class BoxPairBatch:
    """b1 = prediction, b2 = ground truth, float32 parameter planes [P, n]:
    P = 5 (cx, cy, w, h, theta) or P = 7 (cx, cy, cz, w, h, d, theta)."""
    b1: np.ndarray
    b2: np.ndarray
    grad: np.ndarray  # float32 [n], dL/dIoU ~ U(-1, 1)

    @property
    def n(self) -> int:
        return self.b1.shape[1]

    @property
    def dims(self) -> int:
        return 3 if self.b1.shape[0] == 7 else 2

    def take(self, idx) -> "BoxPairBatch":
        idx = np.asarray(idx)
        return BoxPairBatch(np.ascontiguousarray(self.b1[:, idx]), np.ascontiguousarray(self.b2[:, idx]),
                            np.ascontiguousarray(self.grad[idx]))

    def rows64(self):
        """(n, P) float64 rows of the float32 parameters (exact conversion), oracle layout."""
        return self.b1.T.astype(np.float64), self.b2.T.astype(np.float64)


def _box_chunk(rng, m, dims):
    cls = rng.choice(len(_KITTI), size=m, p=_KITTI[:, 0])
    row = _KITTI[cls]
    length = np.maximum(rng.normal(row[:, 1], row[:, 2]), 0.25 * row[:, 1])
    width = np.maximum(rng.normal(row[:, 3], row[:, 4]), 0.25 * row[:, 3])
    cx = rng.uniform(0.0, 70.4, size=m)
    cy = rng.uniform(-40.0, 40.0, size=m)
    th = rng.uniform(-math.pi, math.pi, size=m)
    gt = (cx, cy, length, width, th)
    good = _jitter(rng, *gt, 0.1, 0.1, 0.1)
    poor = _jitter(rng, *gt, 0.5, 0.3, math.pi / 2)
    is_poor = rng.uniform(size=m) < 0.10
    pred = tuple(np.where(is_poor, p, g) for g, p in zip(good, poor))
    g = rng.uniform(-1, 1, size=m)
    if dims == 2:
        return (*pred, *gt, g)
    rd = _KITTI_D[cls]
    d = np.maximum(rng.normal(rd[:, 0], rd[:, 1]), 0.25 * rd[:, 0])
    cz = rng.normal(_KITTI_CZ[0], _KITTI_CZ[1], size=m)
    s_c = np.where(is_poor, 0.5, 0.1)
    s_d = np.where(is_poor, 0.3, 0.1)
    pz = cz + rng.normal(0, 1, size=m) * s_c * d
    pd = d * np.exp(rng.normal(0, 1, size=m) * s_d)
    pcx, pcy, pl, pw, pt = pred
    return (pcx, pcy, pz, pl, pw, pd, pt, cx, cy, cz, length, width, d, th, g)


def gen_box_pairs(n: int = 1 << 24, dims: int = 2, seed: int | None = None) -> BoxPairBatch:
    """cfg3's KITTI matched/poor prediction-target distribution as box parameters
    (dims=2: RotatedBox2, dims=3: yaw-only Box3 with KITTI heights)."""
    seed = seed_for(3) + 101 * dims if seed is None else seed
    a = _chunked(n, seed, lambda rng, m: _box_chunk(rng, m, dims))
    P = 5 if dims == 2 else 7
    b1 = np.ascontiguousarray(np.stack(a[0:P]).astype(np.float32))
    b2 = np.ascontiguousarray(np.stack(a[P:2 * P]).astype(np.float32))
    return BoxPairBatch(b1, b2, a[2 * P].astype(np.float32))


def _scene_from_objects(rng, objs, per_object, thr):
    cx, cy, length, width, th = (np.repeat(a, per_object) for a in objs)
    props = _jitter(rng, cx, cy, length, width, th, 0.2, 0.15, 0.2, flip=0.10)
    scores = rng.uniform(size=cx.size)
    order = np.argsort(-scores, kind="stable")
    polys = boxes_to_polys(*(p[order] for p in props))
    return Scene(polys, scores[order].astype(np.float32), thr)


def gen_cfg2_scene(n_objects: int = 40, per_object: int = 50, seed: int | None = None,
                   thr: float = 0.7) -> Scene:
    """KITTI-scale scene: 40 objects x 50 proposals, raw (not margin-filtered)."""
    seed = seed_for(2) if seed is None else seed
    rng = np.random.Generator(np.random.PCG64(seed))
    return _scene_from_objects(rng, _kitti_objects(rng, n_objects), per_object, thr)


# ----------------------------------------------------------------------------
# cfg4: convex octagons
# ----------------------------------------------------------------------------
def _ellipse_octagon(rng, m):
    c = rng.uniform(-10, 10, size=(m, 2))
    a = rng.uniform(1, 3, size=m)
    b = a * rng.uniform(0.6, 1.0, size=m)
    phi = rng.uniform(-math.pi, math.pi, size=m)           # ellipse orientation
    phi0 = rng.uniform(0, 2 * math.pi, size=m)             # first vertex angle
    k = np.arange(8)[None, :]
    alpha = (k + rng.uniform(-0.3, 0.3, size=(m, 8))) * (math.pi / 4) + phi0[:, None]
    ex, ey = a[:, None] * np.cos(alpha), b[:, None] * np.sin(alpha)
    cp, sp = np.cos(phi)[:, None], np.sin(phi)[:, None]
    return c[:, :1] + cp * ex - sp * ey, c[:, 1:] + sp * ex + cp * ey


def _cfg4_chunk(rng, m):
    x1, y1 = _ellipse_octagon(rng, m)
    x2, y2 = _ellipse_octagon(rng, m)
    shift = rng.normal(0, 1, size=(m, 2))
    x2 = x2 - x2.mean(1, keepdims=True) + x1.mean(1, keepdims=True) + shift[:, :1]
    y2 = y2 - y2.mean(1, keepdims=True) + y1.mean(1, keepdims=True) + shift[:, 1:]
    # 10%: concentric near-regular pairs rotated pi/8 (+-N(0,0.02)), +-2% radial noise
    reg = rng.uniform(size=m) < 0.10
    c = rng.uniform(-10, 10, size=(m, 2))
    R = rng.uniform(1, 3, size=m)
    phi0 = rng.uniform(0, 2 * math.pi, size=m)
    dphi = math.pi / 8 + rng.normal(0, 0.02, size=m)
    k = np.arange(8)[None, :] * (math.pi / 4)
    r1 = R[:, None] * (1 + rng.uniform(-0.02, 0.02, size=(m, 8)))
    r2 = R[:, None] * (1 + rng.uniform(-0.02, 0.02, size=(m, 8)))
    a1 = k + phi0[:, None]
    a2 = a1 + dphi[:, None]
    rx1, ry1 = c[:, :1] + r1 * np.cos(a1), c[:, 1:] + r1 * np.sin(a1)
    rx2, ry2 = c[:, :1] + r2 * np.cos(a2), c[:, 1:] + r2 * np.sin(a2)
    sel = reg[:, None]
    g = rng.uniform(-1, 1, size=m)
    return (np.where(sel, rx1, x1), np.where(sel, ry1, y1),
            np.where(sel, rx2, x2), np.where(sel, ry2, y2), g)


def gen_cfg4_pairs(n: int = 1 << 22, seed: int | None = None) -> PairBatch:
    seed = seed_for(4) if seed is None else seed
    x1, y1, x2, y2, g = _chunked(n, seed, _cfg4_chunk)
    f = lambda a: np.ascontiguousarray(a.astype(np.float32).reshape(-1))  # noqa: E731
    return PairBatch(Polys(f(x1), f(y1), 8), Polys(f(x2), f(y2), 8), g.astype(np.float32))


# ----------------------------------------------------------------------------
# general convex quadrilaterals (test workload: every K=4 walk-table state)
# ----------------------------------------------------------------------------
def _ellipse_quad(rng, m, c, a, b):
    phi = rng.uniform(-math.pi, math.pi, size=m)
    phi0 = rng.uniform(0, 2 * math.pi, size=m)
    k = np.arange(4)[None, :]
    alpha = (k + rng.uniform(-0.35, 0.35, size=(m, 4))) * (math.pi / 2) + phi0[:, None]
    ex, ey = a[:, None] * np.cos(alpha), b[:, None] * np.sin(alpha)
    cp, sp = np.cos(phi)[:, None], np.sin(phi)[:, None]
    return c[:, :1] + cp * ex - sp * ey, c[:, 1:] + sp * ex + cp * ey


def _quad_chunk(rng, m):
    """Non-rectangular convex quads on ellipses (points in angular order on an ellipse
    are in convex position, CCW).  Mix: 60 % partner shifted by N(0, 1.5^2) with an
    independent shape; 20 % partner inside-ish (scaled 0.2-0.6 about a point near the
    centre: containment both ways, runs of up to 3 FromP2 bytes); 20 % same ellipse,
    partner rotated ~pi/4 (up to 8 crossings)."""
    c = rng.uniform(-10, 10, size=(m, 2))
    a = rng.uniform(1, 3, size=m)
    b = a * rng.uniform(0.3, 1.0, size=m)
    x1, y1 = _ellipse_quad(rng, m, c, a, b)
    kind = rng.uniform(size=m)
    c2 = c + rng.normal(0, 1.5, size=(m, 2))
    a2 = rng.uniform(1, 3, size=m)
    b2 = a2 * rng.uniform(0.3, 1.0, size=m)
    small = (kind >= 0.6) & (kind < 0.8)
    sc = np.where(small, rng.uniform(0.2, 0.6, size=m), 1.0)
    c2 = np.where(small[:, None], c + rng.normal(0, 0.3, size=(m, 2)), c2)
    a2, b2 = np.where(small, a * sc, a2), np.where(small, b * sc, b2)
    rot = kind >= 0.8
    c2 = np.where(rot[:, None], c, c2)
    a2, b2 = np.where(rot, a * rng.uniform(0.9, 1.1, size=m), a2), np.where(rot, b, b2)
    x2, y2 = _ellipse_quad(rng, m, c2, a2, b2)
    swap = rng.uniform(size=m) < 0.5                        # containment both ways
    x1, x2 = np.where(swap[:, None], x2, x1), np.where(swap[:, None], x1, x2)
    y1, y2 = np.where(swap[:, None], y2, y1), np.where(swap[:, None], y1, y2)
    g = rng.uniform(-1, 1, size=m)
    return x1, y1, x2, y2, g


def gen_quad_pairs(n: int = 4096, seed: int | None = None) -> PairBatch:
    """General convex quadrilateral pairs Poly2<float,4> (tests only; seed 1134000 + 41)."""
    seed = BASE_SEED + 41 if seed is None else seed
    x1, y1, x2, y2, g = _chunked(n, seed, _quad_chunk)
    f = lambda a: np.ascontiguousarray(a.astype(np.float32).reshape(-1))  # noqa: E731
    return PairBatch(Polys(f(x1), f(y1), 4), Polys(f(x2), f(y2), 4), g.astype(np.float32))


# ----------------------------------------------------------------------------
# thin / sliver polygons (test workload: "numerical stability ... arbitrary
# shape input"; the float conditioning of the area sum on high-aspect shapes)
# ----------------------------------------------------------------------------
def _thin_poly(rng, m, verts, c, a, b, phi):
    """`verts`-gons inscribed in ellipses (semi-axes a >> b, orientation phi): angles
    (k + U(-0.3, 0.3)) 2 pi / verts + phi0 — in angular order, so convex and CCW."""
    phi0 = rng.uniform(0, 2 * math.pi, size=m)
    k = np.arange(verts)[None, :]
    alpha = (k + rng.uniform(-0.3, 0.3, size=(m, verts))) * (2 * math.pi / verts) + phi0[:, None]
    ex, ey = a[:, None] * np.cos(alpha), b[:, None] * np.sin(alpha)
    cp, sp = np.cos(phi)[:, None], np.sin(phi)[:, None]
    return c[:, :1] + cp * ex - sp * ey, c[:, 1:] + sp * ex + cp * ey


def gen_thin_pairs(n: int, K: int, verts: int, aspect: float, seed: int | None = None,
                   extent: float = 354.0) -> PairBatch:
    """Pairs of thin convex `verts`-gons (verts <= K; padded to K by repeating the last
    vertex, include/dgal.h) of aspect ratio `aspect` (ellipse semi-axes a, a / aspect,
    a ~ U[1, 30] m), centred anywhere in [-extent, extent]^2 (scene coordinates, the
    nuScenes square of cfg5).  The partner's centre lies inside p1's ellipse; half the
    pairs cross at a random angle (sliver intersections far from both polygons'
    vertices), half overlap lengthwise (orientation N(0, 0.05^2)).  Tests only."""
    seed = BASE_SEED + 61 + 1000 * K + 100 * verts + int(aspect) if seed is None else seed
    rng = np.random.Generator(np.random.PCG64(seed))
    c1 = rng.uniform(-extent, extent, size=(n, 2))
    a1 = rng.uniform(1, 30, size=n)
    phi1 = rng.uniform(-math.pi, math.pi, size=n)
    x1, y1 = _thin_poly(rng, n, verts, c1, a1, a1 / aspect, phi1)
    u, v = rng.uniform(-0.8, 0.8, size=n) * a1, rng.uniform(-0.5, 0.5, size=n) * (a1 / aspect)
    c2 = c1 + np.stack([np.cos(phi1) * u - np.sin(phi1) * v, np.sin(phi1) * u + np.cos(phi1) * v], 1)
    a2 = rng.uniform(1, 30, size=n)
    cross_ = rng.uniform(size=n) < 0.5
    phi2 = phi1 + np.where(cross_, rng.uniform(-math.pi, math.pi, size=n), rng.normal(0, 0.05, size=n))
    x2, y2 = _thin_poly(rng, n, verts, c2, a2, a2 / aspect, phi2)
    pad = lambda a: np.concatenate([a, np.repeat(a[:, -1:], K - verts, 1)], 1)  # noqa: E731
    f = lambda a: np.ascontiguousarray(pad(a).astype(np.float32).reshape(-1))  # noqa: E731
    g = rng.uniform(-1, 1, size=n).astype(np.float32)
    return PairBatch(Polys(f(x1), f(y1), K), Polys(f(x2), f(y2), K), g)


# ----------------------------------------------------------------------------
# cfg5: nuScenes-like clustered proposals
# ----------------------------------------------------------------------------
# (share, length, width)
_NUSC = np.array([
    (0.50, 4.63, 1.97),   # car
    (0.10, 6.93, 2.51),   # truck
    (0.03, 10.5, 2.94),   # bus
    (0.02, 12.29, 2.90),  # trailer
    (0.02, 6.37, 2.85),   # construction vehicle
    (0.15, 0.73, 0.67),   # pedestrian
    (0.04, 2.11, 0.77),   # motorcycle
    (0.04, 1.70, 0.60),   # bicycle
    (0.05, 0.41, 0.41),   # traffic cone
    (0.05, 2.53, 0.50),   # barrier
])


def gen_cfg5_scene(n_objects: int = 2000, per_object: int = 50, seed: int | None = None,
                   density: float = 0.004, thr: float = 0.7) -> Scene:
    """nuScenes-density scene (0.004 objects/m^2 -> a 707 m square at 2000 objects)."""
    seed = seed_for(5) if seed is None else seed
    rng = np.random.Generator(np.random.PCG64(seed))
    side = math.sqrt(n_objects / density)
    p = _NUSC[:, 0] / _NUSC[:, 0].sum()
    cls = rng.choice(len(_NUSC), size=n_objects, p=p)
    length = _NUSC[cls, 1] * np.exp(rng.normal(0, 0.1, size=n_objects))
    width = _NUSC[cls, 2] * np.exp(rng.normal(0, 0.1, size=n_objects))
    cx = rng.uniform(-side / 2, side / 2, size=n_objects)
    cy = rng.uniform(-side / 2, side / 2, size=n_objects)
    th = rng.uniform(-math.pi, math.pi, size=n_objects)
    return _scene_from_objects(rng, (cx, cy, length, width, th), per_object, thr)


def gen_config(cfg: int, n: int | None = None, seed: int | None = None):
    """Config `cfg` at its BASELINE size (or `n` pairs / boxes)."""
    if cfg == 1:
        return gen_cfg1_pairs(n or 1024, seed)
    if cfg == 3:
        return gen_cfg3_pairs(n or (1 << 24), seed)
    if cfg == 4:
        return gen_cfg4_pairs(n or (1 << 22), seed)
    if cfg == 2:
        n = n or 2000
        return gen_cfg2_scene(max(1, n // 50), 50, seed)
    if cfg == 5:
        n = n or 100_000
        return gen_cfg5_scene(max(1, n // 50), 50, seed)
    raise ValueError(f"unknown config {cfg}")
