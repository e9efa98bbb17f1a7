"""Shared test helpers: hand-built polygons (float64), the margin filter (calls the
oracle only — tests may), flag-byte decoding.  No product code here."""
from __future__ import annotations

import math

import numpy as np

import oracle
import synth


def box(cx, cy, l, w, th):
    """Rectangle corners in float64 (same corner convention as synth)."""
    c, s = math.cos(th), math.sin(th)
    pts = []
    for sx, sy in ((-0.5, -0.5), (0.5, -0.5), (0.5, 0.5), (-0.5, 0.5)):
        lx, wy = sx * l, sy * w
        pts.append((cx + c * lx - s * wy, cy + s * lx + c * wy))
    return np.array(pts, dtype=np.float64)


def regular(n, circumradius, phase=0.0, centre=(0.0, 0.0)):
    a = phase + 2 * math.pi * np.arange(n) / n
    return np.stack([centre[0] + circumradius * np.cos(a), centre[1] + circumradius * np.sin(a)], 1)


def as_pairs(P_list, Q_list):
    """Lists of (K,2) arrays -> ((x1,y1),(x2,y2)) planes of shape (n,K)."""
    P = np.stack(P_list)
    Q = np.stack(Q_list)
    return (P[..., 0], P[..., 1]), (Q[..., 0], Q[..., 1])


def fwd1(Pv, Qv):
    p1, p2 = as_pairs([Pv], [Qv])
    r = oracle.iou_paired_fwd(p1, p2)
    return r["iou"][0], int(r["nx"][0]), [int(b) for b in r["xflags"][0][: r["nx"][0]]], r["area_i"][0]


def bwd1(Pv, Qv, g=1.0):
    p1, p2 = as_pairs([Pv], [Qv])
    gx1, gy1, gx2, gy2 = oracle.iou_paired_bwd(p1, p2, np.array([g]))
    return np.stack([gx1[0], gy1[0]], 1), np.stack([gx2[0], gy2[0]], 1)


def decode(b):
    """flag byte -> (tag, i, j): tag 1 FromP1(j), 2 FromP2(j), 3 Cross(i,j), 0 CrossP2P2 (R2)."""
    return b >> 6, (b >> 3) & 7, b & 7


def margin_filter(batch: "synth.PairBatch", n: int) -> "synth.PairBatch":
    """First n pairs of `batch` that are a stated margin away from degeneracy
    (R13: decision distance >= 1e-3 sqrt(min area), crossing |sin| >= 1e-2)."""
    ok = oracle.margin_ok(batch.p1, batch.p2)
    idx = np.nonzero(ok)[0]
    assert idx.size >= n, f"margin filter kept {idx.size} < {n}"
    return batch.take(idx[:n])


def margin_batch(cfg: int, n: int, oversample: float = 1.25):
    """cfg (1, 3 or 4) pairs, margin-filtered, prefix-stable."""
    raw = synth.gen_config(cfg, int(n * oversample) + 64)
    return margin_filter(raw, n)


def footprint(rows):
    """(n, 5|7) box rows -> (n, 5) BEV rows (cx, cy, w, h, theta)."""
    rows = np.asarray(rows, np.float64)
    return rows if rows.shape[1] == 5 else rows[:, [0, 1, 3, 4, 6]]


def box_margin_ok(rows1, rows2, zmargin=1e-3):
    """R13 margin filter on the BEV corners (oracle, double) and, for 3D boxes, a
    gap of the z extents away from ties (so min/max subgradients are unambiguous)."""
    x1, y1 = oracle.box_corners(footprint(rows1))
    x2, y2 = oracle.box_corners(footprint(rows2))
    ok = oracle.margin_ok((x1, y1), (x2, y2))
    if np.asarray(rows1).shape[1] == 7:
        r1, r2 = np.asarray(rows1, np.float64), np.asarray(rows2, np.float64)
        t1, t2 = r1[:, 2] + r1[:, 5] / 2, r2[:, 2] + r2[:, 5] / 2
        b1, b2 = r1[:, 2] - r1[:, 5] / 2, r2[:, 2] - r2[:, 5] / 2
        s = np.maximum(r1[:, 5], r2[:, 5])
        ok &= (np.abs(t1 - t2) > zmargin * s) & (np.abs(b1 - b2) > zmargin * s)
        ok &= np.abs(np.minimum(t1, t2) - np.maximum(b1, b2)) > zmargin * s
    return ok


def box_margin_batch(dims, n, seed=None):
    """First n margin-passing pairs of the box generator (raw draw is 2n)."""
    raw = synth.gen_box_pairs(2 * n, dims, seed=seed)
    r1, r2 = raw.rows64()
    idx = np.nonzero(box_margin_ok(r1, r2))[0][:n]
    return raw.take(idx)
