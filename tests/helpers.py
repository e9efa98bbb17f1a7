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
