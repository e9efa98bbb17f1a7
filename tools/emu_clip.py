"""Debugging aid (not a test oracle): a scalar float32 emulation of the device
clip in dgal_core.cuh (clip_intervals + the flags walk of iou_fwd), to study
near-degenerate pairs on the CPU.  Operation order follows the kernel; FMA is
emulated as one float64 op rounded to float32 and rcp.approx as 1/x, so results
match the device closely but not bit for bit."""
from __future__ import annotations

import struct

import numpy as np

f32 = np.float32
TINY = f32(1e-30)
BIG = f32(1e30)


def fma(a, b, c):
    return f32(np.float64(a) * np.float64(b) + np.float64(c))


def enc(v, j):
    u = struct.unpack("<I", struct.pack("<f", float(v)))[0]
    return f32(struct.unpack("<f", struct.pack("<I", (u & ~7) | j))[0])


def strip(v):
    u = struct.unpack("<I", struct.pack("<f", float(v)))[0]
    return f32(struct.unpack("<f", struct.pack("<I", u & ~7))[0])


def dec(v):
    return struct.unpack("<I", struct.pack("<f", float(v)))[0] & 7


def sat(x):
    return f32(min(max(float(x), 0.0), 1.0)) if not np.isnan(x) else f32(0)


def cross(ax, ay, bx, by):
    return f32(f32(ax * by) - f32(ay * bx))


def clip(P, Q, verbose=False):
    """P, Q: (K, 2) float32 (already recentred).  Returns a dict of the clip state."""
    K = len(P)
    P = np.asarray(P, f32); Q = np.asarray(Q, f32)
    g = np.array([P[(i + 1) % K] - P[i] for i in range(K)], f32)
    fv = np.array([Q[(i + 1) % K] - Q[i] for i in range(K)], f32)
    C1 = [f32(f32(P[i, 0] * P[(i + 1) % K, 1]) - f32(P[(i + 1) % K, 0] * P[i, 1])) for i in range(K)]
    C2 = [f32(f32(Q[i, 0] * Q[(i + 1) % K, 1]) - f32(Q[(i + 1) % K, 0] * Q[i, 1])) for i in range(K)]
    A1 = f32(0); A2 = f32(0)
    for i in range(K):
        A1 = f32(A1 + C1[i]); A2 = f32(A2 + C2[i])
    d = np.zeros((K, K), f32); e = np.zeros((K, K), f32)
    for i in range(K):
        for j in range(K):
            Dx = f32(P[i, 0] - Q[j, 0]); Dy = f32(P[i, 1] - Q[j, 1])
            d[i, j] = f32(cross(fv[j, 0], fv[j, 1], Dx, Dy) + TINY)
            e[j, i] = f32(cross(Dx, Dy, g[i, 0], g[i, 1]) - TINY)
    separated = False
    for j in range(K):
        separated |= (d[:, j].max() < TINY)
    cxm = f32(sum(Q[:, 0]) * f32(1.0 / K)); cym = f32(sum(Q[:, 1]) * f32(1.0 / K))
    cin = all(cross(g[i, 0], g[i, 1], f32(cxm - P[i, 0]), f32(cym - P[i, 1])) > 0 for i in range(K))
    emin = e.min()
    HI0 = f32(struct.unpack("<f", struct.pack("<I", 0x3F800008))[0])
    inside = [bool(np.all(d[i, :] > 0)) for i in range(K)]
    t0 = np.zeros(K, f32); t1 = np.zeros(K, f32)
    for i in range(K):
        i1 = (i + 1) % K
        lo, hi = f32(0), HI0
        for j in range(K):
            a, b = d[i, j], d[i1, j]
            den = f32(f32(a - b) + TINY)
            r = f32(1.0 / den)
            m = sat(f32(-den * BIG))
            ve = enc(f32(a * r), j)
            lo = max(lo, f32(m * ve))
            hi = min(hi, fma(m, BIG, ve))
        t0[i], t1[i] = lo, hi
    ax = Q[:, 0].copy(); ay = Q[:, 1].copy()
    bx = np.roll(Q[:, 0], -1).copy(); by = np.roll(Q[:, 1], -1).copy()
    ev_out = ev_in = 0
    evs = []
    T0 = np.zeros(K, f32); T1 = np.zeros(K, f32); VAL = [False] * K; HIN = [False] * K; HOUT = [False] * K
    for i in range(K):
        i1 = (i + 1) % K
        a0 = f32(0) if inside[i] else (min(t0[i], f32(1)) if inside[i1] else t0[i])
        a1 = f32(1) if inside[i1] else (max(min(t1[i], f32(1)), f32(0)) if inside[i] else min(t1[i], f32(1)))
        valid = inside[i] or inside[i1] or (strip(a0) < strip(a1))
        has_in = valid and not inside[i]
        has_out = valid and not inside[i1]
        T0[i], T1[i], VAL[i], HIN[i], HOUT[i] = a0, a1, valid, has_in, has_out
        ji = dec(t0[i]) if has_in else 8
        jo = dec(t1[i]) if has_out else 8
        if has_in: ev_in |= 1 << ji
        if has_out: ev_out |= 1 << jo
        xin = (fma(a0, g[i, 0], P[i, 0]), fma(a0, g[i, 1], P[i, 1]))
        xout = (fma(a1, g[i, 0], P[i, 0]), fma(a1, g[i, 1], P[i, 1]))
        for j in range(K):
            if jo == j: ax[j], ay[j] = xout
            if ji == j: bx[j], by[j] = xin
        evs.append((i, bool(valid), bool(has_in), ji, bool(has_out), jo, float(a0), float(a1)))
    KM = (1 << K) - 1
    ev = ev_out | ev_in
    if ev == 0:
        anyvalid = any(VAL)
        in2 = KM if (not anyvalid and cin) else 0
    else:
        evd = ev | (ev << K)
        endin = ev_out & ~ev_in
        st = endin | (endin << K)
        sh = 1
        while sh < 2 * K:
            st = (st & evd) | ((st << sh) & ~evd)
            evd |= evd << sh
            sh <<= 1
        in2 = (st >> (K - 1)) & KM
    on2 = ev | in2
    p2e = f32(0)
    for i in range(K):
        if HOUT[i]:
            jo = dec(t1[i]); X = (fma(T1[i], g[i, 0], P[i, 0]), fma(T1[i], g[i, 1], P[i, 1]))
            p2e = f32(p2e + cross(X[0], X[1], Q[jo, 0], Q[jo, 1]))
        if HIN[i]:
            ji = dec(t0[i]); X = (fma(T0[i], g[i, 0], P[i, 0]), fma(T0[i], g[i, 1], P[i, 1]))
            w = Q[(ji + 1) % K]
            p2e = f32(p2e + cross(w[0], w[1], X[0], X[1]))
    Ai = f32(0)
    for k in range(K):
        Ai = fma(max(f32(T1[k] - T0[k]), f32(0)) if VAL[k] else f32(0), C1[k], Ai)
        Ai = f32(Ai + (C2[k] if (on2 >> k) & 1 else f32(0)))
    Ai = f32(Ai + p2e)
    Ai = min(Ai, min(A1, A2))
    # flags walk
    seq = []
    for i in range(K):
        if not VAL[i]: continue
        seq.append(0xC0 | (i << 3) | dec(t0[i]) if HIN[i] else 0x40 | i)
        if HOUT[i]:
            jo = dec(t1[i])
            seq.append(0xC0 | (i << 3) | jo)
            p0 = (jo + 1) % K
            L = 0
            while L < K and (in2 >> ((p0 + L) % K)) & 1: L += 1
            seq += [0x80 | ((p0 + q) % K) for q in range(L)]
    if not seq and in2 == KM:
        seq = [0x80 | j for j in range(K)]
    nonempty = (not separated) and Ai > 0 and 3 <= len(seq) <= 2 * K
    Au = f32(f32(A1 + A2) - Ai)
    iou = float(min(f32(Ai / Au), f32(1))) if nonempty and Au > 0 else 0.0
    out = dict(iou=iou, nx=len(seq) if nonempty else 0, seq=[hex(b) for b in seq], Ai=float(Ai), A1=float(A1),
               A2=float(A2), separated=bool(separated), in2=in2, ev_out=ev_out, ev_in=ev_in, events=evs,
               t0=t0, t1=t1, d=d, e=e)
    if verbose:
        for k, v in out.items():
            if k not in ("d", "e"):
                print(f"  {k}: {v}")
    return out
