"""CPU oracle (double precision) for batched convex-polygon IoU — TEST INFRASTRUCTURE.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
reference legs may import this package.  The product path never does, and the
oracle imports nothing from the product package (they share no code).

ctypes binding of oracle/liboracle.so (built from oracle/oracle.c by
`__graft_entry__.build()` or `make oracle`).  Every function takes the float32
SoA buffers of synth/ (converted exactly to float64) or float64 arrays.
See oracle/oracle.c for the definition-level algorithm and its citations.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "liboracle.so")
_SRC = os.path.join(_HERE, "oracle.c")

CFLAGS = ["-O2", "-ffp-contract=off", "-fno-fast-math", "-fopenmp", "-shared", "-fPIC",
          "-std=c11", "-Wall", "-Wextra"]


def build(force: bool = False) -> str:
    """Compile liboracle.so in-tree (gcc, plain C11, double, no FMA contraction)."""
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", *CFLAGS, "-o", _SO, _SRC, "-lm"])
    return _SO


_lib = None
_P = ctypes.c_void_p
_I64 = ctypes.c_int64


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_SO)
        L.oracle_iou_paired_fwd.argtypes = [ctypes.c_int, _I64, _P, _P, _P, _P, _P, _P, _P, _P, _P,
                                            ctypes.c_int]
        L.oracle_iou_paired_bwd.argtypes = [ctypes.c_int, _I64, _P, _P, _P, _P, _P, _P, _P, _P, _P,
                                            ctypes.c_int]
        L.oracle_intersect_one.argtypes = [ctypes.c_int, _P, _P, _P, _P, _P, _P, _P, _P, _P]
        L.oracle_area.argtypes = [ctypes.c_int, _I64, _P, _P, _P]
        L.oracle_iou_pairwise.argtypes = [ctypes.c_int, _I64, _P, _P, _I64, _P, _P, _P, ctypes.c_int]
        L.oracle_iou_pairs_indexed.argtypes = [ctypes.c_int, _I64, _P, _P, _P, _P, _P, _P, _P,
                                               ctypes.c_int]
        L.oracle_nms_greedy.argtypes = [_I64, _P, ctypes.c_double, _P]
        L.oracle_nms_scan_mask.argtypes = [_I64, _I64, _P, _P]
        L.oracle_sh_intersect.argtypes = [ctypes.c_int, _I64, _P, _P, _P, _P, _P, _P, _P]
        L.oracle_margin.argtypes = [ctypes.c_int, _I64, _P, _P, _P, _P, _P, _P, ctypes.c_int]
        L.oracle_box_iou_paired.argtypes = [ctypes.c_int, _I64, _P, _P, _P, _P, _P, _P, _P, _P, ctypes.c_int]
        L.oracle_box_corners.argtypes = [_I64, _P, _P, _P]
        L.oracle_box_corners_vjp.argtypes = [_I64, _P, _P, _P, _P]
        L.oracle_max_threads.restype = ctypes.c_int
        _lib = L
    return _lib


def max_threads() -> int:
    return lib().oracle_max_threads()


def _d(a):
    return np.ascontiguousarray(np.asarray(a, dtype=np.float64))


def _ptr(a):
    return a.ctypes.data_as(ctypes.c_void_p) if a is not None else None


def _soa(p):
    """Accept a synth.Polys, or an (x, y) tuple of arrays -> float64 flat planes + K."""
    if hasattr(p, "K"):
        return _d(p.x).reshape(-1), _d(p.y).reshape(-1), p.K
    x, y = p
    x, y = _d(x), _d(y)
    return x.reshape(-1), y.reshape(-1), x.shape[-1] if x.ndim == 2 else None


def _pair_planes(p1, p2, K=None):
    x1, y1, K1 = _soa(p1)
    x2, y2, K2 = _soa(p2)
    K = K or K1 or K2
    assert K is not None and x1.size == x2.size and x1.size % K == 0
    return K, x1.size // K, x1, y1, x2, y2


def iou_paired_fwd(p1, p2, K=None, nthreads=0):
    """-> dict(iou f64[n], nx u8[n], xflags u8[n, 2K], area_i f64[n], status u8[n])"""
    K, n, x1, y1, x2, y2 = _pair_planes(p1, p2, K)
    iou = np.empty(n, np.float64)
    nx = np.empty(n, np.uint8)
    xf = np.empty((n, 2 * K), np.uint8)
    ai = np.empty(n, np.float64)
    st = np.empty(n, np.uint8)
    rc = lib().oracle_iou_paired_fwd(K, n, _ptr(x1), _ptr(y1), _ptr(x2), _ptr(y2), _ptr(iou),
                                     _ptr(nx), _ptr(xf), _ptr(ai), _ptr(st), nthreads)
    assert rc == 0
    return dict(iou=iou, nx=nx, xflags=xf, area_i=ai, status=st)


def iou_paired_bwd(p1, p2, grad, K=None, nthreads=0):
    """-> (gx1, gy1, gx2, gy2) each f64[n, K]"""
    K, n, x1, y1, x2, y2 = _pair_planes(p1, p2, K)
    g = _d(grad).reshape(-1)
    assert g.size == n
    outs = [np.empty(n * K, np.float64) for _ in range(4)]
    rc = lib().oracle_iou_paired_bwd(K, n, _ptr(x1), _ptr(y1), _ptr(x2), _ptr(y2), _ptr(g),
                                     *[_ptr(o) for o in outs], nthreads)
    assert rc == 0
    return tuple(o.reshape(n, K) for o in outs)


def intersect_one(P, Q):
    """P, Q: (K, 2) arrays.  -> (verts (nv,2), flags list[int], (A1, A2, Ai))"""
    P, Q = _d(P), _d(Q)
    K = P.shape[0]
    vx = np.zeros(4 * K + K * K, np.float64)
    vy = np.zeros_like(vx)
    fl = np.zeros(vx.size, np.uint8)
    nv = ctypes.c_int(0)
    areas = np.zeros(3, np.float64)
    px, py, qx, qy = (np.ascontiguousarray(a) for a in (P[:, 0], P[:, 1], Q[:, 0], Q[:, 1]))
    rc = lib().oracle_intersect_one(K, _ptr(px), _ptr(py), _ptr(qx), _ptr(qy), _ptr(vx), _ptr(vy),
                                    _ptr(fl), ctypes.cast(ctypes.pointer(nv), ctypes.c_void_p),
                                    _ptr(areas))
    assert rc == 0
    n = nv.value
    return np.stack([vx[:n], vy[:n]], 1), [int(b) for b in fl[:n]], tuple(areas)


def area(x, y):
    """x, y: (n, K) -> f64[n] shoelace areas."""
    x, y = _d(x), _d(y)
    if x.ndim == 1:
        x, y = x[None], y[None]
    n, K = x.shape
    out = np.empty(n, np.float64)
    assert lib().oracle_area(K, n, _ptr(x), _ptr(y), _ptr(out)) == 0
    return out


def iou_pairwise(rows, cols, K=None, nthreads=0):
    rx, ry, K1 = _soa(rows)
    cx, cy, K2 = _soa(cols)
    K = K or K1 or K2
    nr, m = rx.size // K, cx.size // K
    out = np.empty((nr, m), np.float64)
    assert lib().oracle_iou_pairwise(K, nr, _ptr(rx), _ptr(ry), m, _ptr(cx), _ptr(cy), _ptr(out),
                                     nthreads) == 0
    return out


def iou_pairs_indexed(rows, cols, ri, ci, K=None, nthreads=0):
    rx, ry, K1 = _soa(rows)
    cx, cy, K2 = _soa(cols)
    K = K or K1 or K2
    ri = np.ascontiguousarray(ri, dtype=np.int64)
    ci = np.ascontiguousarray(ci, dtype=np.int64)
    out = np.empty(ri.size, np.float64)
    assert lib().oracle_iou_pairs_indexed(K, ri.size, _ptr(ri), _ptr(ci), _ptr(rx), _ptr(ry),
                                          _ptr(cx), _ptr(cy), _ptr(out), nthreads) == 0
    return out


def nms_greedy(iou_matrix, thr):
    m = _d(iou_matrix)
    n = m.shape[0]
    keep = np.empty(n, np.uint8)
    assert lib().oracle_nms_greedy(n, _ptr(m), float(thr), _ptr(keep)) == 0
    return keep


def nms_scan_mask(mask):
    """mask: uint64 [n, words]; bit j of row i (j > i) = box i suppresses box j."""
    mask = np.ascontiguousarray(mask, dtype=np.uint64)
    n, words = mask.shape
    keep = np.empty(n, np.uint8)
    assert lib().oracle_nms_scan_mask(n, words, _ptr(mask), _ptr(keep)) == 0
    return keep


def sh_intersect(p1, p2, K=None):
    """Secondary oracle (tests only): literal Sutherland-Hodgman with flags."""
    K, n, x1, y1, x2, y2 = _pair_planes(p1, p2, K)
    nx = np.empty(n, np.uint8)
    xf = np.empty((n, 2 * K), np.uint8)
    ai = np.empty(n, np.float64)
    assert lib().oracle_sh_intersect(K, n, _ptr(x1), _ptr(y1), _ptr(x2), _ptr(y2), _ptr(nx),
                                     _ptr(xf), _ptr(ai)) == 0
    return dict(nx=nx, xflags=xf, area_i=ai)


def margin(p1, p2, K=None, nthreads=0):
    """-> (dist_rel f64[n], sin_min f64[n]) (R13)."""
    K, n, x1, y1, x2, y2 = _pair_planes(p1, p2, K)
    d = np.empty(n, np.float64)
    s = np.empty(n, np.float64)
    assert lib().oracle_margin(K, n, _ptr(x1), _ptr(y1), _ptr(x2), _ptr(y2), _ptr(d), _ptr(s),
                               nthreads) == 0
    return d, s


#: R13 acceptance thresholds
MARGIN_DIST = 1e-3
MARGIN_SIN = 1e-2


def margin_ok(p1, p2, K=None, nthreads=0):
    d, s = margin(p1, p2, K, nthreads)
    return (d >= MARGIN_DIST) & (s >= MARGIN_SIN)


# ---------------------------------------------------------------------------
# rotated boxes: rows (cx, cy, w, h, theta) or (cx, cy, cz, w, h, d, theta)
# ---------------------------------------------------------------------------
def box_iou_paired(b1, b2, grad=None, nthreads=0):
    """-> dict(iou, nx, xflags[n, 8], gb1, gb2 (if grad))"""
    b1, b2 = _d(b1), _d(b2)
    n, npar = b1.shape
    dims = 3 if npar == 7 else 2
    iou = np.empty(n, np.float64)
    nx = np.empty(n, np.uint8)
    xf = np.empty((n, 8), np.uint8)
    g = None if grad is None else _d(grad).reshape(-1)
    gb1 = np.empty_like(b1) if g is not None else None
    gb2 = np.empty_like(b2) if g is not None else None
    assert lib().oracle_box_iou_paired(dims, n, _ptr(b1), _ptr(b2), _ptr(iou), _ptr(nx), _ptr(xf), _ptr(g),
                                       _ptr(gb1), _ptr(gb2), nthreads) == 0
    out = dict(iou=iou, nx=nx, xflags=xf)
    if g is not None:
        out.update(gb1=gb1, gb2=gb2)
    return out


def box_corners(b):
    """(n, 5) 2D box params -> (x, y) each (n, 4) float64."""
    b = _d(b)
    n = b.shape[0]
    x = np.empty(n * 4, np.float64)
    y = np.empty(n * 4, np.float64)
    assert lib().oracle_box_corners(n, _ptr(b), _ptr(x), _ptr(y)) == 0
    return x.reshape(n, 4), y.reshape(n, 4)


def box_corners_vjp(b, gx, gy):
    """box_to_polygon_grad: (n, 5) params, (n, 4) corner cotangents -> (n, 5)."""
    b, gx, gy = _d(b), _d(gx), _d(gy)
    n = b.shape[0]
    out = np.empty((n, 5), np.float64)
    assert lib().oracle_box_corners_vjp(n, _ptr(b), _ptr(gx), _ptr(gy), _ptr(out)) == 0
    return out
