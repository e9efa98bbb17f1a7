// dgal_exact.cuh — double-precision area of the RECORDED intersection, for the pairs
// whose float area sum is ill-conditioned (thin / sliver shapes).
// "Conditioning".
//
// The float forward sums Green's terms about p1.v0 (dgal_core.cuh clip_intervals):
// every term is a cross product of coordinates of size up to R (the extent of the
// pair from p1.v0), so its rounding error is ~eps R^2 — harmless for boxes and
// octagons (R^2 / A_u of a few), but for an intersection of thin shapes (aspect
// 100-300: R^2 / A_u ~ the aspect) it reaches 1e-5 of IoU.  The crossing points of
// nearly parallel long edges add an error of the same order (their float parameters
// are conditioned by 1/sin; the area they enclose by L^2 sin).  Both are removed by
// redoing the area in double from the flag record:
//
//   area of intersect(p1, p2, xflags): the nx vertices the flag bytes
//   name (R2) — FromP1(i) -> v_i, FromP2(j) -> w_j, Cross(i, j) -> the intersection
//   of the lines through p1 edge i and p2 edge j — in the recorded CCW order,
//   summed by the shoelace formula about the first of them.
//
// Float inputs are exact in double, their differences are exact (exponents within
// 29 bits) and products of two differences are exact (48-bit mantissas), so the
// only roundings are the crossing division and the sums: ~1e-16 relative.
//
// Used only when a pair is flagged (pair_is_thin below): the split forward and the
// backward recompute in-kernel (rare, divergent), the fused kernels hand the pair to
// their refine pass.
//
// Included by dgal_core.cuh (before the backward section, which uses it); relies on
// the Poly / Seq / paired-FP32 helpers defined above that point.
#pragma once

namespace dgal {

// Vertex access for the exact rebuild: raw float polygon vertices (not recentred),
// vertex k of p1 at px[k], of p2 at qx[k] (unit stride: the per-thread rings and
// the [pair][k] backward tiles).
struct RawPolyVerts {
    const float *px, *py, *qx, *qy;
    __device__ __forceinline__ void p(int k, double &x, double &y) const { x = px[k]; y = py[k]; }
    __device__ __forceinline__ void q(int k, double &x, double &y) const { x = qx[k]; y = qy[k]; }
};

// the same with a stride between vertices (per-thread [k][thread] shared-memory tables)
struct StridedVerts {
    const float *px, *py, *qx, *qy;
    int st;
    __device__ __forceinline__ void p(int k, double &x, double &y) const { x = px[k * st]; y = py[k * st]; }
    __device__ __forceinline__ void q(int k, double &x, double &y) const { x = qx[k * st]; y = qy[k * st]; }
};

struct AreasX2 {
    double a1, a2, ai;   // twice the areas of p1, p2 and of the recorded intersection
};

// s / m: the flag bytes and nx of the pair (bytes beyond m ignored).  All
// coordinates are taken relative to p1.v0 (the polygon areas) and the intersection's
// first vertex (its shoelace), in double.  POLYS = false skips A_1, A_2 (the
// backward: its float A_1, A_2 are accurate to ~eps R^2 / A, enough for the
// S:303 coefficients; only the area of a sliver intersection is not).
template <int K, bool POLYS = true, class VERTS>
__device__ __forceinline__ AreasX2 areas_exact(const VERTS &V, const Seq<K> s, int m)
{
    constexpr int KM = K - 1;
    double ox, oy;
    V.p(0, ox, oy);
    AreasX2 r{0.0, 0.0, 0.0};
#pragma unroll 1
    for (int k = 0; k < (POLYS ? K : 0); ++k) {
        double ax, ay, bx, by, cx, cy, dx, dy;
        V.p(k, ax, ay);
        V.p((k + 1) & KM, bx, by);
        V.q(k, cx, cy);
        V.q((k + 1) & KM, dx, dy);
        ax -= ox; ay -= oy; bx -= ox; by -= oy; cx -= ox; cy -= oy; dx -= ox; dy -= oy;
        r.a1 += ax * by - ay * bx;
        r.a2 += cx * dy - cy * dx;
    }
    double fx = 0.0, fy = 0.0, lx = 0.0, ly = 0.0, acc = 0.0;
#pragma unroll 1
    for (int p = 0; p < m && p < 2 * K; ++p) {
        const uint64_t w = (K == 8 && p >= 8) ? s.w[Seq<K>::NW - 1] : s.w[0];
        const uint32_t b = (uint32_t)(w >> (8 * (p & 7))) & 0xFFu;
        const int tag = (int)(b >> 6), i = (int)((b >> 3) & KM), j = (int)(b & KM);
        double x, y;
        if (tag == 1) {
            V.p(j, x, y);
        } else if (tag == 2) {
            V.q(j, x, y);
        } else {   // Cross(i, j) (tag 3; tag 0, CrossP2P2, is never emitted: R8)
            double vx, vy, v1x, v1y, wx, wy, w1x, w1y;
            V.p(i, vx, vy);
            V.p((i + 1) & KM, v1x, v1y);
            V.q(j, wx, wy);
            V.q((j + 1) & KM, w1x, w1y);
            const double gx = v1x - vx, gy = v1y - vy, hx = w1x - wx, hy = w1y - wy;
            const double den = gx * hy - gy * hx;
            double t = (den != 0.0) ? ((wx - vx) * hy - (wy - vy) * hx) / den : 0.5;
            // the float clip recorded a crossing on the edge: keep it there (off the
            // edge only when the lines nearly coincide, where any point of the edge is
            // within their distance of the true boundary)
            t = fmin(fmax(t, 0.0), 1.0);
            x = fma(t, gx, vx);
            y = fma(t, gy, vy);
        }
        x -= ox;
        y -= oy;
        if (p == 0) {
            fx = x; fy = y;
        } else {
            acc += (lx - fx) * (y - fy) - (ly - fy) * (x - fx);
        }
        lx = x;
        ly = y;
    }
    r.ai = acc;
    return r;
}

// IoU from the exact areas, for the polygon path (2D)
__device__ __forceinline__ float iou_from_areas(const AreasX2 &a)
{
    if (!(a.ai > 0.0)) return 0.f;
    const double u = (a.a1 + a.a2) - a.ai;
    return (u > 0.0) ? (float)fmin(a.ai / u, 1.0) : 0.f;
}

// The forward's outputs of a thin pair from its record (iou_fwd THIN: seq / nx hold
// the walk whatever the float area's sign): areas in double, IoU, and the record
// cleared when the exact intersection is empty.
template <int K, class VERTS>
__device__ __forceinline__ void fwd_thin_fix(const VERTS &V, Seq<K> &s, int &m, float &iou, AreasX2 *out = nullptr)
{
    const AreasX2 a = areas_exact<K>(V, s, m);
    if (out) *out = a;
    iou = iou_from_areas(a);
    if (!(a.ai > 0.0)) {
        m = 0;
#pragma unroll
        for (int q = 0; q < Seq<K>::NW; ++q) s.w[q] = 0ull;
    }
}

}  // namespace dgal
