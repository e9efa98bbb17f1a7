/*
 * oracle/oracle.c -- plain, slow, double-precision CPU oracle for batched
 * differentiable IoU of convex polygons (DGAL, arXiv 2011.11134).
 *
 * TEST INFRASTRUCTURE.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load, call or link this library.
 * The product path (paper_2011_11134_b200/) never does.  It shares no source,
 * header, table or constant generator with the CUDA path (csrc/, include/).
 *
 * Citations: "P:n" = PAPER.md line n, "S:n" = SPEC.md line n, "R#" = a reading
 * listed in DESIGN.md §3 (taken from SURVEY.md §8(c)).
 *
 * What it computes (the paper's §II-B listing):
 *   iou(p1,p2) = area(p1 ∩ p2) / (area(p1) + area(p2) - area(p1 ∩ p2)),
 *   plus nx = #vertices of p1 ∩ p2 and xflags = their provenance bytes, and
 *   iou_grad: d IoU / d(vertices of p1 and p2), scaled by the upstream grad.
 *
 * The forward is written from the DEFINITION of the convex intersection, not
 * from any clipping algorithm (SURVEY §8(c) "Oracle algorithm"):
 *   1. candidates: p1 vertices inside-or-on p2 (FromP1), p2 vertices inside p1
 *      (FromP2), proper segment crossings (Cross);  de-duplicated with the
 *      priority FromP1 > FromP2 > Cross;
 *   2. < 3 points -> empty;
 *   3. CCW order by atan2 about the mean;
 *   4. shoelace area; area <= 0 -> empty (R7);
 *   5. canonical start (R3): the first vertex met walking p1's boundary
 *      counter-clockwise from p1's vertex 0 (FromP2(0) when p1's boundary does
 *      not touch p1 ∩ p2, i.e. p2 inside p1);
 *   6. IoU.
 * The backward is the analytic chain rule of S:303 over the oracle's own
 * vertices/flags: area_grad of the intersection, routed by flag
 * (S:278-283); a crossing vertex is differentiated as the intersection of the
 * two supporting lines (implicit differentiation, derived in DESIGN.md §3.4).
 * Its correctness is pinned by central finite differences (tests/).
 *
 * Flag byte encoding (R2, following the worked examples S:102-103):
 *   FromP1(i) = 0x40 | i,  FromP2(j) = 0x80 | j,  Cross(i,j) = 0xC0 | i<<3 | j,
 *   padding = 0x00.
 *
 * Build: gcc -O2 -ffp-contract=off -fno-fast-math -fopenmp -shared -fPIC
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#ifdef _OPENMP
#include <omp.h>
#endif

#define OR_MAXK 8
#define OR_MAXC (OR_MAXK + OR_MAXK + OR_MAXK * OR_MAXK) /* candidate points */

typedef struct { double x, y; } vec2;

static vec2 v2(double x, double y) { vec2 r = {x, y}; return r; }
static vec2 vsub(vec2 a, vec2 b) { return v2(a.x - b.x, a.y - b.y); }
static vec2 vadd(vec2 a, vec2 b) { return v2(a.x + b.x, a.y + b.y); }
static vec2 vscale(vec2 a, double s) { return v2(a.x * s, a.y * s); }
static double vcross(vec2 a, vec2 b) { return a.x * b.y - a.y * b.x; }
static double vdot(vec2 a, vec2 b) { return a.x * b.x + a.y * b.y; }
/* u-perp as used by the area gradient: (u_y, -u_x) */
static vec2 vperp(vec2 u) { return v2(u.y, -u.x); }

/* Shoelace area of a polygon: 1/2 sum (x_k y_{k+1} - x_{k+1} y_k). */
static double shoelace(const vec2 *p, int n)
{
    double s = 0.0;
    for (int k = 0; k < n; ++k) {
        vec2 a = p[k], b = p[(k + 1) % n];
        s += a.x * b.y - b.x * a.y;
    }
    return 0.5 * s;
}

/* ------------------------------------------------------------------------ */
/* Forward: the intersection polygon by definition                           */
/* ------------------------------------------------------------------------ */
typedef struct {
    int n;                 /* vertex count after normalisation (0 = empty)   */
    int overflow;          /* > 2K distinct candidates (degenerate input)    */
    vec2 v[OR_MAXC];
    uint8_t flag[OR_MAXC];
    double area;           /* area of the intersection, 0 when empty        */
} isect_t;

/* Signed "inside" value of point q w.r.t. the directed edge a->b of a CCW
 * polygon: cross(b - a, q - a) >= 0 means left of (inside) the edge line. */
static double side(vec2 a, vec2 b, vec2 q) { return vcross(vsub(b, a), vsub(q, a)); }

/*
 * Canonical start (R3): the vertex with the smallest position along p1's boundary,
 * measured CCW from p1's vertex 0: FromP1(i) sits at i, Cross(i, j) at i + t with
 * t its parameter on p1 edge i; FromP2 vertices are not on p1's boundary.  If no
 * vertex is on p1's boundary (p2 inside p1) the sequence starts at its smallest
 * byte (FromP2 with the smallest index).
 */
static int canonical_start(int K, const vec2 *P, const vec2 *v, const uint8_t *f, int n)
{
    int best = -1;
    double bkey = 0.0;
    for (int k = 0; k < n; ++k) {
        int tag = f[k] >> 6, i = (f[k] >> 3) & 7, j = f[k] & 7;
        double key;
        if (tag == 1) key = (double)j;
        else if (tag == 3) {
            vec2 a = P[i], e = vsub(P[(i + 1) % K], P[i]);
            key = (double)i + vdot(vsub(v[k], a), e) / vdot(e, e);
        } else continue;
        if (best < 0 || key < bkey) { best = k; bkey = key; }
    }
    if (best >= 0) return best;
    int m = 0;
    for (int k = 1; k < n; ++k)
        if (f[k] < f[m]) m = k;
    return m;
}

static void intersect_by_definition(int K, const vec2 *P, const vec2 *Q, isect_t *out)
{
    vec2 cand[OR_MAXC];
    uint8_t cflag[OR_MAXC];
    int nc = 0;

    /* dedupe tolerance: 1e-9 x the coordinate scale of the pair (its extent: the
     * callers put the pair in its local frame, to_local) */
    double scale = 0.0;
    for (int k = 0; k < K; ++k) {
        scale = fmax(scale, fmax(fabs(P[k].x), fabs(P[k].y)));
        scale = fmax(scale, fmax(fabs(Q[k].x), fabs(Q[k].y)));
    }
    if (!(scale > 0.0)) scale = 1.0;
    const double tol = 1e-9 * scale;
    /* on-boundary tolerance: absorbs the double rounding of coordinates (~1e-16
     * scale), far below any float32 input resolution (~1e-7 scale) */
    const double ton = 1e-12 * scale;

    /* (1a) p1 vertices inside-or-on p2 (boundary-inclusive, R5).  "On" is taken
     * within a rounding tolerance (distance to the edge line >= -ton): a vertex
     * that lies on the other polygon's edge in exact arithmetic (collinear edges,
     * nested boxes) must not be lost to the rounding of its coordinates. */
    for (int i = 0; i < K; ++i) {
        int in = 1;
        for (int j = 0; j < K; ++j) {
            vec2 f = vsub(Q[(j + 1) % K], Q[j]);
            if (side(Q[j], Q[(j + 1) % K], P[i]) < -ton * sqrt(vdot(f, f))) { in = 0; break; }
        }
        if (in) { cand[nc] = P[i]; cflag[nc] = (uint8_t)(0x40 | i); ++nc; }
    }
    /* (1b) p2 vertices inside-or-on p1 (same rounding tolerance), unless coincident with
     * an accepted point */
    for (int j = 0; j < K; ++j) {
        int in = 1;
        for (int i = 0; i < K; ++i) {
            vec2 e = vsub(P[(i + 1) % K], P[i]);
            if (side(P[i], P[(i + 1) % K], Q[j]) < -ton * sqrt(vdot(e, e))) { in = 0; break; }
        }
        if (!in) continue;
        int dup = 0;
        for (int c = 0; c < nc; ++c)
            if (fabs(cand[c].x - Q[j].x) <= tol && fabs(cand[c].y - Q[j].y) <= tol) { dup = 1; break; }
        if (!dup) { cand[nc] = Q[j]; cflag[nc] = (uint8_t)(0x80 | j); ++nc; }
    }
    /* (1c) crossings of segment i of p1 with segment j of p2 */
    for (int i = 0; i < K; ++i) {
        vec2 a = P[i], e = vsub(P[(i + 1) % K], P[i]);
        for (int j = 0; j < K; ++j) {
            vec2 r = Q[j], f = vsub(Q[(j + 1) % K], Q[j]);
            double den = vcross(e, f);
            if (den == 0.0) continue;                     /* parallel segments */
            double t = vcross(vsub(r, a), f) / den;       /* along p1 edge i  */
            double u = vcross(vsub(r, a), e) / den;       /* along p2 edge j  */
            if (t < 0.0 || t > 1.0 || u < 0.0 || u > 1.0) continue;
            vec2 X = vadd(a, vscale(e, t));
            int dup = 0;
            for (int c = 0; c < nc; ++c)
                if (fabs(cand[c].x - X.x) <= tol && fabs(cand[c].y - X.y) <= tol) { dup = 1; break; }
            if (!dup) { cand[nc] = X; cflag[nc] = (uint8_t)(0xC0 | (i << 3) | j); ++nc; }
        }
    }

    out->n = 0; out->overflow = 0; out->area = 0.0;
    if (nc < 3) return;                                  /* (2) empty       */

    /* (3) CCW order: sort by angle about the mean (insertion sort) */
    vec2 m = v2(0.0, 0.0);
    for (int c = 0; c < nc; ++c) m = vadd(m, cand[c]);
    m = vscale(m, 1.0 / nc);
    double ang[OR_MAXC];
    for (int c = 0; c < nc; ++c) ang[c] = atan2(cand[c].y - m.y, cand[c].x - m.x);
    for (int a = 1; a < nc; ++a) {
        double ka = ang[a]; vec2 kv = cand[a]; uint8_t kf = cflag[a];
        int b = a - 1;
        while (b >= 0 && ang[b] > ka) { ang[b + 1] = ang[b]; cand[b + 1] = cand[b]; cflag[b + 1] = cflag[b]; --b; }
        ang[b + 1] = ka; cand[b + 1] = kv; cflag[b + 1] = kf;
    }

    /* (4) shoelace; degenerate -> empty (R7) */
    double A = shoelace(cand, nc);
    if (!(A > 0.0)) return;

    /* (5) canonical start (R3) */
    int s = canonical_start(K, P, cand, cflag, nc);
    for (int c = 0; c < nc; ++c) {
        out->v[c] = cand[(s + c) % nc];
        out->flag[c] = cflag[(s + c) % nc];
    }
    out->n = nc;
    out->overflow = nc > 2 * K;
    out->area = A;
}

static void load_poly(int K, const double *x, const double *y, vec2 *p)
{
    for (int k = 0; k < K; ++k) p[k] = v2(x[k], y[k]);
}

/* Local frame of a pair: both polygons translated by -o (o = p1's vertex 0, returned).
 * IoU, flags and vertex gradients are translation invariant ("rigid
 * invariance"); computing them about a point of the pair keeps every coordinate,
 * shoelace product and dedupe tolerance at the size of the pair instead of its
 * distance from the origin (a 0.2 m box 10 km away: the absolute-coordinate shoelace
 * and a 1e-9 x |coordinate| dedupe tolerance put 1e-4 on the IoU).  The differences
 * of float-valued inputs are exact in double. */
static vec2 to_local(int K, vec2 *P, vec2 *Q)
{
    vec2 o = P[0];
    for (int k = 0; k < K; ++k) { P[k] = vsub(P[k], o); Q[k] = vsub(Q[k], o); }
    return o;
}

/* IoU of one pair.  Returns IoU; fills nx/xflags (2K bytes). */
static double iou_pair(int K, const vec2 *P, const vec2 *Q, isect_t *I,
                       double *A1o, double *A2o)
{
    intersect_by_definition(K, P, Q, I);
    double A1 = shoelace(P, K), A2 = shoelace(Q, K);
    if (A1o) *A1o = A1;
    if (A2o) *A2o = A2;
    /* |P1 n P2| <= min(|P1|, |P2|) (set inclusion): a polygon of zero area (all
     * vertices equal: its zero-length edges constrain nothing, so the other polygon's
     * vertices all test "inside" it) has an empty intersection, IoU 0 (0 <= IoU
     * <= 1 always; without this a point p2 inside p1 gave IoU = A1 / rounding) */
    if (!(A1 > 0.0) || !(A2 > 0.0)) { I->n = 0; I->area = 0.0; return 0.0; }
    double Au = A1 + A2 - I->area;
    if (I->n == 0 || !(Au > 0.0)) return 0.0;           /* R10 guard */
    return I->area / Au;
}

static int resolve_threads(int nthreads)
{
#ifdef _OPENMP
    return nthreads > 0 ? nthreads : omp_get_max_threads();
#else
    (void)nthreads;
    return 1;
#endif
}

int oracle_max_threads(void) { return resolve_threads(0); }

/* ------------------------------------------------------------------------ */
/* Exported forward                                                          */
/* ------------------------------------------------------------------------ */
/*
 * oracle_iou_paired_fwd: for every pair k in [0, n):
 *   iou[k], nx[k], xflags[k*2K .. k*2K+2K-1] (padding 0x00), area_i[k] (nullable),
 *   status[k] (nullable): 0 ok, 1 more than 2K distinct vertices (degenerate).
 * Inputs are (n*K) doubles per coordinate plane (SoA, S:45-52 / P:67).
 */
int oracle_iou_paired_fwd(int K, int64_t n,
                          const double *x1, const double *y1,
                          const double *x2, const double *y2,
                          double *iou, uint8_t *nx, uint8_t *xflags,
                          double *area_i, uint8_t *status, int nthreads)
{
    if (K < 3 || K > OR_MAXK || n < 0) return 1;
    int nt = resolve_threads(nthreads);
#pragma omp parallel for schedule(static) num_threads(nt)
    for (int64_t k = 0; k < n; ++k) {
        vec2 P[OR_MAXK], Q[OR_MAXK];
        isect_t I;
        load_poly(K, x1 + k * K, y1 + k * K, P);
        load_poly(K, x2 + k * K, y2 + k * K, Q);
        to_local(K, P, Q);
        double v = iou_pair(K, P, Q, &I, NULL, NULL);
        int cap = 2 * K, nv = I.n < cap ? I.n : cap;
        iou[k] = v;
        if (nx) nx[k] = (uint8_t)nv;
        if (xflags) {
            for (int c = 0; c < cap; ++c) xflags[k * cap + c] = c < nv ? I.flag[c] : 0;
        }
        if (area_i) area_i[k] = I.area;
        if (status) status[k] = (uint8_t)I.overflow;
    }
    return 0;
}

/* One pair, with the intersection vertices (tests: flag faithfulness). */
int oracle_intersect_one(int K, const double *x1, const double *y1,
                         const double *x2, const double *y2,
                         double *vx, double *vy, uint8_t *flags, int *nv,
                         double *areas /* [3] = A1, A2, Ai */)
{
    if (K < 3 || K > OR_MAXK) return 1;
    vec2 P[OR_MAXK], Q[OR_MAXK];
    isect_t I;
    load_poly(K, x1, y1, P);
    load_poly(K, x2, y2, Q);
    const vec2 o = to_local(K, P, Q);
    double A1, A2;
    (void)iou_pair(K, P, Q, &I, &A1, &A2);
    for (int c = 0; c < I.n; ++c) { vx[c] = I.v[c].x + o.x; vy[c] = I.v[c].y + o.y; flags[c] = I.flag[c]; }
    *nv = I.n;
    if (areas) { areas[0] = A1; areas[1] = A2; areas[2] = I.area; }
    return 0;
}

/* Area of n polygons with K vertices each. */
int oracle_area(int K, int64_t n, const double *x, const double *y, double *out)
{
    if (K < 1 || K > 64) return 1;
    for (int64_t k = 0; k < n; ++k) {
        vec2 P[64];
        load_poly(K, x + k * K, y + k * K, P);
        for (int v = K - 1; v >= 0; --v) P[v] = vsub(P[v], P[0]);   /* about vertex 0 */
        out[k] = shoelace(P, K);
    }
    return 0;
}

/* ------------------------------------------------------------------------ */
/* Backward: iou_grad                                   */
/* ------------------------------------------------------------------------ */
/* d area / d vertex k of a CCW polygon:
 *   dA/dx_k = (y_{k+1} - y_{k-1}) / 2,  dA/dy_k = (x_{k-1} - x_{k+1}) / 2.   */
static vec2 area_grad_at(const vec2 *p, int n, int k)
{
    vec2 nx_ = p[(k + 1) % n], pv = p[(k + n - 1) % n];
    return v2(0.5 * (nx_.y - pv.y), 0.5 * (pv.x - nx_.x));
}

/*
 * VJP of X = line(P,Q) ∩ line(R,S) w.r.t. P, Q, R, S for cotangent G.
 * Derivation: X satisfies cross(X-P, e) = 0 and
 * cross(X-R, f) = 0 with e = Q-P, f = S-R, D = cross(e, f).  Differentiating
 * both constraints and solving for dX gives
 *   dX/dR . d = cross(d, S-X)/D * e      dX/dS . d = cross(d, X-R)/D * e
 *   dX/dP . d = -cross(d, Q-X)/D * f     dX/dQ . d = -cross(d, X-P)/D * f
 * so with cross(d, u) = d . perp(u):
 *   gR = (G.e)/D perp(S-X),  gS = (G.e)/D perp(X-R),
 *   gP = -(G.f)/D perp(Q-X), gQ = -(G.f)/D perp(X-P).
 */
static void crossing_vjp(vec2 P, vec2 Q, vec2 R, vec2 S, vec2 X, vec2 G,
                         vec2 *gP, vec2 *gQ, vec2 *gR, vec2 *gS)
{
    vec2 e = vsub(Q, P), f = vsub(S, R);
    double D = vcross(e, f);
    double ae = vdot(G, e) / D, af = vdot(G, f) / D;
    *gR = vscale(vperp(vsub(S, X)), ae);
    *gS = vscale(vperp(vsub(X, R)), ae);
    *gP = vscale(vperp(vsub(Q, X)), -af);
    *gQ = vscale(vperp(vsub(X, P)), -af);
}

/* Intersection point of line (P,Q) and line (R,S). */
static vec2 line_cross(vec2 P, vec2 Q, vec2 R, vec2 S)
{
    vec2 e = vsub(Q, P), f = vsub(S, R);
    double t = vcross(vsub(R, P), f) / vcross(e, f);
    return vadd(P, vscale(e, t));
}

/*
 * Vertex gradients of  ci * A(p1 ∩ p2) + cu1 * A(p1) + cu2 * A(p2)  (the A_i, A_1,
 * A_2 paths of S:303): area_grad of p1 and p2 plus the area_grad of the
 * intersection routed by flag through the crossing VJP.
 */
static void area_paths_grad(int K, const vec2 *P, const vec2 *Q, const isect_t *I, double ci, double cu1,
                            double cu2, vec2 *g1, vec2 *g2)
{
    for (int k = 0; k < K; ++k) {
        g1[k] = vscale(area_grad_at(P, K, k), cu1);
        g2[k] = vscale(area_grad_at(Q, K, k), cu2);
    }
    /* vertices rebuilt from the flags, ascending order */
    vec2 X[OR_MAXC];
    for (int c = 0; c < I->n; ++c) {
        uint8_t b = I->flag[c];
        int tag = b >> 6, i = (b >> 3) & 7, j = b & 7;
        if (tag == 1) X[c] = P[j];
        else if (tag == 2) X[c] = Q[j];
        else X[c] = line_cross(P[i], P[(i + 1) % K], Q[j], Q[(j + 1) % K]);
    }
    for (int c = 0; c < I->n; ++c) {
        vec2 G = vscale(area_grad_at(X, I->n, c), ci);
        uint8_t b = I->flag[c];
        int tag = b >> 6, i = (b >> 3) & 7, j = b & 7;
        if (tag == 1) {
            g1[j] = vadd(g1[j], G);
        } else if (tag == 2) {
            g2[j] = vadd(g2[j], G);
        } else if (tag == 3) {
            vec2 gP, gQ, gR, gS;
            crossing_vjp(P[i], P[(i + 1) % K], Q[j], Q[(j + 1) % K], X[c], G, &gP, &gQ, &gR, &gS);
            g1[i] = vadd(g1[i], gP);
            g1[(i + 1) % K] = vadd(g1[(i + 1) % K], gQ);
            g2[j] = vadd(g2[j], gR);
            g2[(j + 1) % K] = vadd(g2[(j + 1) % K], gS);
        }
    }
}

static void iou_grad_pair(int K, const vec2 *P, const vec2 *Q, double g,
                          vec2 *g1, vec2 *g2)
{
    for (int k = 0; k < K; ++k) { g1[k] = v2(0.0, 0.0); g2[k] = v2(0.0, 0.0); }
    isect_t I;
    double A1, A2;
    (void)iou_pair(K, P, Q, &I, &A1, &A2);
    double Ai = I.area, Au = A1 + A2 - Ai;
    if (I.n == 0 || !(Au > 0.0)) return;                 /* zero subgradient */

    /* dIoU/dAi = (Au + Ai)/Au^2, dIoU/dA1 = dIoU/dA2 = -Ai/Au^2 */
    double ci = g * (Au + Ai) / (Au * Au);
    double cu = -g * Ai / (Au * Au);
    area_paths_grad(K, P, Q, &I, ci, cu, cu, g1, g2);
}

/*
 * oracle_iou_paired_bwd: grad_iou[k] = dL/dIoU of pair k;  outputs
 * dL/d(p1 vertices) and dL/d(p2 vertices) in the input SoA layout.
 * The oracle recomputes its own intersection and flags (it takes no input
 * from the CUDA path).
 */
int oracle_iou_paired_bwd(int K, int64_t n,
                          const double *x1, const double *y1,
                          const double *x2, const double *y2,
                          const double *grad_iou,
                          double *gx1, double *gy1, double *gx2, double *gy2,
                          int nthreads)
{
    if (K < 3 || K > OR_MAXK || n < 0) return 1;
    int nt = resolve_threads(nthreads);
#pragma omp parallel for schedule(static) num_threads(nt)
    for (int64_t k = 0; k < n; ++k) {
        vec2 P[OR_MAXK], Q[OR_MAXK], g1[OR_MAXK], g2[OR_MAXK];
        load_poly(K, x1 + k * K, y1 + k * K, P);
        load_poly(K, x2 + k * K, y2 + k * K, Q);
        to_local(K, P, Q);
        iou_grad_pair(K, P, Q, grad_iou[k], g1, g2);
        for (int v = 0; v < K; ++v) {
            gx1[k * K + v] = g1[v].x; gy1[k * K + v] = g1[v].y;
            gx2[k * K + v] = g2[v].x; gy2[k * K + v] = g2[v].y;
        }
    }
    return 0;
}

/* ------------------------------------------------------------------------ */
/* Pairwise IoU and NMS (north_star)            */
/* ------------------------------------------------------------------------ */
/* out[r*m + c] = IoU(rows[r], cols[c]); rows play p1 (subject), cols p2 (R4). */
int oracle_iou_pairwise(int K, int64_t nr, const double *rx, const double *ry,
                        int64_t m, const double *cx, const double *cy,
                        double *out, int nthreads)
{
    if (K < 3 || K > OR_MAXK || nr < 0 || m < 0) return 1;
    int nt = resolve_threads(nthreads);
#pragma omp parallel for schedule(dynamic, 1) num_threads(nt)
    for (int64_t r = 0; r < nr; ++r) {
        vec2 P[OR_MAXK], Q[OR_MAXK];
        isect_t I;
        vec2 P0[OR_MAXK];
        load_poly(K, rx + r * K, ry + r * K, P0);
        for (int64_t c = 0; c < m; ++c) {
            for (int v = 0; v < K; ++v) P[v] = P0[v];
            load_poly(K, cx + c * K, cy + c * K, Q);
            to_local(K, P, Q);
            out[r * m + c] = iou_pair(K, P, Q, &I, NULL, NULL);
        }
    }
    return 0;
}

/* Sparse pairwise: IoU of the listed (row, col) pairs only. */
int oracle_iou_pairs_indexed(int K, int64_t npairs, const int64_t *ri, const int64_t *ci,
                             const double *rx, const double *ry,
                             const double *cx, const double *cy,
                             double *out, int nthreads)
{
    if (K < 3 || K > OR_MAXK || npairs < 0) return 1;
    int nt = resolve_threads(nthreads);
#pragma omp parallel for schedule(static) num_threads(nt)
    for (int64_t k = 0; k < npairs; ++k) {
        vec2 P[OR_MAXK], Q[OR_MAXK];
        isect_t I;
        load_poly(K, rx + ri[k] * K, ry + ri[k] * K, P);
        load_poly(K, cx + ci[k] * K, cy + ci[k] * K, Q);
        to_local(K, P, Q);
        out[k] = iou_pair(K, P, Q, &I, NULL, NULL);
    }
    return 0;
}

/*
 * Textbook greedy NMS on a dense IoU matrix (boxes pre-sorted by score):
 *   for i ascending: if !removed[i]: keep i; for j > i: if IoU(i,j) > thr: removed[j].
 */
int oracle_nms_greedy(int64_t n, const double *iou, double thr, uint8_t *keep)
{
    uint8_t *removed = (uint8_t *)calloc((size_t)(n > 0 ? n : 1), 1);
    if (!removed) return 2;
    for (int64_t i = 0; i < n; ++i) {
        keep[i] = 0;
        if (removed[i]) continue;
        keep[i] = 1;
        for (int64_t j = i + 1; j < n; ++j)
            if (iou[i * n + j] > thr) removed[j] = 1;
    }
    free(removed);
    return 0;
}

/*
 * Greedy scan over a given suppression bit mask (R14: keep parity is checked
 * as oracle_scan(gpu_mask) == gpu_keep).  mask row i has `words` uint64; only
 * bits j > i are read (bit j of row i: box i suppresses box j).
 */
int oracle_nms_scan_mask(int64_t n, int64_t words, const uint64_t *mask, uint8_t *keep)
{
    uint8_t *removed = (uint8_t *)calloc((size_t)(n > 0 ? n : 1), 1);
    if (!removed) return 2;
    for (int64_t i = 0; i < n; ++i) {
        keep[i] = 0;
        if (removed[i]) continue;
        keep[i] = 1;
        for (int64_t j = i + 1; j < n; ++j)
            if ((mask[i * words + (j >> 6)] >> (j & 63)) & 1u) removed[j] = 1;
    }
    free(removed);
    return 0;
}

/* ------------------------------------------------------------------------ */
/* Secondary oracle (tests only): literal Sutherland-Hodgman clip      */
/* ------------------------------------------------------------------------ */
/*
 * p1 is the subject, p2 the clipper.  Every working vertex carries a
 * flag and every working edge a supporting-line id: P1-edge i (id = i) or
 * P2-edge j (id = 8 + j).  Clip by half-plane j keeps points with
 * side >= 0 (boundary-inclusive, R5).  A crossing on an edge with id P1-i is
 * Cross(i,j); on an edge with id P2-j1 it snaps to the shared p2 vertex when
 * j1, j are adjacent (FromP2), else CrossP2P2 (tag 00) (R8).
 * Output: canonical start (R3), empty when < 3 vertices or area <= 0.
 */
int oracle_sh_intersect(int K, int64_t n,
                        const double *x1, const double *y1,
                        const double *x2, const double *y2,
                        uint8_t *nx, uint8_t *xflags, double *area_i)
{
    if (K < 3 || K > OR_MAXK || n < 0) return 1;
    for (int64_t k = 0; k < n; ++k) {
        vec2 P[OR_MAXK], Q[OR_MAXK];
        load_poly(K, x1 + k * K, y1 + k * K, P);
        load_poly(K, x2 + k * K, y2 + k * K, Q);
        to_local(K, P, Q);
        vec2 cur[4 * OR_MAXK], nxt[4 * OR_MAXK];
        uint8_t cf[4 * OR_MAXK], nf[4 * OR_MAXK];
        int ce[4 * OR_MAXK], ne[4 * OR_MAXK];   /* id of edge cur[c] -> cur[c+1] */
        int nc = K;
        for (int i = 0; i < K; ++i) { cur[i] = P[i]; cf[i] = (uint8_t)(0x40 | i); ce[i] = i; }
        for (int j = 0; j < K && nc > 0; ++j) {
            vec2 a = Q[j], b = Q[(j + 1) % K];
            double d[4 * OR_MAXK];
            for (int c = 0; c < nc; ++c) d[c] = side(a, b, cur[c]);
            int nn = 0;
            for (int c = 0; c < nc; ++c) {
                int pc = (c + nc - 1) % nc;
                int in_c = d[c] >= 0.0, in_p = d[pc] >= 0.0;
                if (in_c) {
                    if (!in_p) {   /* entering: crossing on edge pc -> c */
                        double t = d[pc] / (d[pc] - d[c]);
                        vec2 X = vadd(cur[pc], vscale(vsub(cur[c], cur[pc]), t));
                        int eid = ce[pc];
                        uint8_t fl;
                        if (eid < 8) fl = (uint8_t)(0xC0 | (eid << 3) | j);
                        else {
                            int j1 = eid - 8;
                            if ((j1 + 1) % K == j) { fl = (uint8_t)(0x80 | j); X = Q[j]; }
                            else if ((j + 1) % K == j1) { fl = (uint8_t)(0x80 | j1); X = Q[j1]; }
                            else fl = (uint8_t)(((j1 & 7) << 3) | j);
                        }
                        nxt[nn] = X; nf[nn] = fl; ne[nn] = eid; ++nn;
                    }
                    nxt[nn] = cur[c]; nf[nn] = cf[c]; ne[nn] = ce[c]; ++nn;
                } else if (in_p) { /* exiting: crossing on edge pc -> c */
                    double t = d[pc] / (d[pc] - d[c]);
                    vec2 X = vadd(cur[pc], vscale(vsub(cur[c], cur[pc]), t));
                    int eid = ce[pc];
                    uint8_t fl;
                    if (eid < 8) fl = (uint8_t)(0xC0 | (eid << 3) | j);
                    else {
                        int j1 = eid - 8;
                        if ((j1 + 1) % K == j) { fl = (uint8_t)(0x80 | j); X = Q[j]; }
                        else if ((j + 1) % K == j1) { fl = (uint8_t)(0x80 | j1); X = Q[j1]; }
                        else fl = (uint8_t)(((j1 & 7) << 3) | j);
                    }
                    nxt[nn] = X; nf[nn] = fl; ne[nn] = 8 + j; ++nn;
                }
            }
            nc = nn > 4 * OR_MAXK ? 4 * OR_MAXK : nn;
            memcpy(cur, nxt, sizeof(vec2) * nc);
            memcpy(cf, nf, nc);
            memcpy(ce, ne, sizeof(int) * nc);
        }
        double A = nc >= 3 ? shoelace(cur, nc) : 0.0;
        int cap = 2 * K;
        for (int c = 0; c < cap; ++c) xflags[k * cap + c] = 0;
        if (nc < 3 || !(A > 0.0) || nc > cap) {
            nx[k] = 0; if (area_i) area_i[k] = 0.0;
            continue;
        }
        int s = canonical_start(K, P, cur, cf, nc);
        for (int c = 0; c < nc; ++c) xflags[k * cap + c] = cf[(s + c) % nc];
        nx[k] = (uint8_t)nc;
        if (area_i) area_i[k] = A;
    }
    return 0;
}

/* ------------------------------------------------------------------------ */
/* Margin from degeneracy (R13) — used by the tests' input filter             */
/* ------------------------------------------------------------------------ */
/*
 * For each pair: dist[k] = (smallest decision distance) / sqrt(min(A1, A2)), over
 *   (a) every p1 vertex vs every p2 edge line,
 *   (b) every p2 vertex vs every p1 edge line,
 *   (c) every Cross vertex of p1 ∩ p2 vs every other edge line of p1 and p2;
 * sinmin[k] = smallest |sin| of the crossing angle over the Cross vertices
 * (1 when there is none).  A pair is "a stated margin away from degeneracy"
 * (north_star) iff dist >= 1e-3 and sinmin >= 1e-2 (R13).
 */
static double dist_to_line(vec2 a, vec2 b, vec2 q)
{
    vec2 e = vsub(b, a);
    return fabs(vcross(e, vsub(q, a))) / sqrt(vdot(e, e));
}

int oracle_margin(int K, int64_t n, const double *x1, const double *y1,
                  const double *x2, const double *y2, double *dist, double *sinmin,
                  int nthreads)
{
    if (K < 3 || K > OR_MAXK || n < 0) return 1;
    int nt = resolve_threads(nthreads);
#pragma omp parallel for schedule(static) num_threads(nt)
    for (int64_t k = 0; k < n; ++k) {
        vec2 P[OR_MAXK], Q[OR_MAXK];
        isect_t I;
        load_poly(K, x1 + k * K, y1 + k * K, P);
        load_poly(K, x2 + k * K, y2 + k * K, Q);
        to_local(K, P, Q);
        double A1, A2;
        (void)iou_pair(K, P, Q, &I, &A1, &A2);
        double dmin = INFINITY, smin = 1.0;
        for (int i = 0; i < K; ++i)
            for (int j = 0; j < K; ++j) {
                dmin = fmin(dmin, dist_to_line(Q[j], Q[(j + 1) % K], P[i]));
                dmin = fmin(dmin, dist_to_line(P[i], P[(i + 1) % K], Q[j]));
            }
        for (int c = 0; c < I.n; ++c) {
            uint8_t b = I.flag[c];
            if ((b >> 6) != 3) continue;
            int i = (b >> 3) & 7, j = b & 7;
            vec2 e = vsub(P[(i + 1) % K], P[i]), f = vsub(Q[(j + 1) % K], Q[j]);
            smin = fmin(smin, fabs(vcross(e, f)) / sqrt(vdot(e, e) * vdot(f, f)));
            for (int o = 0; o < K; ++o) {
                if (o != i) dmin = fmin(dmin, dist_to_line(P[o], P[(o + 1) % K], I.v[c]));
                if (o != j) dmin = fmin(dmin, dist_to_line(Q[o], Q[(o + 1) % K], I.v[c]));
            }
        }
        dist[k] = dmin / sqrt(fmin(A1, A2));
        sinmin[k] = smin;
    }
    return 0;
}

/* ------------------------------------------------------------------------ */
/* Rotated boxes: 2D (cx, cy, w, h, theta) and yaw-only 3D (cx, cy, cz, w, h, d,
 * theta) — SURVEY §8(f) f1 / f3, SPEC metrics-boxes             */
/* ------------------------------------------------------------------------ */
/* box_to_polygon: corners c + R(theta)(+-w/2, +-h/2), CCW, starting
 * at (-w/2, -h/2). */
static const double kBoxSx[4] = {-0.5, 0.5, 0.5, -0.5};
static const double kBoxSy[4] = {-0.5, -0.5, 0.5, 0.5};

static void box_corners(double cx, double cy, double w, double h, double th, vec2 *P)
{
    double c = cos(th), s = sin(th);
    for (int k = 0; k < 4; ++k) {
        double lx = kBoxSx[k] * w, ly = kBoxSy[k] * h;
        P[k] = v2(cx + c * lx - s * ly, cy + s * lx + c * ly);
    }
}

/* box_to_polygon_grad: VJP of the corner map.  out[0..4] += dL/d(cx,
 * cy, w, h, theta) for corner cotangents G[0..3]. */
static void box_corners_vjp(double w, double h, double th, const vec2 *G, double *out)
{
    double c = cos(th), s = sin(th);
    for (int k = 0; k < 4; ++k) {
        double lx = kBoxSx[k] * w, ly = kBoxSy[k] * h;
        out[0] += G[k].x;                                           /* d/dcx */
        out[1] += G[k].y;                                           /* d/dcy */
        out[2] += G[k].x * c * kBoxSx[k] + G[k].y * s * kBoxSx[k];  /* d/dw  */
        out[3] += -G[k].x * s * kBoxSy[k] + G[k].y * c * kBoxSy[k]; /* d/dh  */
        /* d/dtheta: d(R u)/dtheta = (-s ux - c uy, c ux - s uy) */
        out[4] += G[k].x * (-s * lx - c * ly) + G[k].y * (c * lx - s * ly);
    }
}

/* overlap of the vertical extents [cz - d/2, cz + d/2] */
static double z_overlap(double z1, double d1, double z2, double d2, int *top1, int *bot1)
{
    double t1 = z1 + 0.5 * d1, t2 = z2 + 0.5 * d2, b1 = z1 - 0.5 * d1, b2 = z2 - 0.5 * d2;
    *top1 = t1 <= t2;
    *bot1 = b1 >= b2;
    double dz = fmin(t1, t2) - fmax(b1, b2);
    return dz > 0.0 ? dz : 0.0;
}

/*
 * One box pair.  dims = 2: boxes are (cx, cy, w, h, theta); dims = 3: (cx, cy, cz,
 * w, h, d, theta) and IoU = V_i / (V_1 + V_2 - V_i), V_i = A_i dz.
 * Fills iou, the BEV intersection I, and (if g1/g2) dL/d(box params) for dL/dIoU = g.
 */
static double box_pair(int dims, const double *b1, const double *b2, isect_t *I, double g,
                       double *gb1, double *gb2)
{
    const int np = dims == 3 ? 7 : 5;
    double w1, h1, th1, w2, h2, th2, z1 = 0, d1 = 1, z2 = 0, d2 = 1;
    if (dims == 3) {
        z1 = b1[2]; w1 = b1[3]; h1 = b1[4]; d1 = b1[5]; th1 = b1[6];
        z2 = b2[2]; w2 = b2[3]; h2 = b2[4]; d2 = b2[5]; th2 = b2[6];
    } else {
        w1 = b1[2]; h1 = b1[3]; th1 = b1[4];
        w2 = b2[2]; h2 = b2[3]; th2 = b2[4];
    }
    vec2 P[4], Q[4];
    box_corners(b1[0], b1[1], w1, h1, th1, P);
    box_corners(b2[0], b2[1], w2, h2, th2, Q);
    to_local(4, P, Q);
    double A1, A2;
    (void)iou_pair(4, P, Q, I, &A1, &A2);
    int top1 = 1, bot1 = 1;
    double dz = dims == 3 ? z_overlap(z1, d1, z2, d2, &top1, &bot1) : 1.0;
    double V1 = A1 * d1, V2 = A2 * d2, Vi = I->area * dz, Vu = V1 + V2 - Vi;
    if (gb1) for (int p = 0; p < np; ++p) { gb1[p] = 0.0; gb2[p] = 0.0; }
    if (I->n == 0 || !(Vi > 0.0) || !(Vu > 0.0)) return 0.0;
    double iou = Vi / Vu;
    if (!gb1) return iou;
    /* dIoU/dVi = (Vu + Vi)/Vu^2, dIoU/dV1 = dIoU/dV2 = -Vi/Vu^2 (S:303 with V for A) */
    double cVi = g * (Vu + Vi) / (Vu * Vu), cVu = -g * Vi / (Vu * Vu);
    vec2 g1[4], g2[4];
    area_paths_grad(4, P, Q, I, cVi * dz, cVu * d1, cVu * d2, g1, g2);
    double o1[5] = {0, 0, 0, 0, 0}, o2[5] = {0, 0, 0, 0, 0};
    box_corners_vjp(w1, h1, th1, g1, o1);
    box_corners_vjp(w2, h2, th2, g2, o2);
    if (dims == 3) {
        /* product rule through dz (+-1/0 subgradient of min/max) and d */
        double gdz = cVi * I->area;
        gb1[0] = o1[0]; gb1[1] = o1[1]; gb1[3] = o1[2]; gb1[4] = o1[3]; gb1[6] = o1[4];
        gb2[0] = o2[0]; gb2[1] = o2[1]; gb2[3] = o2[2]; gb2[4] = o2[3]; gb2[6] = o2[4];
        gb1[2] = gdz * ((top1 ? 1.0 : 0.0) - (bot1 ? 1.0 : 0.0));
        gb2[2] = gdz * ((top1 ? 0.0 : 1.0) - (bot1 ? 0.0 : 1.0));
        gb1[5] = cVu * A1 + gdz * 0.5 * ((top1 ? 1.0 : 0.0) + (bot1 ? 1.0 : 0.0));
        gb2[5] = cVu * A2 + gdz * 0.5 * ((top1 ? 0.0 : 1.0) + (bot1 ? 0.0 : 1.0));
    } else {
        for (int p = 0; p < 5; ++p) { gb1[p] = o1[p]; gb2[p] = o2[p]; }
    }
    return iou;
}

/*
 * oracle_box_iou_paired: boxes as n x (5 | 7) row-major doubles.  Outputs iou[n],
 * nx[n], xflags[n*8] (of the BEV intersection, as for Poly2<float,4>), and — if
 * grad_iou != NULL — dL/d(box params) in gb1, gb2 (same shape as the boxes).
 */
int oracle_box_iou_paired(int dims, int64_t n, const double *b1, const double *b2, double *iou,
                          uint8_t *nx, uint8_t *xflags, const double *grad_iou, double *gb1, double *gb2,
                          int nthreads)
{
    if ((dims != 2 && dims != 3) || n < 0) return 1;
    const int np = dims == 3 ? 7 : 5;
    int nt = resolve_threads(nthreads);
#pragma omp parallel for schedule(static) num_threads(nt)
    for (int64_t k = 0; k < n; ++k) {
        isect_t I;
        double g = grad_iou ? grad_iou[k] : 0.0;
        double v = box_pair(dims, b1 + k * np, b2 + k * np, &I, g, grad_iou ? gb1 + k * np : NULL,
                            grad_iou ? gb2 + k * np : NULL);
        if (iou) iou[k] = v;
        int nv = v > 0.0 ? (I.n < 8 ? I.n : 8) : 0;
        if (nx) nx[k] = (uint8_t)nv;
        if (xflags)
            for (int c = 0; c < 8; ++c) xflags[k * 8 + c] = c < nv ? I.flag[c] : 0;
    }
    return 0;
}

/* Corners of n boxes (2D params, n x 5) as SoA x[n*4], y[n*4] (tests: margin filter). */
int oracle_box_corners(int64_t n, const double *b, double *x, double *y)
{
    for (int64_t k = 0; k < n; ++k) {
        vec2 P[4];
        box_corners(b[k * 5 + 0], b[k * 5 + 1], b[k * 5 + 2], b[k * 5 + 3], b[k * 5 + 4], P);
        for (int v = 0; v < 4; ++v) { x[k * 4 + v] = P[v].x; y[k * 4 + v] = P[v].y; }
    }
    return 0;
}

/* box_to_polygon_grad for n 2D boxes (n x 5) with corner cotangents gx, gy (n x 4). */
int oracle_box_corners_vjp(int64_t n, const double *b, const double *gx, const double *gy, double *out)
{
    for (int64_t k = 0; k < n; ++k) {
        vec2 G[4];
        for (int v = 0; v < 4; ++v) G[v] = v2(gx[k * 4 + v], gy[k * 4 + v]);
        double o[5] = {0, 0, 0, 0, 0};
        box_corners_vjp(b[k * 5 + 2], b[k * 5 + 3], b[k * 5 + 4], G, o);
        for (int p = 0; p < 5; ++p) out[k * 5 + p] = o[p];
    }
    return 0;
}
