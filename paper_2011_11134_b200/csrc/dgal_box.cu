// dgal_box.cu — rotated-box front end of the paired IoU path (SURVEY §8(f) f1 and
// f3; SPEC metrics-boxes S:336-418; "2D IoU Loss and 3D IoU Loss for
// rotated bounding boxes").  DESIGN.md §4.7.
//
// The boxes are read as parameters (20 B per 2D box, 28 B per yaw-only 3D box
// instead of 32 B of corners) and turned into Poly<4> in registers:
//   box_to_polygon: corners c + R(theta)(+-w/2, +-h/2), CCW from (-w/2, -h/2),
// taken relative to the centre of box 1 and then to its corner 0 (IoU is
// translation invariant; corners near 0 keep the decision predicates accurate).  The clip, the flags and the
// backward phases are the polygon path's (dgal_core.cuh).  3D: V = A d, V_i =
// A_i dz with dz the overlap of the z extents.  The backward maps the
// corner gradients to the box parameters (box_to_polygon_grad) and adds
// the dz / d terms of the product rule.
//
// Layout: parameter p of box k is b[k * sk + p * sp]; planes (sk = 1, sp = n:
// coalesced, the fast layout) or rows (sk = P, sp = 1: a torch [n, P] tensor).
// Parameter order: 2D (cx, cy, w, h, theta), 3D (cx, cy, cz, w, h, d, theta).
#include "dgal_core.cuh"
#include "dgal_internal.h"
#include "dgal_pipe.cuh"
#include "dgal_refine.cuh"

namespace dgal {

namespace {

// backward / fused CTA shapes (A/B on B200, 2^24 KITTI pairs: backward 256 x 3 CTAs
// 0.62 / 0.68 ms (2D / 3D) -> 128 x 7 / 128 x 6 0.59 / 0.65; fused 256 x 2 0.64 /
// 0.78 -> 128 x 4 0.59 / 0.74; the largest CTA counts without spills)
#ifndef DGAL_BOX_BWD_TILE
#define DGAL_BOX_BWD_TILE 128
#endif
#ifndef DGAL_BOX_BWD2_MINB
#define DGAL_BOX_BWD2_MINB 7
#endif
#ifndef DGAL_BOX_BWD3_MINB
#define DGAL_BOX_BWD3_MINB 6
#endif
#ifndef DGAL_BOX_FUSED_PK
#define DGAL_BOX_FUSED_PK true   // 2D: gradient part in paired FP32 (A/B: 0.593 -> 0.584 ms; 3D 0.674 -> 0.683, not used)
#endif
#ifndef DGAL_BOX_FUSED_T
#define DGAL_BOX_FUSED_T 128
#endif
constexpr int kBoxTile = DGAL_BOX_BWD_TILE;  // backward tile = CTA size
constexpr int kBoxFusedT = DGAL_BOX_FUSED_T;
#ifndef DGAL_BOX_FUSED_NT
#define DGAL_BOX_FUSED_NT 8   // tiles per CTA with the prefetch ring (DGAL_BOX_PF)
#endif
// CTAs per SM the box forward / fused kernels are register-budgeted for (the
// largest without local-memory spills, tools/sass_stats.py)
#ifndef DGAL_BOX_FWD2_MINB
#define DGAL_BOX_FWD2_MINB 6
#endif
#ifndef DGAL_BOX_FWD3_MINB
#define DGAL_BOX_FWD3_MINB 4
#endif
// forward CTA shape (as the K = 4 polygon forward: 128 threads, 8 tiles per CTA so
// the walk-table fill is amortised)
#ifndef DGAL_BOX_FWD_T
#define DGAL_BOX_FWD_T 128
#endif
#ifndef DGAL_BOX_FWD_NT
#define DGAL_BOX_FWD_NT 8
#endif
constexpr int kBoxFwdT = DGAL_BOX_FWD_T, kBoxFwdNT = DGAL_BOX_FWD_NT;
#ifndef DGAL_BOX_FUSED2_MINB
#define DGAL_BOX_FUSED2_MINB 4
#endif
#ifndef DGAL_BOX_FUSED3_MINB
#define DGAL_BOX_FUSED3_MINB 4
#endif

template <int DIMS>
struct Box {
    float cx, cy, cz, w, h, d, th;
};

template <int DIMS>
__device__ __forceinline__ Box<DIMS> load_box(const float *__restrict__ b, int64_t k, int64_t sk, int64_t sp)
{
    const float *p = b + k * sk;
    Box<DIMS> r;
    r.cx = __ldg(p);
    r.cy = __ldg(p + sp);
    if (DIMS == 3) {
        r.cz = __ldg(p + 2 * sp); r.w = __ldg(p + 3 * sp); r.h = __ldg(p + 4 * sp);
        r.d = __ldg(p + 5 * sp); r.th = __ldg(p + 6 * sp);
    } else {
        r.cz = 0.f; r.w = __ldg(p + 2 * sp); r.h = __ldg(p + 3 * sp); r.d = 1.f; r.th = __ldg(p + 4 * sp);
    }
    return r;
}

// Per-thread prefetch ring of box parameters (DGAL_BOX_PF): parameter q of box 1 /
// box 2 of this thread's pair at v[stage][q][tid] / v[stage][P + q][tid], copied
// with 4-byte cp.async (any layout: planes or rows), dL/dIoU at g[stage][tid].
// Each thread copies and reads only its own words (no CTA barrier).
#ifndef DGAL_BOX_PF
#define DGAL_BOX_PF 1
#endif
template <int DIMS, int T>
struct BoxRing {
    static constexpr int P = DIMS == 3 ? 7 : 5;
    float v[2][2 * P][T];
    float g[2][T];
    __device__ __forceinline__ void prefetch(int stage, const float *__restrict__ b1, const float *__restrict__ b2,
                                             const float *__restrict__ grad, int64_t k, int64_t sk, int64_t sp,
                                             int tid)
    {
#pragma unroll
        for (int q = 0; q < P; ++q) {
            cp_async4(&v[stage][q][tid], b1 + k * sk + q * sp);
            cp_async4(&v[stage][P + q][tid], b2 + k * sk + q * sp);
        }
        if (grad) cp_async4(&g[stage][tid], grad + k);
    }
    __device__ __forceinline__ Box<DIMS> get(int stage, int which, int tid) const
    {
        const float *r = &v[stage][which * P][0];
        Box<DIMS> b;
        b.cx = r[0 * T + tid];
        b.cy = r[1 * T + tid];
        if (DIMS == 3) {
            b.cz = r[2 * T + tid]; b.w = r[3 * T + tid]; b.h = r[4 * T + tid]; b.d = r[5 * T + tid];
            b.th = r[6 * T + tid];
        } else {
            b.cz = 0.f; b.w = r[2 * T + tid]; b.h = r[3 * T + tid]; b.d = 1.f; b.th = r[4 * T + tid];
        }
        return b;
    }
};

// cos / sin of theta; theta is accepted unbounded.  sincospif(p) of the float
// p = theta * (1/pi) is exact for that p (exact argument reduction inside, no
// Payne-Hanek slow path, no local memory), but p misses theta / pi by up to
// |theta / pi| * 6e-8 of a half turn — 1e-6 of IoU at |theta| = 16, 1e-5 at ~100 rad,
// 9e-5 at 1000 (tools/probes/theta_range.py).  The missing part d = theta/pi - p is
// formed exactly by FMA (the rounding error of the product, plus theta times the low
// part of 1/pi) and applied to first order: sin(pi (p + d)) = sin(pi p) + pi d cos(pi p)
// (the second-order term is < 1e-7 up to |theta| ~ 1e4).  Five FMA-pipe operations,
// no branch.
__device__ __forceinline__ void box_sincos(float th, float &s, float &c)
{
    constexpr float kInvPiHi = 0.318309886183790672f;       // float(1/pi)
    constexpr float kInvPiLo = 1.2841276e-08f;              // 1/pi - float(1/pi)
    const float p = th * kInvPiHi;
    const float pd = fmaf(th, kInvPiLo, fmaf(th, kInvPiHi, -p)) * 3.14159265358979324f;   // pi d
    float s0, c0;
    sincospif(p, &s0, &c0);
    s = fmaf(pd, c0, s0);
    c = fmaf(-pd, s0, c0);
}

// box_to_polygon relative to the origin o: (cx - ox, cy - oy) = (dcx, dcy).
// Contraction-free, so the same parameters always give bitwise the same corners
// (forward and backward agree; identical boxes give identical polygons).
__device__ __forceinline__ void box_poly(float dcx, float dcy, float w, float h, float c, float s, Poly<4> &P)
{
    const float hw = 0.5f * w, hh = 0.5f * h;
    const float cw = __fmul_rn(c, hw), sw = __fmul_rn(s, hw);
    const float ch = __fmul_rn(c, hh), sh = __fmul_rn(s, hh);
    // R (lx, ly) = (c lx - s ly, s lx + c ly) at (-hw,-hh), (hw,-hh), (hw,hh), (-hw,hh)
    P.x[0] = __fadd_rn(dcx, __fsub_rn(sh, cw)); P.y[0] = __fsub_rn(dcy, __fadd_rn(sw, ch));
    P.x[1] = __fadd_rn(dcx, __fadd_rn(cw, sh)); P.y[1] = __fadd_rn(dcy, __fsub_rn(sw, ch));
    P.x[2] = __fadd_rn(dcx, __fsub_rn(cw, sh)); P.y[2] = __fadd_rn(dcy, __fadd_rn(sw, ch));
    P.x[3] = __fsub_rn(dcx, __fadd_rn(cw, sh)); P.y[3] = __fadd_rn(dcy, __fsub_rn(ch, sw));
}

struct Trig {
    float c1, s1, c2, s2;
};

// Corner k of a box in double from its float parameters, as the oracle builds it
// (S:347): centre (dcx, dcy) relative to the frame, cos / sin of theta by sincospi.
__device__ __forceinline__ void box_corner_d(double dcx, double dcy, double w, double h, double s, double c, int k,
                                             double &x, double &y)
{
    const double lx = ((k == 1 || k == 2) ? 0.5 : -0.5) * w, ly = ((k >= 2) ? 0.5 : -0.5) * h;
    x = dcx + (c * lx - s * ly);
    y = dcy + (s * lx + c * ly);
}

// The corners of a box pair in double (frame: box 1's centre; box 2's offset is exact
// in double), the vertex source of the thin-pair areas (dgal_exact.cuh): the float
// corners of a long thin box carry ~eps L of rounding against a width L / aspect
// (aspect 300, L = 60 m at 300 m: up to 1.4e-5 of IoU from the corners alone), the
// oracle's are built from the same float parameters in double.
struct BoxCornersD {
    double dcx, dcy, s1, c1, s2, c2;
    float w1, h1, w2, h2;
    template <int DIMS>
    __device__ __forceinline__ BoxCornersD(const Box<DIMS> &a, const Box<DIMS> &b)
        : dcx((double)b.cx - (double)a.cx), dcy((double)b.cy - (double)a.cy), w1(a.w), h1(a.h), w2(b.w), h2(b.h)
    {
        sincospi((double)a.th * 0.318309886183790671537767526745, &s1, &c1);
        sincospi((double)b.th * 0.318309886183790671537767526745, &s2, &c2);
    }
    __device__ __forceinline__ void p(int k, double &x, double &y) const { box_corner_d(0.0, 0.0, w1, h1, s1, c1, k, x, y); }
    __device__ __forceinline__ void q(int k, double &x, double &y) const { box_corner_d(dcx, dcy, w2, h2, s2, c2, k, x, y); }
};

template <int DIMS>
__device__ __forceinline__ Trig box_pair_polys(const Box<DIMS> &a, const Box<DIMS> &b, Poly<4> &P, Poly<4> &Q)
{
    Trig t;
    box_sincos(a.th, t.s1, t.c1);
    box_sincos(b.th, t.s2, t.c2);
    box_poly(0.f, 0.f, a.w, a.h, t.c1, t.s1, P);
    box_poly(__fsub_rn(b.cx, a.cx), __fsub_rn(b.cy, a.cy), b.w, b.h, t.c2, t.s2, Q);
    // then on p1's corner 0, as the polygon path (same floats for identical boxes;
    // p1.v0 == 0 exactly lets the compiler fold it)
    const float ox = P.x[0], oy = P.y[0];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        P.x[k] = __fsub_rn(P.x[k], ox); P.y[k] = __fsub_rn(P.y[k], oy);
        Q.x[k] = __fsub_rn(Q.x[k], ox); Q.y[k] = __fsub_rn(Q.y[k], oy);
    }
    P.x[0] = 0.f;
    P.y[0] = 0.f;
    return t;
}

// overlap of the z extents [cz - d/2, cz + d/2]; top1 / bot1: the top /
// bottom of the overlap is box 1's (ties to box 1, as in the oracle)
struct ZOver {
    float dz;
    bool top1, bot1;
};

template <int DIMS>
__device__ __forceinline__ ZOver z_overlap(const Box<DIMS> &a, const Box<DIMS> &b)
{
    ZOver z{1.f, true, true};
    if (DIMS == 3) {
        // relative to box 1's centre (dzc exact for nearby centres, Sterbenz): tops and
        // bottoms computed at absolute heights round at ulp(cz) — 6e-5 of IoU at cz ~ 1000 m
        // (tools/probes/box_z.py), while IoU is invariant under a common vertical shift
        const float dzc = __fsub_rn(b.cz, a.cz);
        const float t1 = 0.5f * a.d, t2 = fmaf(0.5f, b.d, dzc);
        const float b1 = -0.5f * a.d, b2 = fmaf(-0.5f, b.d, dzc);
        z.top1 = t1 <= t2;
        z.bot1 = b1 >= b2;
        z.dz = fmaxf(fminf(t1, t2) - fmaxf(b1, b2), 0.f);
    }
    return z;
}

// box_to_polygon_grad: corner cotangents G -> (cx, cy, w, h, theta).
//   d/dc = sum G_k;  d/dw = sum sx_k R^T G_k . e_x;  d/dh = sum sy_k R^T G_k . e_y;
//   d/dtheta = sum G_k . R' u_k = w (-s ax + c ay) + h (-c bx - s by),
// with (ax, ay) = sum sx_k G_k, (bx, by) = sum sy_k G_k, sx = (-,+,+,-)/2, sy = (-,-,+,+)/2.
struct BoxGrad {
    float cx, cy, w, h, th;
};

__device__ __forceinline__ BoxGrad box_vjp(float w, float h, float c, float s, const Poly<4> &G)
{
    BoxGrad o;
    o.cx = (G.x[0] + G.x[1]) + (G.x[2] + G.x[3]);
    o.cy = (G.y[0] + G.y[1]) + (G.y[2] + G.y[3]);
    const float ax = 0.5f * ((G.x[1] + G.x[2]) - (G.x[0] + G.x[3]));
    const float ay = 0.5f * ((G.y[1] + G.y[2]) - (G.y[0] + G.y[3]));
    const float bx = 0.5f * ((G.x[2] + G.x[3]) - (G.x[0] + G.x[1]));
    const float by = 0.5f * ((G.y[2] + G.y[3]) - (G.y[0] + G.y[1]));
    o.w = fmaf(c, ax, s * ay);
    o.h = fmaf(c, by, -s * bx);
    o.th = fmaf(w, fmaf(c, ay, -s * ax), -h * fmaf(c, bx, s * by));
    return o;
}

template <int DIMS>
__device__ __forceinline__ void store_box_grad(float *__restrict__ gb, int64_t k, int64_t sk, int64_t sp,
                                               const BoxGrad &g, float gcz, float gd)
{
    float *p = gb + k * sk;
    p[0] = g.cx;
    p[sp] = g.cy;
    if (DIMS == 3) {
        p[2 * sp] = gcz; p[3 * sp] = g.w; p[4 * sp] = g.h; p[5 * sp] = gd; p[6 * sp] = g.th;
    } else {
        p[2 * sp] = g.w; p[3 * sp] = g.h; p[4 * sp] = g.th;
    }
}

// dz / d terms of the 3D product rule: dL/d(dz) = cvi A_i; dz/dcz = +-1 / 0
// and dz/dd = 1/2 per end owned; dL/dd1 += cvu A_1 (through V_1 = A_1 d1).
template <int DIMS>
__device__ __forceinline__ void z_grads(const VolCoef &co, const ZOver &z, float &gcz1, float &gd1, float &gcz2,
                                        float &gd2)
{
    gcz1 = gd1 = gcz2 = gd2 = 0.f;
    if (DIMS == 3) {
        const float gdz = co.cvi * co.ai;
        const float t1 = z.top1 ? 1.f : 0.f, b1 = z.bot1 ? 1.f : 0.f;
        gcz1 = gdz * (t1 - b1);
        gcz2 = gdz * ((1.f - t1) - (1.f - b1));
        gd1 = fmaf(co.cvu, co.a1, gdz * 0.5f * (t1 + b1));
        gd2 = fmaf(co.cvu, co.a2, gdz * 0.5f * ((1.f - t1) + (1.f - b1)));
    }
}

}  // namespace

// ---------------------------------------------------------------------------
// forward: IoU (2D) or 3D IoU, nx / xflags of the BEV intersection
// ---------------------------------------------------------------------------
template <int DIMS>
__global__ void __launch_bounds__(kBoxFwdT, DIMS == 2 ? DGAL_BOX_FWD2_MINB : DGAL_BOX_FWD3_MINB)
box_fwd_kernel(int64_t n, const float *__restrict__ b1, const float *__restrict__ b2, int64_t sk, int64_t sp,
               float *__restrict__ iou, uint8_t *__restrict__ nx, uint8_t *__restrict__ xflags)
{
    constexpr int T = kBoxFwdT;
    constexpr bool PF = DGAL_BOX_PF;
    // per-thread p2 vertex table (kP2Smem, QTable rows), [thread][slot] with an odd stride
    // (conflict-free): x at slots 0..5, y at 6..11, the zero slots 5 and 11 written once
    // (the "no event" vertex of clip_intervals)
    constexpr int kQS = 13;
    __shared__ float sq[kQS * T];
    float *const sqt = sq + threadIdx.x * kQS;
    __shared__ WalkLut4 wlut;     // flag-walk tables
    __shared__ __align__(16) BoxRing<DIMS, PF ? T : 1> ring;   // tile t+1 in flight while tile t computes
    const int tid = threadIdx.x;
    const int64_t k0 = (int64_t)blockIdx.x * (kBoxFwdNT * T) + tid;
    Box<DIMS> a, b;
    if (PF) {
        if (k0 < n) ring.prefetch(0, b1, b2, nullptr, k0, sk, sp, tid);
        cp_async_commit();
    } else if (k0 < n) {   // the first tile's loads go out before the table fill
        a = load_box<DIMS>(b1, k0, sk, sp);
        b = load_box<DIMS>(b2, k0, sk, sp);
    }
    load_walk_lut4(wlut, tid, T);
    sqt[5] = 0.f;
    sqt[11] = 0.f;
    __syncthreads();
    uint32_t thinmask = 0;   // tiles whose pair is thin (R^2 > kThinRatio A_u)
#pragma unroll 1
    for (int t = 0; t < kBoxFwdNT; ++t) {
        const int64_t k = k0 + (int64_t)t * T;
        if (k >= n) break;
        if (PF) {
            if (t + 1 < kBoxFwdNT && k + T < n) ring.prefetch((t + 1) & 1, b1, b2, nullptr, k + T, sk, sp, tid);
            cp_async_commit();
            cp_async_wait<1>();   // this thread's copies of tile t have landed
            a = ring.get(t & 1, 0, tid);
            b = ring.get(t & 1, 1, tid);
        } else if (t > 0) {
            a = load_box<DIMS>(b1, k, sk, sp);
            b = load_box<DIMS>(b2, k, sk, sp);
        }
        Poly<4> P, Q;
        box_pair_polys<DIMS>(a, b, P, Q);
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            sqt[q] = Q.x[q];
            sqt[6 + q] = Q.y[q];
        }
        sqt[4] = Q.x[0];
        sqt[10] = Q.y[0];
        const FwdOut<4, true> r = iou_fwd<4, true, kP2Smem, DGAL_THIN, true>(P, Q, QTable{sqt, sqt + 6, 1}, &wlut);
        thinmask |= (uint32_t)r.thin << t;   // thin pair: fixed after the loop
        float v = r.iou;
        int m = r.nx;
        uint64_t seq = r.seq.w[0];
        const float A1x2 = r.A1x2, A2x2 = r.A2x2, Aix2 = r.Aix2;
        if (DIMS == 3) {
            const ZOver z = z_overlap<DIMS>(a, b);
            const float Vix2 = Aix2 * z.dz;
            const float Vux2 = (A1x2 * a.d + A2x2 * b.d) - Vix2;
            const bool ok = m > 0 && Vix2 > 0.f && Vux2 > 0.f;
            v = ok ? iou_div(Vix2, Vux2) : 0.f;
            m = ok ? m : 0;
            seq = ok ? seq : 0ull;
        }
        __stcs(iou + k, v);
        nx[k] = (uint8_t)m;
        __stcs(reinterpret_cast<unsigned long long *>(xflags) + k, (unsigned long long)seq);
    }
    // thin pairs (rare; dgal_exact.cuh): the areas of the stored record in double from
    // the corners rebuilt in double from the parameters (BoxCornersD), IoU / volumes
#pragma unroll 1
    while (thinmask) {
        const int t = __ffs(thinmask) - 1;
        thinmask &= thinmask - 1u;
        const int64_t k = k0 + (int64_t)t * T;
        const Box<DIMS> a = load_box<DIMS>(b1, k, sk, sp), b = load_box<DIMS>(b2, k, sk, sp);
        Poly<4> P, Q;
        Seq<4> s2;
        s2.w[0] = reinterpret_cast<const unsigned long long *>(xflags)[k];
        int m = nx[k];
        float v;
        AreasX2 e;
        fwd_thin_redo<4>(BoxCornersD(a, b), s2, m, v, &e);
        if (DIMS == 3 && m > 0) {
            const ZOver z = z_overlap<DIMS>(a, b);
            const double Vi = e.ai * z.dz, Vu = (e.a1 * a.d + e.a2 * b.d) - Vi;
            v = (Vi > 0.0 && Vu > 0.0) ? (float)fmin(Vi / Vu, 1.0) : 0.f;
            if (!(Vi > 0.0 && Vu > 0.0)) { m = 0; s2.w[0] = 0ull; }
        }
        iou[k] = v;
        nx[k] = (uint8_t)m;
        reinterpret_cast<unsigned long long *>(xflags)[k] = s2.w[0];
    }
}

// ---------------------------------------------------------------------------
// backward through the recorded nx / xflags (the polygon path's phases)
// ---------------------------------------------------------------------------
// Exact corners for the refinement of ill-conditioned crossings (bwd_crossing_exact):
// the float corners carry ~6e-8 relative rounding, which a crossing of nearly
// parallel edges amplifies ~1/sin, so they are rebuilt in double from the (float)
// box parameters, as the oracle does: cos / sin by sincospi (exact
// reduction, no local memory), frame = box 1's centre.
struct BoxGeometry {
    // the float corners carry ~2-3 ulp of rounding (sin / cos, products), which a
    // crossing amplifies ~1/sin: at |sin| ~ 2^-10 that was up to 4e-4 relative in the
    // parameter gradients, so box crossings are redone in double below 2^-7
    static constexpr float kRefine = 0.0078125f;
    const float *p;   // staged parameters [param][pair]: cx1, cy1, w1, h1, th1, cx2, cy2, w2, h2, th2
    __device__ __forceinline__ static void corner(double dcx, double dcy, double w, double h, double th, int k,
                                                  double &x, double &y)
    {
        double s, c;
        sincospi(th * 0.318309886183790671537767526745, &s, &c);
        box_corner_d(dcx, dcy, w, h, s, c, k, x, y);
    }
    __device__ __forceinline__ void get(int pt, int i, int i1, int j, int j1, double &vx, double &vy, double &v1x,
                                        double &v1y, double &wx, double &wy, double &w1x, double &w1y) const
    {
        DGAL_ASSERT(pt >= 0 && pt < kBoxTile && i >= 0 && i < 4 && i1 >= 0 && i1 < 4 && j >= 0 && j < 4 && j1 >= 0 && j1 < 4);
        const double dcx = (double)p[5 * kBoxTile + pt] - (double)p[pt];
        const double dcy = (double)p[6 * kBoxTile + pt] - (double)p[kBoxTile + pt];
        const double w1 = p[2 * kBoxTile + pt], h1 = p[3 * kBoxTile + pt], t1 = p[4 * kBoxTile + pt];
        const double w2 = p[7 * kBoxTile + pt], h2 = p[8 * kBoxTile + pt], t2 = p[9 * kBoxTile + pt];
        corner(0.0, 0.0, w1, h1, t1, i, vx, vy);
        corner(0.0, 0.0, w1, h1, t1, i1, v1x, v1y);
        corner(dcx, dcy, w2, h2, t2, j, wx, wy);
        corner(dcx, dcy, w2, h2, t2, j1, w1x, w1y);
    }
};

struct BoxBwdSmem {
    float x1[kBoxTile * 4], y1[kBoxTile * 4], x2[kBoxTile * 4], y2[kBoxTile * 4];  // corners, [pair][k]
    float bp[10 * kBoxTile];                                                     // BEV params, [param][pair]
    float scr[4 * 4 * kBoxTile];                                                 // [slot][pair]
    uint16_t queue[kBoxTile / 32][32 * 8];
    FlagLut lut;
};

// A thin pair of the box backward (rare): the intersection area in double from the
// corner tile, the gradients again — out of line, everything re-read, so its code
// does not enter the hot path's register allocation.
template <int DIMS>
__device__ __noinline__ void box_bwd_thin_redo(const float *__restrict__ b1, const float *__restrict__ b2,
                                               int64_t sk, int64_t sp, const float *__restrict__ grad,
                                               const uint8_t *__restrict__ nx, const uint8_t *__restrict__ xflags,
                                               float *__restrict__ gb1, float *__restrict__ gb2, int64_t k,
                                               BoxBwdSmem &S)
{
    const Box<DIMS> a = load_box<DIMS>(b1, k, sk, sp), b = load_box<DIMS>(b2, k, sk, sp);
    const ZOver z = z_overlap<DIMS>(a, b);
    Seq<4> s2;
    s2.w[0] = __ldcs(reinterpret_cast<const unsigned long long *>(xflags) + k);
    Poly<4> G1, G2;
    VolCoef co;
    bwd_thin_redo<4, kBoxTile>(S.x1, S.y1, S.x2, S.y2, s2, nx[k], __ldcs(grad + k), S.scr, S.lut, G1, G2,
                               Extrude{z.dz, a.d, b.d}, &co);
    Trig t;
    box_sincos(a.th, t.s1, t.c1);
    box_sincos(b.th, t.s2, t.c2);
    float gcz1, gd1, gcz2, gd2;
    z_grads<DIMS>(co, z, gcz1, gd1, gcz2, gd2);
    store_box_grad<DIMS>(gb1, k, sk, sp, box_vjp(a.w, a.h, t.c1, t.s1, G1), gcz1, gd1);
    store_box_grad<DIMS>(gb2, k, sk, sp, box_vjp(b.w, b.h, t.c2, t.s2, G2), gcz2, gd2);
}

template <int DIMS>
__global__ void __launch_bounds__(kBoxTile, DIMS == 2 ? DGAL_BOX_BWD2_MINB : DGAL_BOX_BWD3_MINB)
box_bwd_kernel(int64_t n, const float *__restrict__ b1, const float *__restrict__ b2, int64_t sk, int64_t sp,
               const float *__restrict__ grad, const uint8_t *__restrict__ nx, const uint8_t *__restrict__ xflags,
               float *__restrict__ gb1, float *__restrict__ gb2)
{
    __shared__ __align__(16) BoxBwdSmem S;
    const int tid = threadIdx.x;
    const int64_t k = (int64_t)blockIdx.x * kBoxTile + tid;
    const bool live = k < n;
    fill_flag_lut(S.lut, tid, kBoxTile);
    Box<DIMS> a{}, b{};
    Poly<4> P, Q;
    Trig t{1.f, 0.f, 1.f, 0.f};
    Seq<4> sq;
    sq.w[0] = 0ull;
    int m = 0;
    float g = 0.f;
    if (live) {
        a = load_box<DIMS>(b1, k, sk, sp);
        b = load_box<DIMS>(b2, k, sk, sp);
        t = box_pair_polys<DIMS>(a, b, P, Q);
        sq.w[0] = __ldcs(reinterpret_cast<const unsigned long long *>(xflags) + k);
        m = nx[k];
        g = __ldcs(grad + k);
    } else {
#pragma unroll
        for (int q = 0; q < 4; ++q) { P.x[q] = P.y[q] = Q.x[q] = Q.y[q] = 0.f; }
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        S.x1[tid * 4 + q] = P.x[q]; S.y1[tid * 4 + q] = P.y[q];
        S.x2[tid * 4 + q] = Q.x[q]; S.y2[tid * 4 + q] = Q.y[q];
    }
    const ZOver z = z_overlap<DIMS>(a, b);
    {
        const float bv[10] = {a.cx, a.cy, a.w, a.h, a.th, b.cx, b.cy, b.w, b.h, b.th};
#pragma unroll
        for (int q = 0; q < 10; ++q) S.bp[q * kBoxTile + tid] = bv[q];
    }
    __syncthreads();  // flag table, corner tile, parameters
    Poly<4> G1, G2;
    VolCoef co;
    const BoxGeometry geo{S.bp};
    const bool thin = bwd_tile_pair<4, kBoxTile, BoxGeometry>(S.x1, S.y1, S.x2, S.y2, sq, m, g, live, S.scr,
                                                              S.queue[tid >> 5], S.lut, G1, G2,
                                                              Extrude{z.dz, a.d, b.d}, &co, &geo);
    if (!live) return;
    float gcz1, gd1, gcz2, gd2;
    z_grads<DIMS>(co, z, gcz1, gd1, gcz2, gd2);
    store_box_grad<DIMS>(gb1, k, sk, sp, box_vjp(a.w, a.h, t.c1, t.s1, G1), gcz1, gd1);
    store_box_grad<DIMS>(gb2, k, sk, sp, box_vjp(b.w, b.h, t.c2, t.s2, G2), gcz2, gd2);
    if (thin) box_bwd_thin_redo<DIMS>(b1, b2, sk, sp, grad, nx, xflags, gb1, gb2, k, S);
}

// ---------------------------------------------------------------------------
// fused loss forward + backward (f2 on boxes): no nx / xflags round trip
// ---------------------------------------------------------------------------
template <int DIMS>
__global__ void __launch_bounds__(kBoxFusedT, DIMS == 2 ? DGAL_BOX_FUSED2_MINB : DGAL_BOX_FUSED3_MINB)
box_fused_kernel(int64_t n, const float *__restrict__ b1, const float *__restrict__ b2, int64_t sk, int64_t sp,
                 const float *__restrict__ grad, float scale, float *__restrict__ iou, float *__restrict__ gb1,
                 float *__restrict__ gb2, RefineQueue *__restrict__ refine)
{
    constexpr int T = kBoxFusedT;
    constexpr bool PF = DGAL_BOX_PF;
    constexpr int NT = PF ? DGAL_BOX_FUSED_NT : 1;
    __shared__ float pt[16 * T];   // per-thread piece table (kP2PiecesSmem), [slot][thread]
    __shared__ __align__(16) BoxRing<DIMS, PF ? T : 1> ring;   // tile t+1 in flight while tile t computes
    const int tid = threadIdx.x;
    const int64_t k0 = (int64_t)blockIdx.x * (NT * T) + tid;
    if (PF) {
        if (k0 < n) ring.prefetch(0, b1, b2, grad, k0, sk, sp, tid);
        cp_async_commit();
    }
#pragma unroll 1
    for (int it = 0; it < NT; ++it) {
        const int64_t k = k0 + (int64_t)it * T;
        if (k >= n) break;
        Box<DIMS> a, b;
        float g = scale;
        if (PF) {
            if (it + 1 < NT && k + T < n) ring.prefetch((it + 1) & 1, b1, b2, grad, k + T, sk, sp, tid);
            cp_async_commit();
            cp_async_wait<1>();   // this thread's copies of tile it have landed
            a = ring.get(it & 1, 0, tid);
            b = ring.get(it & 1, 1, tid);
            if (grad) g = ring.g[it & 1][tid];
        } else {
            a = load_box<DIMS>(b1, k, sk, sp);
            b = load_box<DIMS>(b2, k, sk, sp);
            if (grad) g = __ldcs(grad + k);
        }
        Poly<4> P, Q, G1, G2;
        const Trig t = box_pair_polys<DIMS>(a, b, P, Q);
        const ZOver z = z_overlap<DIMS>(a, b);
        VolCoef co;
        bool need;
        const float v = iou_fused<4, kP2PiecesSmem, DIMS == 2 && DGAL_BOX_FUSED_PK, 0>(
            P, Q, g, G1, G2, Extrude{z.dz, a.d, b.d}, &co, QTable{pt + tid, pt + 8 * T + tid, T}, &need,
            IllTab{nullptr, 0, BoxGeometry::kRefine});
        refine_mark(refine, k, need);   // redone exactly by box_fused_refine_kernel
        if (iou) __stcs(iou + k, v);
        float gcz1, gd1, gcz2, gd2;
        z_grads<DIMS>(co, z, gcz1, gd1, gcz2, gd2);
        store_box_grad<DIMS>(gb1, k, sk, sp, box_vjp(a.w, a.h, t.c1, t.s1, G1), gcz1, gd1);
        store_box_grad<DIMS>(gb2, k, sk, sp, box_vjp(b.w, b.h, t.c2, t.s2, G2), gcz2, gd2);
    }
}

// ---------------------------------------------------------------------------
// Refine pass of the fused box kernel (dgal_refine.cuh): the marked pairs redone
// with the split path's arithmetic — box_fwd's clip with flags (+ the thin-pair
// areas in double), then box_bwd's phases (crossings refined in double from the
// box parameters, BoxGeometry), the extrusion and box_to_polygon_grad.
// ---------------------------------------------------------------------------
static_assert(kRefT == kBoxTile, "the refine tile is the backward tile (BoxGeometry strides)");
struct BoxRefineSmem {
    BoxBwdSmem b;
};

template <int DIMS>
__global__ void __launch_bounds__(kRefT, 4)
box_fused_refine_kernel(int64_t n, const float *__restrict__ b1, const float *__restrict__ b2, int64_t sk,
                        int64_t sp, const float *__restrict__ grad, float scale, float *__restrict__ iou,
                        float *__restrict__ gb1, float *__restrict__ gb2, RefineQueue *__restrict__ refine)
{
    extern __shared__ __align__(16) unsigned char smem_raw[];
    BoxRefineSmem &R = *reinterpret_cast<BoxRefineSmem *>(smem_raw);
    BoxBwdSmem &S = R.b;
    const int tid = threadIdx.x;
    const unsigned int total = refine_count(refine);
    if ((unsigned int)blockIdx.x * kRefT < total) {
        fill_flag_lut(S.lut, tid, kRefT);
        __syncthreads();
    }
    {
#pragma unroll 1
        for (unsigned int base = blockIdx.x * kRefT; base < total; base += gridDim.x * kRefT) {
            const unsigned int e = base + tid;
            const bool live = e < total;
            const int64_t k = live ? (int64_t)refine->idx[e] : 0;
            Box<DIMS> a{}, b{};
            Poly<4> P, Q;
            Trig t{1.f, 0.f, 1.f, 0.f};
            if (live) {
                a = load_box<DIMS>(b1, k, sk, sp);
                b = load_box<DIMS>(b2, k, sk, sp);
                t = box_pair_polys<DIMS>(a, b, P, Q);
            } else {
#pragma unroll
                for (int q = 0; q < 4; ++q) { P.x[q] = P.y[q] = Q.x[q] = Q.y[q] = 0.f; }
            }
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                S.x1[tid * 4 + q] = P.x[q]; S.y1[tid * 4 + q] = P.y[q];
                S.x2[tid * 4 + q] = Q.x[q]; S.y2[tid * 4 + q] = Q.y[q];
            }
            {
                const float bv[10] = {a.cx, a.cy, a.w, a.h, a.th, b.cx, b.cy, b.w, b.h, b.th};
#pragma unroll
                for (int q = 0; q < 10; ++q) S.bp[q * kBoxTile + tid] = bv[q];
            }
            const ZOver z = z_overlap<DIMS>(a, b);
            FwdOut<4, true> r = iou_fwd<4, true, kP2Regs, true>(P, Q);
            float A1x2 = r.A1x2, A2x2 = r.A2x2, Aix2 = r.Aix2;
            if (r.thin) {
                AreasX2 e;
                fwd_thin_redo<4>(BoxCornersD(a, b), r.seq, r.nx, r.iou, &e);
                A1x2 = (float)e.a1; A2x2 = (float)e.a2; Aix2 = (float)e.ai;
            }
            int m = r.nx;
            float v = r.iou;
            if (DIMS == 3) {
                const float Vix2 = Aix2 * z.dz;
                const float Vux2 = (A1x2 * a.d + A2x2 * b.d) - Vix2;
                const bool ok = m > 0 && Vix2 > 0.f && Vux2 > 0.f;
                v = ok ? iou_div(Vix2, Vux2) : 0.f;
                m = ok ? m : 0;
            }
            if (live && iou) iou[k] = v;
            const float g = live ? (grad ? grad[k] : scale) : 0.f;
            __syncwarp();   // the warp's tile is staged
            Poly<4> G1, G2;
            VolCoef co;
            const BoxGeometry geo{S.bp};
            const bool thin = bwd_tile_pair<4, kBoxTile, BoxGeometry>(S.x1, S.y1, S.x2, S.y2, r.seq, live ? m : 0, g,
                                                                      live, S.scr, S.queue[tid >> 5], S.lut, G1, G2,
                                                                      Extrude{z.dz, a.d, b.d}, &co, &geo);
            if (thin)
                bwd_thin_redo<4, kBoxTile>(S.x1, S.y1, S.x2, S.y2, r.seq, m, g, S.scr, S.lut, G1, G2,
                                           Extrude{z.dz, a.d, b.d}, &co);
            if (live) {
                float gcz1, gd1, gcz2, gd2;
                z_grads<DIMS>(co, z, gcz1, gd1, gcz2, gd2);
                store_box_grad<DIMS>(gb1, k, sk, sp, box_vjp(a.w, a.h, t.c1, t.s1, G1), gcz1, gd1);
                store_box_grad<DIMS>(gb2, k, sk, sp, box_vjp(b.w, b.h, t.c2, t.s2, G2), gcz2, gd2);
            }
            __syncwarp();
        }
    }
    __syncthreads();
    if (tid == 0) refine_finish(refine);
}

// ---------------------------------------------------------------------------
// launchers
// ---------------------------------------------------------------------------
namespace {
inline void box_strides(int dims, int layout, int64_t n, int64_t &sk, int64_t &sp)
{
    const int P = dims == 3 ? 7 : 5;
    if (layout == 0) { sk = 1; sp = n; }   // planes [P][n]
    else { sk = P; sp = 1; }               // rows [n][P]
}
}  // namespace

cudaError_t launch_box_fwd(int dims, int layout, int64_t n, const float *b1, const float *b2, float *iou,
                           uint8_t *nx, uint8_t *xflags, cudaStream_t st)
{
    int64_t sk, sp;
    box_strides(dims, layout, n, sk, sp);
    const unsigned grid = (unsigned)((n + kBoxFwdNT * kBoxFwdT - 1) / (kBoxFwdNT * kBoxFwdT));
    if (dims == 3)
        box_fwd_kernel<3><<<grid, kBoxFwdT, 0, st>>>(n, b1, b2, sk, sp, iou, nx, xflags);
    else
        box_fwd_kernel<2><<<grid, kBoxFwdT, 0, st>>>(n, b1, b2, sk, sp, iou, nx, xflags);
    return cudaGetLastError();
}

cudaError_t launch_box_bwd(int dims, int layout, int64_t n, const float *b1, const float *b2, const float *grad,
                           const uint8_t *nx, const uint8_t *xflags, float *gb1, float *gb2, cudaStream_t st)
{
    int64_t sk, sp;
    box_strides(dims, layout, n, sk, sp);
    const unsigned grid = (unsigned)((n + kBoxTile - 1) / kBoxTile);
    if (dims == 3)
        box_bwd_kernel<3><<<grid, kBoxTile, 0, st>>>(n, b1, b2, sk, sp, grad, nx, xflags, gb1, gb2);
    else
        box_bwd_kernel<2><<<grid, kBoxTile, 0, st>>>(n, b1, b2, sk, sp, grad, nx, xflags, gb1, gb2);
    return cudaGetLastError();
}

cudaError_t launch_box_fused(int dims, int layout, int64_t n, const float *b1, const float *b2, const float *grad,
                             float scale, float *iou, float *gb1, float *gb2, void *refine_ws, cudaStream_t st)
{
    RefineQueue *refine = static_cast<RefineQueue *>(refine_ws);
    int64_t sk, sp;
    box_strides(dims, layout, n, sk, sp);
    constexpr int64_t per = (int64_t)(DGAL_BOX_PF ? DGAL_BOX_FUSED_NT : 1) * kBoxFusedT;
    const unsigned grid = (unsigned)((n + per - 1) / per);
    static DeviceCache c2, c3;
    const int a = (dims == 3 ? c3 : c2).get([&](int) {
        return dims == 3 ? set_smem_attr(box_fused_refine_kernel<3>, sizeof(BoxRefineSmem))
                         : set_smem_attr(box_fused_refine_kernel<2>, sizeof(BoxRefineSmem));
    });
    if (a <= 0) return (cudaError_t)(-a);
    const unsigned rg = (unsigned)refine_grid_for(n);
    if (dims == 3) {
        box_fused_kernel<3><<<grid, kBoxFusedT, 0, st>>>(n, b1, b2, sk, sp, grad, scale, iou, gb1, gb2, refine);
        box_fused_refine_kernel<3><<<rg, kRefT, sizeof(BoxRefineSmem), st>>>(n, b1, b2, sk, sp, grad, scale, iou,
                                                                            gb1, gb2, refine);
    } else {
        box_fused_kernel<2><<<grid, kBoxFusedT, 0, st>>>(n, b1, b2, sk, sp, grad, scale, iou, gb1, gb2, refine);
        box_fused_refine_kernel<2><<<rg, kRefT, sizeof(BoxRefineSmem), st>>>(n, b1, b2, sk, sp, grad, scale, iou,
                                                                            gb1, gb2, refine);
    }
    return cudaGetLastError();
}

}  // namespace dgal
