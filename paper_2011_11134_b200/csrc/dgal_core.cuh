// dgal_core.cuh — register-resident device primitives for batched convex-polygon
// IoU (DGAL, arXiv 2011.11134) on sm_100a.  Everything here is __device__ and
// fully unrolled over the compile-time vertex count K ("templated
// with options for precision and size ... fix-size allocated memory"), so no
// array is ever dynamically indexed and nothing spills to local memory
// (checked by tests/test_build_artifacts.py on the SASS).
//
// Method.  The paper's `intersect(p1, p2, xflags)` is
// realised as an edge-interval clip: every edge of p1 is clipped against the
// closed half-planes of p2 and every edge of p2 against the open half-planes of
// p1 (Cyrus-Beck intervals [t0, t1] on each edge).  In exact arithmetic these
// intervals are exactly the boundary pieces of p1 ∩ p2, so
//   * area:  2 A_i = sum_i (t1-t0)_i cross(v_i, v_i+1) + sum_j (s1-s0)_j cross(w_j, w_j+1)
//     (Green's theorem on each boundary piece, no vertex list needed),
//   * nx / xflags: walking p1's edges in order emits FromP1(i) or the
//     entering Cross(i, j_in), then the exiting Cross(i, j_out) followed by the
//     run of p2 vertices strictly inside p1 — the CCW vertex sequence of p1 ∩ p2,
//     rotated to start at its smallest byte (R3),
//   * iou_grad: d A_i / d v moves only the boundary pieces lying on the
//     edges incident to v (shape derivative), so with n_i = perp(v_i+1 - v_i):
//       dA_i/dv_i += n_i ∫_{t0}^{t1} (1-t) dt,   dA_i/dv_i+1 += n_i ∫_{t0}^{t1} t dt,
//     where the interval end points are read from the recorded xflags.
// Decision predicates (inside/outside) are evaluated contraction-free
// (__fmul_rn/__fsub_rn) so a point exactly on a line gives exactly 0: identical
// polygons give IoU == 1 exactly (the pairwise diagonal).
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace dgal {

template <int K>
struct Poly {
    float x[K];
    float y[K];
};

// ---------------------------------------------------------------------------
// small helpers
// ---------------------------------------------------------------------------
__device__ __forceinline__ float cross_rn(float ax, float ay, float bx, float by)
{
    // a x b with both products rounded separately: exact 0 for parallel
    // bitwise-equal operands (used for every inside/outside decision).
    return __fsub_rn(__fmul_rn(ax, by), __fmul_rn(ay, bx));
}

__device__ __forceinline__ float rcp_approx(float x)
{
    float r;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}

template <int K>
__device__ __forceinline__ float pick(const float (&a)[K], int i)
{
    float r = a[0];
#pragma unroll
    for (int k = 1; k < K; ++k) r = (i == k) ? a[k] : r;
    return r;
}

// Streaming loads/stores of the SoA planes.
template <int K>
__device__ __forceinline__ void load_poly(const float *__restrict__ X, const float *__restrict__ Y,
                                          int64_t n, Poly<K> &p)
{
    const float4 *x4 = reinterpret_cast<const float4 *>(X + n * K);
    const float4 *y4 = reinterpret_cast<const float4 *>(Y + n * K);
#pragma unroll
    for (int q = 0; q < K / 4; ++q) {
        float4 a = __ldcs(x4 + q), b = __ldcs(y4 + q);
        p.x[4 * q + 0] = a.x; p.x[4 * q + 1] = a.y; p.x[4 * q + 2] = a.z; p.x[4 * q + 3] = a.w;
        p.y[4 * q + 0] = b.x; p.y[4 * q + 1] = b.y; p.y[4 * q + 2] = b.z; p.y[4 * q + 3] = b.w;
    }
}

template <int K>
__device__ __forceinline__ void store_plane(float *__restrict__ X, int64_t n, const float (&v)[K])
{
    float4 *x4 = reinterpret_cast<float4 *>(X + n * K);
#pragma unroll
    for (int q = 0; q < K / 4; ++q)
        __stcs(x4 + q, make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]));
}

// ---------------------------------------------------------------------------
// flag-byte sequence: 2K bytes in K/4 64-bit words (R2: padding 0x00)
// ---------------------------------------------------------------------------
template <int K>
struct Seq {
    static constexpr int NW = K / 4;  // 64-bit words
    uint64_t w[NW];
};

// OR the (<= 8 byte) value r into the byte string at byte offset pos.
template <int K>
__device__ __forceinline__ void seq_or(Seq<K> &s, uint64_t r, int pos)
{
#pragma unroll
    for (int k = 0; k < Seq<K>::NW; ++k) {
        const int sh = 8 * pos - 64 * k;  // bit offset of r inside word k
        uint64_t part = 0;
        if (sh >= 0 && sh < 64) part = r << sh;
        else if (sh < 0 && sh > -64) part = r >> (-sh);
        s.w[k] |= part;
    }
}

template <int K>
__device__ __forceinline__ uint32_t seq_byte(const Seq<K> &s, int p)
{
    // select the word without a dynamic array index (keeps s in registers)
    uint64_t w = s.w[0];
#pragma unroll
    for (int k = 1; k < Seq<K>::NW; ++k) w = ((p >> 3) == k) ? s.w[k] : w;
    return (uint32_t)(w >> (8 * (p & 7))) & 0xFFu;
}

// Rotate the first n bytes of s left by r bytes (byte r becomes byte 0).
template <int K>
__device__ __forceinline__ Seq<K> seq_rotate(const Seq<K> &s, int n, int r)
{
    Seq<K> o;
#pragma unroll
    for (int k = 0; k < Seq<K>::NW; ++k) o.w[k] = 0;
    if (K == 4) {
        // one word: bytes [r, n) then [0, r)
        const uint64_t x = s.w[0];
        const uint64_t lo = (r > 0) ? (x >> (8 * r)) : x;
        const uint64_t hi = (r > 0) ? (x << (8 * (n - r))) : 0;
        uint64_t m = (n >= 8) ? ~0ull : ((1ull << (8 * n)) - 1ull);
        o.w[0] = (lo | hi) & m;
    } else {
#pragma unroll
        for (int p = 0; p < 2 * K; ++p) {
            if (p < n) {
                int q = p + r;
                q = (q >= n) ? q - n : q;
                const uint64_t b = seq_byte<K>(s, q);
                o.w[p >> 3] |= b << (8 * (p & 7));
            }
        }
    }
    return o;
}

// ---------------------------------------------------------------------------
// forward: intersect + area + IoU
// ---------------------------------------------------------------------------
template <int K, bool FLAGS>
struct FwdOut {
    float iou;
    int nx;
    Seq<K> seq;
};

// p1, p2 must already be recentred on o = p1.v0 (p1.x[0] == p1.y[0] == 0).
template <int K, bool FLAGS>
__device__ __forceinline__ FwdOut<K, FLAGS> iou_fwd(const Poly<K> &P, const Poly<K> &Q)
{
    constexpr uint32_t KMASK = (1u << K) - 1u;

    // edge vectors g_i = v_i+1 - v_i (p1), f_j = w_j+1 - w_j (p2)
    float gx[K], gy[K], fx[K], fy[K];
#pragma unroll
    for (int i = 0; i < K; ++i) {
        const int i1 = (i + 1) % K;
        gx[i] = P.x[i1] - P.x[i]; gy[i] = P.y[i1] - P.y[i];
        fx[i] = Q.x[i1] - Q.x[i]; fy[i] = Q.y[i1] - Q.y[i];
    }
    // shoelace terms: C1_i = v_i x v_i+1, C2_j = w_j x w_j+1
    float C1[K], C2[K];
    float A1x2 = 0.f, A2x2 = 0.f;
#pragma unroll
    for (int i = 0; i < K; ++i) {
        const int i1 = (i + 1) % K;
        C1[i] = P.x[i] * P.y[i1] - P.x[i1] * P.y[i];
        C2[i] = Q.x[i] * Q.y[i1] - Q.x[i1] * Q.y[i];
        // same order as the A_i sum below: identical polygons give A_i == A_1 bitwise
        A1x2 = __fadd_rn(A1x2, C1[i]);
        A2x2 = __fadd_rn(A2x2, C2[i]);
    }

    // ---- p1 edges against the CLOSED half-planes of p2 (inside: d >= 0) ----
    // d[i][j] = f_j x (v_i - w_j), computed one vertex row at a time.
    float drow0[K], dprev[K];
    float satP2[K];  // max_i d[i][j]: <= 0 means p1 lies outside line j (separating)
#pragma unroll
    for (int j = 0; j < K; ++j) {
        drow0[j] = cross_rn(fx[j], fy[j], __fsub_rn(P.x[0], Q.x[j]), __fsub_rn(P.y[0], Q.y[j]));
        dprev[j] = drow0[j];
        satP2[j] = drow0[j];
    }
    float Aix2 = 0.f;
    uint32_t valid1 = 0;
    int jin[K], jout[K];
#pragma unroll
    for (int i = 0; i < K; ++i) {
        float dnext[K];
#pragma unroll
        for (int j = 0; j < K; ++j) {
            if (i + 1 < K) {
                dnext[j] = cross_rn(fx[j], fy[j], __fsub_rn(P.x[i + 1], Q.x[j]),
                                    __fsub_rn(P.y[i + 1], Q.y[j]));
                satP2[j] = fmaxf(satP2[j], dnext[j]);
            } else {
                dnext[j] = drow0[j];
            }
        }
        float t0 = 0.f, t1 = 1.f;
        bool dead = false;
        int ji = -1, jo = -1;
#pragma unroll
        for (int j = 0; j < K; ++j) {
            const float a = dprev[j], b = dnext[j];
            const bool oa = a < 0.f, ob = b < 0.f;
            dead |= oa & ob;
            const float t = a * rcp_approx(a - b);
            if (oa & !ob & (t > t0)) { t0 = t; if (FLAGS) ji = j; }
            if (ob & !oa & (t < t1)) { t1 = t; if (FLAGS) jo = j; }
        }
        const bool v = !dead && (t0 < t1);
        valid1 |= (uint32_t)v << i;
        Aix2 = fmaf(v ? (t1 - t0) : 0.f, C1[i], Aix2);
        jin[i] = ji;
        jout[i] = jo;
#pragma unroll
        for (int j = 0; j < K; ++j) dprev[j] = dnext[j];
    }

    // ---- p2 edges against the OPEN half-planes of p1 (inside: e > 0) ----
    // e[j][i] = g_i x (w_j - v_i) = (v_i - w_j) x g_i
    float erow0[K], eprev[K];
    float satP1[K];  // max_j e[j][i] <= 0: p2 lies outside line i
#pragma unroll
    for (int i = 0; i < K; ++i) {
        erow0[i] = cross_rn(__fsub_rn(P.x[i], Q.x[0]), __fsub_rn(P.y[i], Q.y[0]), gx[i], gy[i]);
        eprev[i] = erow0[i];
        satP1[i] = erow0[i];
    }
    uint32_t in2 = 0;  // bit j: w_j strictly inside p1
#pragma unroll
    for (int j = 0; j < K; ++j) {
        float enext[K];
        bool allin = true;
#pragma unroll
        for (int i = 0; i < K; ++i) {
            allin &= eprev[i] > 0.f;
            if (j + 1 < K) {
                enext[i] = cross_rn(__fsub_rn(P.x[i], Q.x[j + 1]), __fsub_rn(P.y[i], Q.y[j + 1]),
                                    gx[i], gy[i]);
                satP1[i] = fmaxf(satP1[i], enext[i]);
            } else {
                enext[i] = erow0[i];
            }
        }
        in2 |= (uint32_t)allin << j;
        float s0 = 0.f, s1 = 1.f;
        bool dead = false;
#pragma unroll
        for (int i = 0; i < K; ++i) {
            const float a = eprev[i], b = enext[i];
            const bool oa = a <= 0.f, ob = b <= 0.f;
            dead |= oa & ob;
            const float t = a * rcp_approx(a - b);
            if (oa & !ob) s0 = fmaxf(s0, t);
            if (ob & !oa) s1 = fminf(s1, t);
        }
        const bool v = !dead && (s0 < s1);
        Aix2 = fmaf(v ? (s1 - s0) : 0.f, C2[j], Aix2);
#pragma unroll
        for (int i = 0; i < K; ++i) eprev[i] = enext[i];
    }

    // Separating axis (closed): some edge line of either polygon has the other
    // polygon entirely on or outside it -> the intersection has zero area.  This
    // is what makes collinear, opposite-facing edges (touching boxes) empty.
    bool separated = false;
#pragma unroll
    for (int k = 0; k < K; ++k) separated |= (satP2[k] <= 0.f) | (satP1[k] <= 0.f);

    FwdOut<K, FLAGS> out;
#pragma unroll
    for (int k = 0; k < Seq<K>::NW; ++k) out.seq.w[k] = 0;
    out.nx = 0;
    out.iou = 0.f;
    Aix2 = fminf(Aix2, fminf(A1x2, A2x2));
    bool nonempty = !separated && (Aix2 > 0.f);

    if (FLAGS) {
        // Emit the CCW vertex sequence by walking p1's edges in order.
        Seq<K> s;
#pragma unroll
        for (int k = 0; k < Seq<K>::NW; ++k) s.w[k] = 0;
        int cnt = 0;
        uint32_t minb = 0x100u;
        int minpos = 0;
#pragma unroll
        for (int i = 0; i < K; ++i) {
            if ((valid1 >> i) & 1u) {
                const uint32_t b0 = (jin[i] < 0) ? (0x40u | i) : (0xC0u | (i << 3) | (uint32_t)jin[i]);
                if (cnt < 2 * K) seq_or<K>(s, b0, cnt);
                if (b0 < minb) { minb = b0; minpos = cnt; }
                ++cnt;
                if (jout[i] >= 0) {
                    const uint32_t b1 = 0xC0u | (i << 3) | (uint32_t)jout[i];
                    if (cnt < 2 * K) seq_or<K>(s, b1, cnt);
                    if (b1 < minb) { minb = b1; minpos = cnt; }
                    ++cnt;
                    // run of p2 vertices strictly inside p1 following p2 edge jout
                    const int p0 = (jout[i] + 1) % K;
                    const uint32_t rot = ((in2 >> p0) | (in2 << (K - p0))) & KMASK;
                    const int L = __ffs(~rot) - 1;  // trailing ones, <= K
                    if (L > 0) {
                        uint64_t run;
                        if (K == 4) {
                            const uint32_t pat = __funnelshift_r(0x83828180u, 0x83828180u, 8 * p0);
                            run = (uint64_t)(L >= 4 ? pat : (pat & ((1u << (8 * L)) - 1u)));
                        } else {
                            const uint64_t pat = 0x8786858483828180ull;
                            const uint64_t r8 = p0 ? ((pat >> (8 * p0)) | (pat << (64 - 8 * p0))) : pat;
                            run = (L >= 8) ? r8 : (r8 & ((1ull << (8 * L)) - 1ull));
                        }
                        if (cnt < 2 * K) seq_or<K>(s, run, cnt);
                        const bool wraps = p0 + L > K;
                        const uint32_t rb = wraps ? 0x80u : (0x80u | p0);
                        if (rb < minb) { minb = rb; minpos = cnt + (wraps ? K - p0 : 0); }
                        cnt += L;
                    }
                }
            }
        }
        if (cnt == 0 && in2 == KMASK) {  // p2 inside p1: all FromP2 (p1's edges never on the boundary)
            if (K == 4) s.w[0] = 0x83828180ull;
            else { s.w[0] = 0x8786858483828180ull; s.w[1] = 0; }
            cnt = K;
            minpos = 0;
        }
        nonempty = nonempty && cnt >= 3 && cnt <= 2 * K;
        if (nonempty) {
            out.seq = seq_rotate<K>(s, cnt, minpos);
            out.nx = cnt;
        }
    }
    if (nonempty) {
        const float Aux2 = (A1x2 + A2x2) - Aix2;
        out.iou = (Aux2 > 0.f) ? fminf(Aix2 / Aux2, 1.f) : 0.f;
    }
    return out;
}

// ---------------------------------------------------------------------------
// backward: iou_grad through the recorded nx / xflags
// ---------------------------------------------------------------------------
// Returns dL/dv for p1 and p2 (recentred coordinates; the gradient is the same
// in the original frame because IoU is translation invariant, R11).
template <int K>
__device__ __forceinline__ void iou_bwd(const Poly<K> &P, const Poly<K> &Q, float g, int nx,
                                        const Seq<K> &seq, Poly<K> &G1, Poly<K> &G2)
{
#pragma unroll
    for (int k = 0; k < K; ++k) { G1.x[k] = 0.f; G1.y[k] = 0.f; G2.x[k] = 0.f; G2.y[k] = 0.f; }
    if (nx == 0) return;

    float gx[K], gy[K], fx[K], fy[K], C1[K], C2[K];
    float A1x2 = 0.f, A2x2 = 0.f;
#pragma unroll
    for (int i = 0; i < K; ++i) {
        const int i1 = (i + 1) % K;
        gx[i] = P.x[i1] - P.x[i]; gy[i] = P.y[i1] - P.y[i];
        fx[i] = Q.x[i1] - Q.x[i]; fy[i] = Q.y[i1] - Q.y[i];
        C1[i] = P.x[i] * P.y[i1] - P.x[i1] * P.y[i];
        C2[i] = Q.x[i] * Q.y[i1] - Q.x[i1] * Q.y[i];
        A1x2 += C1[i];
        A2x2 += C2[i];
    }

    // Which original vertices are vertices of p1 ∩ p2 (SWAR exact zero-byte test
    // on the 2K flag bytes).
    uint32_t m1 = 0, m2 = 0;
#pragma unroll
    for (int k = 0; k < K; ++k) {
        bool h1 = false, h2 = false;
#pragma unroll
        for (int w = 0; w < Seq<K>::NW; ++w) {
            const uint64_t x1 = seq.w[w] ^ (0x4040404040404040ull | (0x0101010101010101ull * k));
            const uint64_t x2 = seq.w[w] ^ (0x8080808080808080ull | (0x0101010101010101ull * k));
            h1 |= (((x1 - 0x0101010101010101ull) & ~x1 & 0x8080808080808080ull) != 0);
            h2 |= (((x2 - 0x0101010101010101ull) & ~x2 & 0x8080808080808080ull) != 0);
        }
        m1 |= (uint32_t)h1 << k;
        m2 |= (uint32_t)h2 << k;
    }

    // Crossing vertices Cross(i, j): bytes whose two tag bits are both set.
    // X = v_i + t g_i = w_j + s f_j.  P1 edge i ENTERS p2 there iff g_i x f_j < 0;
    // then the boundary piece on edge i starts at t and the piece on p2 edge j
    // ends at s, otherwise the other way round.
    float t0[K], t1[K], s0[K], s1[K];
#pragma unroll
    for (int k = 0; k < K; ++k) { t0[k] = 0.f; t1[k] = 1.f; s0[k] = 0.f; s1[k] = 1.f; }
    uint32_t hc1 = 0, hc2 = 0;
#pragma unroll
    for (int w = 0; w < Seq<K>::NW; ++w) {
        const uint64_t word = seq.w[w];
        uint64_t c3 = word & (word << 1) & 0x8080808080808080ull;
        while (c3) {
            const int pos = __ffsll((long long)c3) - 1;  // bit 7 of the byte
            c3 &= c3 - 1;
            const uint32_t b = (uint32_t)(word >> (pos - 7)) & 0xFFu;
            const int i = (b >> 3) & 7, j = b & 7;
            const float vx = pick<K>(P.x, i), vy = pick<K>(P.y, i);
            const float ex = pick<K>(gx, i), ey = pick<K>(gy, i);
            const float wx = pick<K>(Q.x, j), wy = pick<K>(Q.y, j);
            const float hx = pick<K>(fx, j), hy = pick<K>(fy, j);
            const float Dx = wx - vx, Dy = wy - vy;
            const float den = ex * hy - ey * hx;         // g_i x f_j
            const float r = 1.f / den;
            const float t = (Dx * hy - Dy * hx) * r;     // along p1 edge i
            const float s = (Dx * ey - Dy * ex) * r;     // along p2 edge j
            const bool enter = den < 0.f;                // f_j x g_i > 0: d rises along g_i
#pragma unroll
            for (int k = 0; k < K; ++k) {
                if (k == i) { if (enter) t0[k] = t; else t1[k] = t; }
                if (k == j) { if (enter) s1[k] = s; else s0[k] = s; }
            }
            hc1 |= 1u << i;
            hc2 |= 1u << j;
        }
    }

    // Boundary intervals -> A_i and the per-edge weights
    //   alpha = ∫ (1-t) dt = (t1-t0)(1 - (t0+t1)/2),  beta = ∫ t dt = (t1-t0)(t0+t1)/2.
    float al1[K], be1[K], al2[K], be2[K];
    float Aix2 = 0.f;
#pragma unroll
    for (int i = 0; i < K; ++i) {
        const int i1 = (i + 1) % K;
        const bool on1 = ((m1 >> i) & 1u) | ((m1 >> i1) & 1u) | ((hc1 >> i) & 1u);
        const bool on2 = ((m2 >> i) & 1u) | ((m2 >> i1) & 1u) | ((hc2 >> i) & 1u);
        const float a0 = fminf(fmaxf(t0[i], 0.f), 1.f), a1 = fminf(fmaxf(t1[i], 0.f), 1.f);
        const float b0 = fminf(fmaxf(s0[i], 0.f), 1.f), b1 = fminf(fmaxf(s1[i], 0.f), 1.f);
        const float l1 = on1 ? fmaxf(a1 - a0, 0.f) : 0.f;
        const float l2 = on2 ? fmaxf(b1 - b0, 0.f) : 0.f;
        const float h1 = 0.5f * (a0 + a1), h2 = 0.5f * (b0 + b1);
        al1[i] = l1 * (1.f - h1); be1[i] = l1 * h1;
        al2[i] = l2 * (1.f - h2); be2[i] = l2 * h2;
        Aix2 = fmaf(l1, C1[i], Aix2);
        Aix2 = fmaf(l2, C2[i], Aix2);
    }

    // dIoU/dA_i = (A_u + A_i)/A_u^2, dIoU/dA_1,2 = -A_i/A_u^2
    const float Ai = 0.5f * Aix2;
    const float Au = 0.5f * ((A1x2 + A2x2) - Aix2);
    if (!(Au > 0.f) || !(Ai > 0.f)) return;  // R10 guard
    const float inv = 1.f / Au;
    const float q = Ai * inv;
    const float ci = g * ((1.f + q) * inv);
    const float cu = g * (-q * inv);
    const float hu = 0.5f * cu;  // area_grad of p1/p2 is (n_k + n_k-1)/2 per vertex

    // vertex k collects edge k (as its start, alpha) and edge k-1 (as its end, beta);
    // n = perp(edge) = (e_y, -e_x)
#pragma unroll
    for (int k = 0; k < K; ++k) {
        const int km = (k + K - 1) % K;
        const float wa1 = fmaf(ci, al1[k], hu), wb1 = fmaf(ci, be1[km], hu);
        const float wa2 = fmaf(ci, al2[k], hu), wb2 = fmaf(ci, be2[km], hu);
        G1.x[k] = fmaf(wa1, gy[k], wb1 * gy[km]);
        G1.y[k] = -fmaf(wa1, gx[k], wb1 * gx[km]);
        G2.x[k] = fmaf(wa2, fy[k], wb2 * fy[km]);
        G2.y[k] = -fmaf(wa2, fx[k], wb2 * fx[km]);
    }
}

}  // namespace dgal
