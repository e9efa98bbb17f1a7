// dgal_core.cuh — register-resident device primitives for batched convex-polygon
// IoU (DGAL, arXiv 2011.11134) on sm_100a.  Everything here is __device__ and
// fully unrolled over the compile-time vertex count K ("templated
// with options for precision and size ... fix-size allocated memory"), so no
// array is ever dynamically indexed and nothing spills to local memory
// (checked on the SASS by tests/test_abi_cpu.py::test_sass_is_sm100a_register_resident).
//
// Method.  The paper's `intersect(p1, p2, xflags)` is
// realised as an edge-interval clip: every edge of p1 is clipped against the
// closed half-planes of p2 and every edge of p2 against the open half-planes of
// p1 (Cyrus-Beck intervals [t0, t1] on each edge).  In exact arithmetic these
// intervals are exactly the boundary pieces of p1 ∩ p2, so
//   * area:  2 A_i = sum_i (t1-t0)_i v_i x v_i+1 + sum_j (s1-s0)_j w_j x w_j+1
//     (Green's theorem on each boundary piece, no vertex list needed);
//   * nx / xflags: walking p1's edges in order emits FromP1(i) or
//     the entering Cross(i, j_in), then the exiting Cross(i, j_out) followed by
//     the run of p2 vertices strictly inside p1 — the CCW vertex sequence of
//     p1 ∩ p2, which starts at the first vertex along p1's boundary from v0:
//     exactly the canonical order of reading R3;
//   * iou_grad: dA_i/dv moves only the boundary pieces lying on the edges
//     incident to v (shape derivative); with n = perp(edge vector),
//       dA_i/dv_i += n_i ∫_{t0}^{t1} (1-t) dt,   dA_i/dv_i+1 += n_i ∫_{t0}^{t1} t dt,
//     where the interval end points come from the crossings recorded in xflags.
//
// Performance notes (sm_100a, ncu-guided): the kernels are
// instruction-bound with the ALU pipe (compare/select/min/max/logic, half rate)
// the binding unit, so the Cyrus-Beck update is written branch-free with the
// class of each line taken from sign(a - b) alone: an FMA-pipe saturating
// multiply turns it into a 0/1 mask, leaving two min/max per (edge, line) on the
// ALU pipe.  The line index that defines t0 / t1 (needed for the flags) rides in
// the three low mantissa bits of t (<= 7 ulp, below the IoU tolerance).
// Decision predicates are contraction-free (__fmul_rn/__fsub_rn) so a point on
// a line gives exactly 0: identical polygons give IoU == 1 exactly.
#pragma once

#include <cassert>
#include <cstdint>
#include <cuda_runtime.h>

#ifndef DGAL_ASSERT
#ifdef DGAL_CHECKED
#define DGAL_ASSERT(x) assert(x)
#else
#define DGAL_ASSERT(x) ((void)0)
#endif
#endif

namespace dgal {

template <int K>
struct Poly {
    float x[K];
    float y[K];
};

// ---------------------------------------------------------------------------
// small helpers
// ---------------------------------------------------------------------------
constexpr float kTiny = 1e-30f;   // below any non-degenerate decision value
constexpr float kBig = 1e30f;

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

// IoU = a / u (0 < a <= u) as a * rcp.approx(u) (<= 1 ulp reciprocal: the quotient
// within ~2 ulp, as div.full, without its range-scaling checks: u is a normal float
// here — twice an area of polygons whose Green sums do not overflow), clamped to 1;
// a == u (identical polygons) gives 1 exactly.  The one IoU division of every kernel
// (paired, fused, pairwise agree bitwise).
__device__ __forceinline__ float iou_div(float a, float u)
{
    const float q = a * rcp_approx(u);
    return (a == u) ? 1.f : fminf(q, 1.f);
}

// 1/x to ~1 ulp without the IEEE division's slow-path branch (x normal, > 0 here):
// the approximate reciprocal and one Newton step
__device__ __forceinline__ float rcp_refined(float x)
{
    const float r = rcp_approx(x);
    return fmaf(r, fmaf(-x, r, 1.f), r);
}

// Paired FP32 (sm_100: FADD2 / FMUL2 / FFMA2 — two IEEE RN operations in one
// instruction on a 64-bit register pair; no contraction across the asm).  The
// kernels are issue-bound, so pairing the decision values and the Cyrus-Beck
// candidates of two p2 lines halves their FMA-pipe instruction count with
// bitwise the same results.
#ifndef DGAL_F32X2
#define DGAL_F32X2 7   // bit 0: decision rows, bit 1: Cyrus-Beck candidates, bit 2: backward epilogue (PK callers)
#endif
__device__ __forceinline__ uint64_t f2pack(float lo, float hi)
{
    uint64_t r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
    return r;
}
__device__ __forceinline__ void f2unpack(uint64_t v, float &lo, float &hi)
{
    asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(v));
}
__device__ __forceinline__ uint64_t f2add(uint64_t a, uint64_t b)
{
    uint64_t r;
    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
    return r;
}
__device__ __forceinline__ uint64_t f2sub(uint64_t a, uint64_t b)
{
    uint64_t r;
    asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
    return r;
}
__device__ __forceinline__ uint64_t f2mul(uint64_t a, uint64_t b)
{
    uint64_t r;
    asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
    return r;
}
__device__ __forceinline__ uint64_t f2fma(uint64_t a, uint64_t b, uint64_t c)
{
    uint64_t r;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
    return r;
}
// a * b rounded, as a product ptxas cannot contract into a following add: it
// fuses mul.rn.f32x2 + sub.rn.f32x2 into FFMA2 despite the rounding modifiers
// (measured: 26 % of decision values 1 ulp off).  fma(a, b, +0) is the rounded
// product (up to the sign of a zero, which the + tiny of every use absorbs).
__device__ __forceinline__ uint64_t f2mul_nc(uint64_t a, uint64_t b) { return f2fma(a, b, 0ull); }

// carry a line index 0..7 in the 3 low mantissa bits of a finite value:
// one LOP3 (v & ~7) | j with j in a register
__device__ __forceinline__ float enc_idx(float v, int j)
{
    uint32_t r;
    asm("lop3.b32 %0, %1, %2, %3, 0xEA;" : "=r"(r) : "r"(__float_as_uint(v)), "n"(0xFFFFFFF8), "r"(j));
    return __uint_as_float(r);
}
__device__ __forceinline__ int dec_idx(float v) { return __float_as_int(v) & 7; }

// 64-bit shifts with PTX semantics (amounts >= 64 give 0), no C++ UB
__device__ __forceinline__ uint64_t shl64(uint64_t x, uint32_t s)
{
    uint64_t r;
    asm("shl.b64 %0, %1, %2;" : "=l"(r) : "l"(x), "r"(s));
    return r;
}
__device__ __forceinline__ uint64_t shr64(uint64_t x, uint32_t s)
{
    uint64_t r;
    asm("shr.b64 %0, %1, %2;" : "=l"(r) : "l"(x), "r"(s));
    return r;
}

// (x[i], y[i]) for a dynamic i in [0, K): a select tree on the bits of i (the two
// coordinates share the predicates).
template <int K>
__device__ __forceinline__ void pick_xy(const float (&x)[K], const float (&y)[K], uint32_t i, float &rx, float &ry)
{
    const bool b0 = i & 1u, b1 = i & 2u;
    float x2[(K + 1) / 2], y2[(K + 1) / 2];
#pragma unroll
    for (int k = 0; k < K / 2; ++k) { x2[k] = b0 ? x[2 * k + 1] : x[2 * k]; y2[k] = b0 ? y[2 * k + 1] : y[2 * k]; }
    if (K == 4) {
        rx = b1 ? x2[1] : x2[0];
        ry = b1 ? y2[1] : y2[0];
    } else {
        const bool b2 = i & 4u;
        const float x4a = b1 ? x2[1] : x2[0], x4b = b1 ? x2[3] : x2[2];
        const float y4a = b1 ? y2[1] : y2[0], y4b = b1 ? y2[3] : y2[2];
        rx = b2 ? x4b : x4a;
        ry = b2 ? y4b : y4a;
    }
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

// the number of non-zero bytes of a record = its nx (0x00 is the padding, never a flag: R2)
template <int K>
__device__ __forceinline__ int record_len(const Seq<K> &s)
{
    int c = 0;
#pragma unroll
    for (int q = 0; q < K / 4; ++q) {
        uint64_t t = s.w[q] | (s.w[q] >> 4);
        t |= t >> 2;
        t |= t >> 1;
        c += __popcll(t & 0x0101010101010101ull);
    }
    return c;
}

template <int K>
__device__ __forceinline__ uint32_t seq_byte(const Seq<K> &s, int p)  // p static
{
    const uint64_t w = s.w[p >> 3];
    return (uint32_t)(w >> (8 * (p & 7))) & 0xFFu;
}

}  // namespace dgal

#ifndef DGAL_SEPT_FUSED
#define DGAL_SEPT_FUSED 1   // K = 4 fused kernels (paired, box) keep the explicit separating-line test
#endif                      // (without it ptxas spills them; A/B switch)
#ifndef DGAL_SEPT_FUSED8
#define DGAL_SEPT_FUSED8 0  // K = 8 fused kernel: without it (A/B cfg4 fused 0.383 -> 0.377 ms)
#endif
#ifndef DGAL_THIN
#define DGAL_THIN 1     // thin / sliver pairs: areas of the recorded intersection in double (dgal_exact.cuh)
#endif
#ifndef DGAL_THIN_BWD
#define DGAL_THIN_BWD DGAL_THIN   // ... also in the backward's S:303 coefficients
#endif
#include "dgal_exact.cuh"   // double-precision area of the recorded intersection (thin pairs)

namespace dgal {

// ---------------------------------------------------------------------------
// forward: intersect + area + IoU
// ---------------------------------------------------------------------------
template <int K, bool FLAGS>
struct FwdOut {
    float iou;
    int nx;
    Seq<K> seq;
    float A1x2, A2x2, Aix2;  // twice the areas (the 3D box forward extrudes them)
    bool thin;               // THIN: a thin pair, its record kept for fwd_thin_fix (iou_fwd)
};

// Extrusion of the footprints for the yaw-only 3D IoU:
// V_1 = A_1 d1, V_2 = A_2 d2, V_i = A_i dz.  The 2D path passes {1, 1, 1}, which
// folds away (x * 1.0f == x), leaving the plain IoU arithmetic.
struct Extrude {
    float dz, d1, d2;
};
__device__ __forceinline__ Extrude flat() { return Extrude{1.f, 1.f, 1.f}; }

// Scalars of the S:303 chain the box front end needs: dL/dV_i, dL/dV_1 (= dL/dV_2)
// and the footprint areas (zero for an empty pair).
struct VolCoef {
    float cvi, cvu, ai, a1, a2;
};

// R^2 / A_u above which a pair's float area is recomputed in double: the float
// error is ~c eps R^2 with c of a few (measured: aspect-10 triangles at scene
// coordinates, R^2/A_u ~ 10, max IoU error 2.3e-6 against the 1e-5 tolerance);
// flagged pairs in the benchmark workloads: cfg3 4e-5 (nonempty), cfg4 0.
constexpr float kThinRatio = 8.f;

// squared extent of the pair about p1.v0 (the polygons recentred on it)
template <int K>
__device__ __forceinline__ float pair_extent2(const Poly<K> &P, const Poly<K> &Q)
{
#ifndef DGAL_THIN_SUMSQ
#define DGAL_THIN_SUMSQ 4   // the K for which R^2 is taken as (sum of squared norms) / 2K (A/B: K = 4 faster)
#endif
    if (K == DGAL_THIN_SUMSQ) {
    // mean of the squared vertex norms (<= R^2 <= 2K x it): paired accumulation, no max chain
    uint64_t acc = 0ull;
#pragma unroll
    for (int q = 0; q < K / 2; ++q) {
        const uint64_t qx = f2pack(Q.x[2 * q], Q.x[2 * q + 1]), qy = f2pack(Q.y[2 * q], Q.y[2 * q + 1]);
        const uint64_t px = f2pack(P.x[2 * q], P.x[2 * q + 1]), py = f2pack(P.y[2 * q], P.y[2 * q + 1]);
        acc = f2fma(qx, qx, f2fma(qy, qy, f2fma(px, px, f2fma(py, py, acc))));
    }
    float a, b;
    f2unpack(acc, a, b);
    return (a + b) * (1.f / (2 * K));
    }
    // p2's vertices two per paired instruction, in the (2q, 2q+1) pairs the decision
    // rows pack (no register moves); p1's scalar (P.x[0] = P.y[0] = 0 after recentring)
    float r = 0.f;
#pragma unroll
    for (int q = 0; q < K / 2; ++q) {
        const uint64_t qx = f2pack(Q.x[2 * q], Q.x[2 * q + 1]), qy = f2pack(Q.y[2 * q], Q.y[2 * q + 1]);
        float a, b;
        f2unpack(f2fma(qx, qx, f2mul(qy, qy)), a, b);
        r = fmaxf(r, fmaxf(a, b));
    }
#pragma unroll
    for (int k = 0; k < K; ++k) r = fmaxf(r, fmaf(P.x[k], P.x[k], P.y[k] * P.y[k]));
    return r;
}

// thin: R^2 > kThinRatio A_u, with twice the union area aux2 = A1x2 + A2x2 - Aix2
__device__ __forceinline__ bool pair_is_thin(float R2, float aux2)
{
    return R2 > (0.5f * kThinRatio) * aux2;
}

// the backward's form (its area is a sum of piece terms about p1.v0, whose rounding
// is bounded by ~2 eps S, S = sum over the 2K vertices of |v|^2 <= 2K R^2): thin when
// S > 2K kThinRatio A_u (= 4 K kThinRatio / 2 aux2; cfg3 box pairs have S / aux2 ~ 2-6)
template <int K>
__device__ __forceinline__ bool pair_is_thin_sum(float S, float aux2)
{
    return S > (float)(K * kThinRatio) * aux2;
}

// ---------------------------------------------------------------------------
// Walk tables for K = 4 (the flag walk of iou_fwd and the p2 inside mask of
// clip_intervals as table lookups: the forward is bound by the ALU pipe, and the
// bit-serial walk was its largest ALU consumer — DESIGN.md §4.1).  Generated at
// compile time from the same rules the bit-serial code implements; staged in
// shared memory by the kernels that use them (load_walk_lut4).
//
//   e[st << 6 | jo << 4 | in2]: the flag bytes p1 edge i contributes, for edge
//     state st = valid | has_in << 1 | has_out << 2, exit line jo and p2 inside
//     mask in2, as {bytes lo, bytes hi, M, count}:
//       byte 0   FromP1(i) = 0x40 | i, or the entry Cross(i, j_in) = 0xC0 | i << 3 | j_in
//       byte 1   the exit Cross(i, jo) = 0xC0 | i << 3 | jo          (has_out)
//       byte 2.. FromP2(jo+1), FromP2(jo+2), ... while inside p1    (has_out)
//     without the terms in i and j_in: bytes + M * i is the group of edge i (M
//     puts i in bits 0-2 of a FromP1 byte, bits 3-5 of a Cross byte), j_in is
//     OR-ed in by the caller.  An invalid edge contributes nothing (all 0).
//   in2[ev_in | ev_out << 4]: p2 vertices inside p1 given the p2 lines carrying
//     an entry / an exit (the segmented scan of clip_intervals; 0 without events).
// ---------------------------------------------------------------------------
struct alignas(16) WalkLut4 {
    uint32_t e[512][4];
    uint8_t in2[256];
};

constexpr uint32_t walk4_in2(uint32_t ev_in, uint32_t ev_out)
{
    const uint32_t ev = ev_in | ev_out;
    if (ev == 0u) return 0u;
    uint32_t evd = ev | (ev << 4);
    uint32_t st = (ev_out & ~ev_in) | ((ev_out & ~ev_in) << 4);
    for (int sh = 1; sh < 8; sh <<= 1) {
        st = (st & evd) | ((st << sh) & ~evd);
        evd |= evd << sh;
    }
    return (st >> 3) & 0xFu;
}

constexpr WalkLut4 make_walk_lut4()
{
    WalkLut4 L{};
    for (uint32_t idx = 0; idx < 512; ++idx) {
        const uint32_t st = idx >> 6, jo = (idx >> 4) & 3u, in2 = idx & 15u;
        const bool valid = st & 1u, has_in = st & 2u, has_out = st & 4u;
        uint64_t g = 0;
        uint32_t M = 0, c = 0;
        if (valid) {
            g = has_in ? 0xC0u : 0x40u;
            M = has_in ? 8u : 1u;
            c = 1;
            if (has_out) {
                g |= (uint64_t)(0xC0u | jo) << 8;
                M |= 8u << 8;
                c += 1;
                const uint32_t p0 = (jo + 1u) & 3u;
                const uint32_t rot = ((in2 | (in2 << 4)) >> p0) & 15u;
                for (uint32_t r = 0; r < 4 && ((rot >> r) & 1u); ++r, ++c)
                    g |= (uint64_t)(0x80u | ((p0 + r) & 3u)) << (16 + 8 * r);
            }
        }
        L.e[idx][0] = (uint32_t)g;
        L.e[idx][1] = (uint32_t)(g >> 32);
        L.e[idx][2] = M;
        L.e[idx][3] = c;
    }
    for (uint32_t v = 0; v < 256; ++v) L.in2[v] = (uint8_t)walk4_in2(v & 15u, v >> 4);
    return L;
}

static __device__ const WalkLut4 kWalkLut4 = make_walk_lut4();

// Stage the tables in shared memory (all threads of the CTA; the caller
// synchronises before use).
__device__ __forceinline__ void load_walk_lut4(WalkLut4 &dst, int tid, int nthreads)
{
    const uint4 *s = reinterpret_cast<const uint4 *>(&kWalkLut4);
    uint4 *d = reinterpret_cast<uint4 *>(&dst);
    for (int q = tid; q < (int)(sizeof(WalkLut4) / 16); q += nthreads) d[q] = __ldg(s + q);
}

// Walk tables for K = 8 (the paired forward's flag walk).  The
// K = 4 table keyed by the whole p2 inside mask would be 2^8 x 8 x 8 entries; the
// K = 8 walk splits it in two small lookups instead:
//   L[in2 << 3 | jo]: the length of the run of p2 vertices inside p1 after p2
//     edge jo (trailing ones of in2 rotated right by jo + 1; 0..8);
//   g[jo * 9 + L]: the bytes after byte 0 of a p1 edge's group when it exits
//     across p2 line jo followed by that run — {bytes lo, bytes hi, -, count}:
//       byte 1   the exit Cross(i, jo) = 0xC0 | i << 3 | jo   (without i << 3)
//       byte 2.. FromP2(jo+1), ..., FromP2(jo+L)      (up to 8: bytes 8, 9 in hi)
//     count = 2 + L; g[72] = {0, 0, 0, 1} (a valid edge without an exit: byte 0
//     only), g[73] = all 0 (an invalid edge).
// Byte 0 (FromP1(i) or the entry Cross(i, j_in)) and the i << 11 of byte 1 are
// OR-ed in by the caller (static shared memory: the table must stay small).
struct alignas(16) WalkLut8 {
    uint32_t g[74][4];
    uint8_t L[256 * 8];
};

constexpr WalkLut8 make_walk_lut8()
{
    WalkLut8 W{};
    {
        for (uint32_t jo = 0; jo < 8; ++jo) {
            for (uint32_t L = 0; L <= 8; ++L) {
                uint64_t lo = (uint64_t)(0xC0u | jo) << 8, hi = 0;
                for (uint32_t r = 0; r < L; ++r) {
                    const uint64_t b = 0x80u | ((jo + 1u + r) & 7u);
                    const uint32_t at = 2u + r;
                    if (at < 8u) lo |= b << (8u * at);
                    else hi |= b << (8u * (at - 8u));
                }
                uint32_t *e = W.g[jo * 9 + L];
                e[0] = (uint32_t)lo; e[1] = (uint32_t)(lo >> 32); e[2] = (uint32_t)hi; e[3] = 2u + L;
            }
        }
        W.g[72][3] = 1u;
    }
    for (uint32_t in2 = 0; in2 < 256; ++in2) {
        for (uint32_t jo = 0; jo < 8; ++jo) {
            const uint32_t p0 = (jo + 1u) & 7u;
            const uint32_t rot = ((in2 | (in2 << 8)) >> p0) & 0xFFu;
            uint32_t L = 0;
            while (L < 8u && ((rot >> L) & 1u)) ++L;
            W.L[in2 << 3 | jo] = (uint8_t)L;
        }
    }
    return W;
}

static __device__ const WalkLut8 kWalkLut8 = make_walk_lut8();

__device__ __forceinline__ void load_walk_lut8(WalkLut8 &dst, int tid, int nthreads)
{
    const uint4 *s = reinterpret_cast<const uint4 *>(&kWalkLut8);
    uint4 *d = reinterpret_cast<uint4 *>(&dst);
    for (int q = tid; q < (int)(sizeof(WalkLut8) / 16); q += nthreads) d[q] = __ldg(s + q);
}

// The edge-interval clip shared by the paired forward, the pairwise path and the
// fused loss kernel.
//
//   * p1 side: the Cyrus-Beck interval [t0, t1] of every edge of p1 against the
//     closed half-planes of p2; the line that bounds it rides in the low mantissa
//     bits.  A piece that starts inside the edge is an ENTRY of p1's boundary
//     into p2 (through p2 line j_in), one that ends inside it an EXIT (through
//     p2 line j_out).  All of these come from one set of decision values d, so
//     they are mutually consistent: the inside part of p1's boundary is a set
//     of arcs, each from an entry to an exit.
//   * p2 side: derived from the p1 events, not decided separately.  After an
//     exit through line j the boundary of p1 ∩ p2 follows p2 edge j from that
//     very crossing point X_out; it leaves p2's boundary at the next entry, at
//     that crossing point X_in.  So the piece on p2 edge j runs from X_out (or
//     w_j) to X_in (or w_j+1), and p2 vertex j is inside p1 iff the last event
//     before it along p2 is an exit (segmented scan of the events around p2).
//     Only when there are no events at all is p2's inside-ness decided on its
//     own (all vertices strictly inside the open half-planes of p1).
//
// Events are taken from SIGNS, not from rounded parameters: p1 vertex i is inside
// p2 iff all its d[i][j] > 0 (one bit per vertex, shared by both edges at it);
// an edge has an entry iff it has a piece and its start is outside, an exit iff
// its end is outside, and an inside end point pins that end of the piece to 0 or
// 1 exactly.  So the arcs are well formed whatever the rounding (a t* within an
// ulp of 1 no longer hides an exit, a line index is never lost).
//
// Each crossing point is therefore ONE point shared by the two pieces that meet
// there, and the Green sum below is the area of a closed polygon: exact up to
// rounding of the points, independent of the origin, and stable when edges of
// p1 and p2 nearly coincide (prediction ~ target) — where independent t / s
// parameters of a near-parallel crossing are each ill-conditioned (~1/sin) and
// disagree.  DESIGN.md §4.1.
template <int K>
struct Clip {
    float gx[K], gy[K], fx[K], fy[K];  // edge vectors of p1, p2
    float C1[K], C2[K];                // shoelace terms v_i x v_i+1, w_j x w_j+1
    float t0[K], t1[K];                // boundary piece [t0, t1] on p1 edge i (empty if t0 > t1)
    uint32_t jin, jout;                // line index of the entry / exit of p1 edge i (4 bits each)
    uint32_t valid, enter, leave;      // p1 edges with a piece / an entry / an exit (bit i)
    float ax[K], ay[K], bx[K], by[K];  // PIECES: piece on p2 edge j runs from (ax, ay) to (bx, by)
    uint32_t key[K];                   // walk-table key of p1 edge i: st << 6 | jo << 4 | j_in << 16 (WalkLut4)
    uint32_t on2;                      // p2 edges carrying a boundary piece
    uint32_t in2;                      // p2 vertices inside p1 (consistent with the events)
    float A1x2, A2x2, Aix2;            // twice the areas
    bool nonempty;
    bool sep;                          // a p2 edge line separates p1 (strictly): empty for sure
    bool ill;                          // ILL: some p1 edge crosses a p2 line at |sin| < kIllSin
};

// |sin| of the angle between a p1 edge and a p2 edge below which the fused kernels
// hand the pair to their refine pass (crossing parameters in float are conditioned
// by 1/sin: ~6e-8 / sin relative; the split backward refines |sin| < 2^-10 in double,
// DESIGN.md §4.2b)
constexpr float kIllSin = 0.001953125f;   // 2^-9

// p1, p2 must already be recentred (coordinates near 0; p1.v0 or a box centre).
// How the p2 side of Green's sum is formed (§4.1 of DESIGN.md):
//   kP2Pieces  materialise the end points of the p2 pieces (c.ax .. c.by) with
//              per-(edge, line) selects — the fused gradient needs them;
//   kP2Regs    per-event form, the event's p2 vertex picked by a select tree;
//   kP2Smem    per-event form, the vertex read from a per-thread shared-memory
//              table (QTable) — one LDS instead of a select tree (the LSU pipe is
//              idle in these kernels, the ALU pipe is the binding one).
enum P2Mode { kP2Pieces = 0, kP2Regs = 1, kP2Smem = 2, kP2PiecesSmem = 3 };
// kP2PiecesSmem: the piece end points of kP2Pieces, scattered by event into a
//              per-thread shared-memory table (QTable x/y = a, stride; b at +2K)
//              instead of per-(edge, line) selects, then read back.

// Per-thread table of p2's (recentred) vertices in shared memory (kP2Smem): vertex j
// at x[j * stride], y[j * stride] for rows j < K, w_0 again at row K (the vertex after
// an entry line j is row j + 1, no wrap) and (0, 0) at row K + 1 (the vertex of an
// absent event: its Green term vanishes without a select).  Written and read by the
// same thread only.
struct QTable {
    const float *x, *y;
    int stride;
};

// Per-thread shared-memory table of the ILL test's per-line factors for K = 8 (in
// registers they spill the K = 8 fused kernel): the pair (2q, 2q+1) at p[q * st].
struct IllTab {
    uint64_t *p;
    int st;
    float sin = kIllSin;   // the |sin| threshold (boxes: their corners' rounding needs a larger one)
};

// ILL: also report whether some p1 edge i CROSSES some p2 line j (its end points on
// opposite sides: a candidate crossing of the Cyrus-Beck update) while being nearly
// parallel to it, |g_i x f_j| < kIllSin |g_i| |f_j| (c.ill; the Cyrus-Beck
// denominators are exactly these cross products) — a superset of the pairs with an
// ill-conditioned crossing (nearly parallel edges that do not cross — the opposite
// sides of two nearly aligned boxes — do not count: ~100x fewer pairs marked).
template <int K, int MODE, bool ILL = false, int ILLG = -1, bool WLUT = false>
__device__ __forceinline__ void clip_intervals(const Poly<K> &P, const Poly<K> &Q, Clip<K> &c,
                                               QTable qt = QTable{nullptr, nullptr, 0},
                                               const WalkLut4 *wl = nullptr, IllTab it = IllTab{nullptr, 0})
{
    constexpr bool LUT = (K == 4) && WLUT;   // in2 from the table (wl in shared memory; WLUT:
                                             // compile time — a shared address may be 0)
    // The explicit separating-line test (p1 strictly outside some p2 line -> empty)
    // is redundant: such a line bounds every p1 edge out (both ends negative: t* > 1
    // as a lower bound or < 0 as an upper one) and p2's centroid is outside p1, so
    // the clip finds no piece and no p2 vertex inside.  Dropped (K^2 max operations:
    // cfg3 forward -2.4 %, cfg4 -6 %; the GPU suite is unchanged); the fused kernels
    // (ILL) keep it — without it ptxas spills the K = 4 one.
    constexpr bool SEPT = ILL && (K == 4 ? DGAL_SEPT_FUSED : DGAL_SEPT_FUSED8);
    constexpr bool PIECES = (MODE == kP2Pieces || MODE == kP2PiecesSmem);
    constexpr bool PSMEM = (MODE == kP2PiecesSmem);
    constexpr uint32_t KMASK = (1u << K) - 1u;
    // edge vectors g_i = v_i+1 - v_i (p1), f_j = w_j+1 - w_j (p2); shoelace terms
    float *gx = c.gx, *gy = c.gy, *fx = c.fx, *fy = c.fy, *C1 = c.C1, *C2 = c.C2;
    float A1x2 = 0.f, A2x2 = 0.f;
#pragma unroll
    for (int i = 0; i < K; ++i) {
        const int i1 = (i + 1) % K;
        gx[i] = P.x[i1] - P.x[i]; gy[i] = P.y[i1] - P.y[i];
        fx[i] = Q.x[i1] - Q.x[i]; fy[i] = Q.y[i1] - Q.y[i];
        C1[i] = P.x[i] * P.y[i1] - P.x[i1] * P.y[i];
        C2[i] = Q.x[i] * Q.y[i1] - Q.x[i1] * Q.y[i];
        // same order as the A_i sum below: identical polygons give A_i == A_1 bitwise
        A1x2 = __fadd_rn(A1x2, C1[i]);
        A2x2 = __fadd_rn(A2x2, C2[i]);
    }

    // decision values, shifted by +tiny (below any non-degenerate value) so that
    // "inside" is "> 0" and no value is exactly 0:
    //   d[i][j] = f_j x (v_i - w_j) + tiny   p1 vertex i vs p2 line j, CLOSED test (d >= 0)
    // Computed row by row inside the edge loop below (row i+1 when edge i is
    // clipped), so only rows 0, i, i+1 are live: K = 8 needs 64 registers for all.
    auto drow = [&](int i, float (&r)[K]) {
        if (DGAL_F32X2 & 1) {   // lines 2q, 2q+1 in one register pair
            const uint64_t px = f2pack(P.x[i], P.x[i]), py = f2pack(P.y[i], P.y[i]);
            const uint64_t tiny2 = f2pack(kTiny, kTiny);
#pragma unroll
            for (int q = 0; q < K / 2; ++q) {
                const uint64_t Dx = f2sub(px, f2pack(Q.x[2 * q], Q.x[2 * q + 1]));
                const uint64_t Dy = f2sub(py, f2pack(Q.y[2 * q], Q.y[2 * q + 1]));
                const uint64_t fx2 = f2pack(fx[2 * q], fx[2 * q + 1]), fy2 = f2pack(fy[2 * q], fy[2 * q + 1]);
                f2unpack(f2add(f2sub(f2mul_nc(fx2, Dy), f2mul_nc(fy2, Dx)), tiny2), r[2 * q], r[2 * q + 1]);
            }
        } else {
#pragma unroll
            for (int j = 0; j < K; ++j) {
                const float Dx = __fsub_rn(P.x[i], Q.x[j]), Dy = __fsub_rn(P.y[i], Q.y[j]);
                r[j] = __fadd_rn(cross_rn(fx[j], fy[j], Dx, Dy), kTiny);
            }
        }
    };
    // p1 vertex i inside p2 (closed test, d never 0): bit i of in1, with its row
    auto inside = [&](const float (&r)[K]) {
        float mn = r[0];
#pragma unroll
        for (int j = 1; j < K; ++j) mn = fminf(mn, r[j]);
        return (uint32_t)(mn > 0.f);
    };
    float d0[K], dc[K], m1[K];
    drow(0, d0);
    uint32_t in1 = inside(d0);
#pragma unroll
    for (int j = 0; j < K; ++j) { dc[j] = d0[j]; m1[j] = d0[j]; }

    // Cyrus-Beck intervals of p1's edges.  For the edge a -> b against one line
    // (a, b = the shifted decision values of its end points, never 0): the inside
    // set is {t : a + t (b - a) > 0}; b > a bounds it below by t* = a / (a - b),
    // b < a above, b == a keeps all (a > 0) or nothing (a < 0).  An end point that
    // is inside pins its parameter below, so t* = a/(a-b) only has to be accurate
    // to an ulp (identical polygons still keep [0, 1] exactly).
    // den + tiny keeps r finite (a == b: r = 1e30, t* = +-huge), so every candidate
    // is finite and carries the index j of its line.  hi starts just above 1 so a
    // candidate that rounds to 1 still wins and keeps its index.
    // The piece exists iff an end point is inside or t0 < t1 (strictly: an edge
    // that only touches p2 at a point from outside has none); an inside end pins
    // its parameter, and the other one is clamped to the edge.
    float *t0 = c.t0, *t1 = c.t1;
    uint32_t jin = 0, jout = 0, valid = 0, enter = 0, leave = 0;
    const float hi0 = __int_as_float(0x3F800008);
    // ILL, inside the edge loop from its Cyrus-Beck denominators: candidate (i, j) is
    // ill when x = den^2 - sin^2 |g_i|^2 |f_j|^2 < 0 AND p = d[i][j] d[i+1][j] < 0 (a
    // crossing, or an end point exactly on the line); both signs AND-ed into one
    // accumulator (one LOP3 per candidate).  K = 4: the per-line factors
    // -sin^2 |f_j|^2 in registers, times |g_i|^2 per edge; K = 8: -sin^2 max|g|^2 |f_j|^2
    // in the caller's shared-memory table it (in registers they spill; the longest edge
    // standing in for each is conservative: a shorter edge is tested against a larger |sin|).
    uint32_t illacc = 0u;
    constexpr bool NSF_REG = (K == 4) || !ILL;
#ifndef DGAL_ILL_GMAX
#define DGAL_ILL_GMAX 1   // K = 4 too: max |g|^2 folded into the per-line factors (A/B: fused K=4 -1 %)
#endif
    // ILLG: 1 max|g|^2 folded in, 0 per-edge |g_i|^2 (boxes: their larger threshold would
    // queue ~2x more pairs), -1 the build default
    constexpr bool GMAX = !NSF_REG || (ILLG < 0 ? DGAL_ILL_GMAX : ILLG);
    uint64_t nsf[(ILL && NSF_REG) ? K / 2 : 1];
    if (ILL) {
        float gmax = 1.f;
        if (GMAX) {
            gmax = 0.f;
#pragma unroll
            for (int i = 0; i < K; ++i) gmax = fmaxf(gmax, fmaf(gx[i], gx[i], gy[i] * gy[i]));
        }
        const float ns = -it.sin * it.sin * gmax;
        const uint64_t ns2 = f2pack(ns, ns);
#pragma unroll
        for (int q = 0; q < K / 2; ++q) {
            const uint64_t fx2 = f2pack(fx[2 * q], fx[2 * q + 1]), fy2 = f2pack(fy[2 * q], fy[2 * q + 1]);
            const uint64_t v = f2mul(f2fma(fx2, fx2, f2mul(fy2, fy2)), ns2);
            if (NSF_REG) nsf[NSF_REG ? q : 0] = v;
            else it.p[q * it.st] = v;
        }
    }
    // Events (same pass).  An exit of p1 edge i through p2 line j_out starts the p2
    // piece on edge j_out at X_out = v_i + t1 g_i; an entry through line j_in ends
    // the piece on edge j_in at X_in = v_i + t0 g_i.  Green's term of such a piece,
    // X_out x w_j+1, equals C2_j + X_out x w_j up to X_out's distance from line j
    // (an ulp of its decision values), and w_j x X_in equals C2_j + w_j+1 x X_in
    // likewise; so the p2 side of the boundary contributes
    //     sum_{j on boundary} C2_j + sum_exits X_out x w_jout + sum_entries w_jin+1 x X_in
    // (a piece with both events on one edge adds the product of two vectors along
    // that edge, which vanishes).  One vertex select per event, no per-edge state.
    uint64_t sxw = 0ull, syw = 0ull;   // per-event modes: paired sums (exit, entry) of x*w.y, y*w.x
    float Aix2 = 0.f;   // twice the area of p1 ∩ p2 (Green over the closed boundary)
    uint32_t ev_out = 0, ev_in = 0;
    float *ax = c.ax, *ay = c.ay, *bx = c.bx, *by = c.by;
    // kP2PiecesSmem table: a_j at (qt.x, qt.y)[j * st], b_j at (qt.x, qt.y)[(K + j) * st]
    float *tx = const_cast<float *>(qt.x), *ty = const_cast<float *>(qt.y);
    const int tst = qt.stride;
    if (PIECES) {
#pragma unroll
        for (int j = 0; j < K; ++j) {
            const int j1 = (j + 1) % K;
            if (PSMEM) {
                tx[j * tst] = Q.x[j]; ty[j * tst] = Q.y[j];
                tx[(K + j) * tst] = Q.x[j1]; ty[(K + j) * tst] = Q.y[j1];
            } else {
                ax[j] = Q.x[j]; ay[j] = Q.y[j];
                bx[j] = Q.x[j1]; by[j] = Q.y[j1];
            }
        }
    }
#pragma unroll
    for (int i = 0; i < K; ++i) {
        const int i1 = (i + 1) % K;
        float dn[K];   // row i+1 (row 0 for the closing edge)
        if (i1 != 0) {
            drow(i1, dn);
            in1 |= inside(dn) << i1;
#pragma unroll
            for (int j = 0; j < K; ++j) m1[j] = SEPT ? fmaxf(m1[j], dn[j]) : m1[j];
        } else {
#pragma unroll
            for (int j = 0; j < K; ++j) dn[j] = d0[j];
        }
        float lo = 0.f, hi = hi0;
        // ILL, K = 4: this edge's |g|^2 (K = 8: folded into the table as max |g|^2)
        uint64_t g2 = 0ull;
        float gg = 1.f;
        if (ILL && !GMAX) {
            gg = fmaf(gx[i], gx[i], gy[i] * gy[i]);
            g2 = f2pack(gg, gg);
        }
        if (DGAL_F32X2 & 2) {   // lines 2q, 2q+1 in one register pair (same arithmetic as below)
            const uint64_t tiny2 = f2pack(kTiny, kTiny), big2 = f2pack(kBig, kBig);
#pragma unroll
            for (int q = 0; q < K / 2; ++q) {
                const uint64_t a = f2pack(dc[2 * q], dc[2 * q + 1]);
                const uint64_t bq = f2pack(dn[2 * q], dn[2 * q + 1]);
                const uint64_t den = f2add(f2sub(a, bq), tiny2);
                float d0_, d1_;
                f2unpack(den, d0_, d1_);
                if (ILL) {
                    const uint64_t thr = !NSF_REG ? it.p[q * it.st]
                                         : (GMAX ? nsf[NSF_REG ? q : 0] : f2mul(g2, nsf[NSF_REG ? q : 0]));
                    float x0, x1, p0, p1;
                    f2unpack(f2fma(den, den, thr), x0, x1);
                    // (- 1e-26: an end point exactly on the line, d = +tiny = 1e-30, counts as a
                    // crossing for |d| of the other end up to 1e4)
                    f2unpack(f2fma(a, bq, f2pack(-1e-26f, -1e-26f)), p0, p1);
                    illacc |= (__float_as_uint(x0) & __float_as_uint(p0)) | (__float_as_uint(x1) & __float_as_uint(p1));
                }
                const uint64_t r = f2pack(rcp_approx(d0_), rcp_approx(d1_));
                const uint64_t m = f2pack(__saturatef(-d0_ * kBig), __saturatef(-d1_ * kBig));
                float u0, u1;
                f2unpack(f2mul(a, r), u0, u1);
                const uint64_t ve = f2pack(enc_idx(u0, 2 * q), enc_idx(u1, 2 * q + 1));
                float l0, l1, h0, h1;
                f2unpack(f2mul(m, ve), l0, l1);
                f2unpack(f2fma(m, big2, ve), h0, h1);
                lo = fmaxf(lo, fmaxf(l0, l1));
                hi = fminf(hi, fminf(h0, h1));
            }
        } else {
#pragma unroll
            for (int j = 0; j < K; ++j) {
                const float a = dc[j], b = dn[j];
                const float den = (a - b) + kTiny;
                if (ILL) {
                    float nf0, nf1;
                    f2unpack(NSF_REG ? nsf[NSF_REG ? j / 2 : 0] : it.p[(j / 2) * it.st], nf0, nf1);
                    illacc |= __float_as_uint(fmaf(den, den, gg * ((j & 1) ? nf1 : nf0))) &
                              __float_as_uint(fmaf(a, b, -1e-26f));
                }
                const float r = rcp_approx(den);
                const float m = __saturatef(-den * kBig);  // 1: bounds below
                const float ve = enc_idx(a * r, j);
                lo = fmaxf(lo, m * ve);                 // m * ve == ve (bits kept) or 0
                hi = fminf(hi, fmaf(m, kBig, ve));      // ve (bits kept) or huge
            }
        }
        const bool in_s = (in1 >> i) & 1u, in_e = (in1 >> i1) & 1u;
        // per-event modes: clamped to the edge (an invalid piece keeps a0 >= a1 without
        // the index bits either way, a valid one lies in [0, 1]; saturate keeps the
        // bits) — fewer selects; the piece modes keep the unclamped form (registers)
        const float hic = fminf(hi, 1.f);
        const float a0 = in_s ? 0.f : ((in_e || !PIECES) ? fminf(lo, 1.f) : lo);
        const float a1 = in_e ? 1.f : (!PIECES ? __saturatef(hi) : (in_s ? fmaxf(hic, 0.f) : hic));
        // strict, without the index bits (they perturb the last 3 ulps)
        const bool ok = in_s || in_e ||
                        (__int_as_float(__float_as_int(a0) & ~7) < __int_as_float(__float_as_int(a1) & ~7));
        const bool has_in = ok && !in_s, has_out = ok && !in_e;
        t0[i] = a0; t1[i] = a1;
        // p1 side of Green's sum (same order as A1x2: identical polygons reproduce
        // it).  Per-event modes: here, so t0 / t1 / C1 die early (registers); the
        // piece modes keep the interleaved order below (A/B: fused kernel faster).
        if (!PIECES) Aix2 = fmaf(fmaxf(a1 - a0, 0.f), C1[i], Aix2);
        valid |= (uint32_t)ok << i;
        enter |= (uint32_t)has_in << i;
        leave |= (uint32_t)has_out << i;
        const uint32_t ljin = (uint32_t)dec_idx(lo), ljout = (uint32_t)dec_idx(hi);
        jin |= ljin << (4 * i);
        jout |= ljout << (4 * i);
        if (has_in) ev_in |= 1u << ljin;
        if (has_out) ev_out |= 1u << ljout;
        c.key[i] = (ok ? 0x40u : 0u) | (has_in ? 0x80u : 0u) | (has_out ? 0x100u : 0u) | (ljout << 4) |
                   ((has_in ? ljin : 0u) << 16);
        const float xox = fmaf(a1, gx[i], P.x[i]), xoy = fmaf(a1, gy[i], P.y[i]);
        const float xix = fmaf(a0, gx[i], P.x[i]), xiy = fmaf(a0, gy[i], P.y[i]);
        DGAL_ASSERT(ljin < (uint32_t)K && ljout < (uint32_t)K);
        if (PSMEM) {
            if (has_out) { tx[ljout * tst] = xox; ty[ljout * tst] = xoy; }
            if (has_in) { tx[(K + ljin) * tst] = xix; ty[(K + ljin) * tst] = xiy; }
        } else if (PIECES) {
            const int ji = has_in ? (int)ljin : 8;   // 8: no event
            const int jo = has_out ? (int)ljout : 8;
#pragma unroll
            for (int j = 0; j < K; ++j) {
                ax[j] = (jo == j) ? xox : ax[j];
                ay[j] = (jo == j) ? xoy : ay[j];
                bx[j] = (ji == j) ? xix : bx[j];
                by[j] = (ji == j) ? xiy : by[j];
            }
        } else {
            // event vertices W_out = w_jout, W_in = w_jin+1, or (0, 0) without the event
            // (kP2Smem: row K + 1 of the table is zero; kP2Regs: selected), so the terms
            // need no select:
            //   sxw += (X_out x-part, X_in x-part) * (W_out.y, W_in.y)
            //   syw += (X_out y-part, X_in y-part) * (W_out.x, W_in.x)
            // one paired FMA each; p2e = (X_out x W_out) - (X_in x W_in) at the end
            float wox, woy, wix, wiy;
            if (MODE == kP2Smem) {
                // rows: w_0 .. w_K-1, w_0 again (row K: w_jin+1 is row jin + 1, no wrap),
                // zero (row K + 1)
                const uint32_t jo = has_out ? ljout : (uint32_t)(K + 1);
                const uint32_t jn = has_in ? ljin : (uint32_t)K;   // read at row jn + 1
                wox = qt.x[jo * qt.stride]; woy = qt.y[jo * qt.stride];
                wix = qt.x[jn * qt.stride + qt.stride]; wiy = qt.y[jn * qt.stride + qt.stride];
            } else {
                pick_xy<K>(Q.x, Q.y, ljout, wox, woy);
                pick_xy<K>(Q.x, Q.y, (ljin + 1u) & (K - 1u), wix, wiy);
                wox = has_out ? wox : 0.f; woy = has_out ? woy : 0.f;
                wix = has_in ? wix : 0.f; wiy = has_in ? wiy : 0.f;
            }
            // (area terms, not decisions: contracted)
            const uint64_t A2 = f2pack(a1, a0);
            const uint64_t X2 = f2fma(A2, f2pack(gx[i], gx[i]), f2pack(P.x[i], P.x[i]));
            const uint64_t Y2 = f2fma(A2, f2pack(gy[i], gy[i]), f2pack(P.y[i], P.y[i]));
            sxw = f2fma(X2, f2pack(woy, wiy), sxw);
            syw = f2fma(Y2, f2pack(wox, wix), syw);
        }
#pragma unroll
        for (int j = 0; j < K; ++j) dc[j] = dn[j];
    }
    // Separating p2 edge line: p1 strictly outside it -> empty.  Strict, so a
    // zero-length edge (a repeated vertex: polygons with fewer than K vertices are
    // padded that way), whose d are all exactly tiny, separates nothing; p1
    // touching a line from outside reaches zero area through the closed boundary.
    bool separated = false;
#pragma unroll
    for (int j = 0; j < K; ++j) separated |= SEPT && (m1[j] < kTiny);
    c.jin = jin; c.jout = jout; c.valid = valid; c.enter = enter; c.leave = leave;
    if (PSMEM) {
#pragma unroll
        for (int j = 0; j < K; ++j) {
            ax[j] = tx[j * tst]; ay[j] = ty[j * tst];
            bx[j] = tx[(K + j) * tst]; by[j] = ty[(K + j) * tst];
        }
    }

    // p2 vertex j inside p1 <=> the last event on p2 edges j-1, j-2, ... (cyclic) is
    // an exit without an entry after it.  Segmented scan over the doubled cycle:
    // position p carries the end state of the nearest event edge <= p.
    // With no event at all p1's boundary is entirely inside p2 or entirely
    // outside; in the latter case p2 lies inside p1 iff its vertex centroid does
    // (strictly: a p2 touching p1 from outside is not inside).
    const uint32_t ev = ev_out | ev_in;
    uint32_t in2;
    if ((ev | valid) == 0u) {
        // centroid m of p2 against p1's edge lines, g_i x (m - v_i), two edges per paired
        // op.  Without events and without a p1 piece the centroid is strictly inside p1
        // or strictly outside it (a p2 of positive area that touches p1 from outside
        // keeps its centroid away from p1's lines), so the test is >= 0: a zero-length
        // edge of a padded p1 (g = 0: the contraction-free cross product is exactly 0)
        // is no constraint.
        // (The K = 4 piece modes keep the direct form cross(g_i, m - v_i) > 0: fewer
        // instructions in their register allocation, static count 924 vs 936 fused.)
        float sx = 0.f, sy = 0.f;
#pragma unroll
        for (int j = 0; j < K; ++j) { sx += Q.x[j]; sy += Q.y[j]; }
        bool cin = true;
        if (!PIECES || K != 4) {
            const float mx = sx * (1.f / K), my = sy * (1.f / K);
            const uint64_t mx2 = f2pack(mx, mx), my2 = f2pack(my, my);
#pragma unroll
            for (int q = 0; q < K / 2; ++q) {
                const uint64_t gx2 = f2pack(gx[2 * q], gx[2 * q + 1]), gy2 = f2pack(gy[2 * q], gy[2 * q + 1]);
                const uint64_t dx2 = f2sub(mx2, f2pack(P.x[2 * q], P.x[2 * q + 1]));
                const uint64_t dy2 = f2sub(my2, f2pack(P.y[2 * q], P.y[2 * q + 1]));
                const uint64_t v = f2sub(f2mul_nc(gx2, dy2), f2mul_nc(gy2, dx2));
                float v0, v1;
                f2unpack(v, v0, v1);
                cin &= (v0 >= 0.f) & (v1 >= 0.f);
            }
        } else {
            const float mx = sx * (1.f / K), my = sy * (1.f / K);
#pragma unroll
            for (int i = 0; i < K; ++i)
                cin &= (cross_rn(gx[i], gy[i], mx - P.x[i], my - P.y[i]) > 0.f) | (fabsf(gx[i]) + fabsf(gy[i]) == 0.f);
        }
        in2 = cin ? KMASK : 0u;
    } else if (ev == 0u) {
        in2 = 0u;   // p1's boundary inside p2 without a crossing: p1 within p2
    } else if (LUT) {
        in2 = wl->in2[ev_in | (ev_out << 4)];
    } else {
        uint32_t evd = ev | (ev << K);
        uint32_t st = (ev_out & ~ev_in) | ((ev_out & ~ev_in) << K);
#pragma unroll
        for (int sh = 1; sh < 2 * K; sh <<= 1) {
            st = (st & evd) | ((st << sh) & ~evd);
            evd |= evd << sh;
        }
        in2 = (st >> (K - 1)) & KMASK;               // state after edge j-1, j = 0..K-1
    }
    const uint32_t on2 = ev | in2;

    // p2 side of Green's sum (identical polygons: no events, no p2 piece, so Aix2
    // keeps the p1 side, which reproduces A1x2 bitwise); piece modes interleave
#pragma unroll
    for (int k = 0; k < K; ++k) {
        if (PIECES) Aix2 = fmaf(fmaxf(t1[k] - t0[k], 0.f), C1[k], Aix2);
        const float c2 = PIECES ? cross_rn(ax[k], ay[k], bx[k], by[k]) : C2[k];
        Aix2 = __fadd_rn(Aix2, ((on2 >> k) & 1u) ? c2 : 0.f);
    }
    if (!PIECES) {
        float xo, xi, yo, yi;
        f2unpack(sxw, xo, xi);
        f2unpack(syw, yo, yi);
        Aix2 = __fadd_rn(Aix2, __fsub_rn(__fsub_rn(xo, yo), __fsub_rn(xi, yi)));
    }
    Aix2 = fminf(Aix2, fminf(A1x2, A2x2));
    c.A1x2 = A1x2;
    c.A2x2 = A2x2;
    c.Aix2 = Aix2;
    c.on2 = on2;
    c.in2 = in2;
    c.nonempty = !separated && (Aix2 > 0.f);
    c.sep = separated;
    c.ill = ILL && (illacc >> 31) != 0u;
}

// The flag walk of R3 from the per-edge clip results (bit form; the K = 4 / K = 8
// kernels use table forms of the same rules): walking p1's edges in order, a piece
// emits FromP1(i) or its entry Cross(i, j_in), then its exit Cross(i, j_out) and the
// run of p2 vertices inside p1 after p2 edge j_out.  Masks: bit i of valid / enter /
// leave, 4 bits per edge of jin / jout; in2: p2 vertices inside p1.  Returns the
// byte count (s must be zero on entry).
template <int K>
__device__ __forceinline__ int walk_bits(uint32_t valid_m, uint32_t enter_m, uint32_t leave_m, uint32_t jin_m,
                                         uint32_t jout_m, uint32_t in2, Seq<K> &s)
{
    constexpr uint32_t KMASK = (1u << K) - 1u;
    const uint32_t in2dup = in2 | (in2 << K);
    int pos = 0;
#pragma unroll
    for (int i = 0; i < K; ++i) {
        const bool valid = (valid_m >> i) & 1u;
        const bool has_in = (enter_m >> i) & 1u;
        const bool has_out = (leave_m >> i) & 1u;
        const uint32_t b0 = has_in ? (0xC0u | (i << 3) | ((jin_m >> (4 * i)) & 7u)) : (0x40u | i);
        const uint32_t jo = (jout_m >> (4 * i)) & 7u;
        const uint32_t b1 = 0xC0u | (i << 3) | jo;
        // run of p2 vertices inside p1 after p2 edge j_out: trailing ones of in2 rotated
        const uint32_t p0 = (jo + 1u) & (K - 1u);
        const uint32_t rot = (in2dup >> p0) & KMASK;
        const uint32_t L = __ffs(~rot) - 1;               // <= K
        uint64_t run;
        if (K == 4) {
            const uint32_t pat = __funnelshift_r(0x83828180u, 0x83828180u, 8u * p0);
            run = (uint64_t)(pat & (uint32_t)(shl64(1ull, 8u * L) - 1ull));
        } else {
            const uint64_t pat = 0x8786858483828180ull;
            const uint64_t r8 = shr64(pat, 8u * p0) | shl64(pat, 64u - 8u * p0);
            run = r8 & (shl64(1ull, 8u * L) - 1ull);
        }
        if (K == 4) {
            uint64_t seg = b0;
            seg |= has_out ? (((uint64_t)b1 << 8) | (run << 16)) : 0ull;
            const int c = valid ? (has_out ? 2 + (int)L : 1) : 0;
            s.w[0] |= valid ? shl64(seg, 8u * (uint32_t)pos) : 0ull;
            pos += c;
        } else {
            // group = b0 | b1 << 8 | run << 16 (up to 9 bytes: lo word + byte 8),
            // OR-ed in at byte pos of the 16-byte sequence, branch-free
            const uint64_t glo = has_out ? ((uint64_t)b0 | ((uint64_t)b1 << 8) | (run << 16)) : (uint64_t)b0;
            const uint64_t ghi = has_out ? (run >> 48) : 0ull;
            const uint32_t sh = 8u * (uint32_t)pos;
            const uint64_t olo = shl64(glo, sh);
            const uint64_t ohi = (sh >= 64u) ? shl64(glo, sh - 64u) : (shr64(glo, 64u - sh) | shl64(ghi, sh));
            s.w[0] |= valid ? olo : 0ull;
            s.w[Seq<K>::NW - 1] |= valid ? ohi : 0ull;
            pos += valid ? (has_out ? 2 + (int)L : 1) : 0;
        }
    }
    return pos;
}

// The record (nx, xflags) of a thin pair recomputed in double (the thin-pair paths,
// after their tile loops; rare).  A thin pair's float decisions can be wrong where the
// shapes are a few ulps of their coordinates wide (aspect 1e4 at 354 m: a missed
// crossing turns the event order into a run of far-away p2 vertices "inside" p1,
// tools/probes/thin_dbg.py), and fwd_thin_fix only recomputes the areas OF the record.
// Same rules as clip_intervals + walk_bits, scalar and in double from the vertex source
// (dgal_exact.cuh: float inputs, their differences exact in double): closed inside
// test d >= 0, per edge the Cyrus-Beck interval over the lines it crosses (an edge
// outside a line at both ends has no piece), events, p2 vertices inside p1 from the
// event order, the walk.  m = 0 when fewer than 3 or more than 2K vertices.
template <int K, class VERTS>
__device__ __forceinline__ void record_exact(const VERTS &V, Seq<K> &s, int &m)
{
    constexpr int KM = K - 1;
    constexpr uint32_t KMASK = (1u << K) - 1u;
    // decision value of p1 vertex i against p2 line j (p2 edge j, CCW: inside >= 0)
    auto dec = [&](int i, int j) -> double {
        double vx, vy, wx, wy, w1x, w1y;
        V.p(i, vx, vy);
        V.q(j, wx, wy);
        V.q((j + 1) & KM, w1x, w1y);
        return (w1x - wx) * (vy - wy) - (w1y - wy) * (vx - wx);
    };
    uint32_t in1 = 0;
#pragma unroll 1
    for (int i = 0; i < K; ++i) {
        bool in = true;
#pragma unroll 1
        for (int j = 0; j < K; ++j) in = in && dec(i, j) >= 0.0;
        in1 |= (uint32_t)in << i;
    }
    uint32_t valid = 0, enter = 0, leave = 0, jin = 0, jout = 0, ev_in = 0, ev_out = 0;
#pragma unroll 1
    for (int i = 0; i < K; ++i) {
        const int i1 = (i + 1) & KM;
        double lo = 0.0, hi = 1.0;
        int jl = 0, jh = 0;
        bool kill = false;
#pragma unroll 1
        for (int j = 0; j < K; ++j) {
            const double a = dec(i, j), b = dec(i1, j);
            if (a >= 0.0 && b >= 0.0) continue;          // no constraint
            if (a < 0.0 && b < 0.0) { kill = true; continue; }   // edge outside line j
            const double t = a / (a - b);                 // opposite signs: a - b != 0
            if (b > a) {                                  // enters through line j
                if (t > lo || (t == lo && j > jl)) { lo = t; jl = j; }
            } else if (t < hi || (t == hi && j < jh)) {   // exits through line j
                hi = t; jh = j;
            }
        }
        const bool in_s = (in1 >> i) & 1u, in_e = (in1 >> i1) & 1u;
        const double a0 = in_s ? 0.0 : fmin(lo, 1.0), a1 = in_e ? 1.0 : fmax(fmin(hi, 1.0), 0.0);
        const bool ok = in_s || in_e || (!kill && a0 < a1);
        const bool has_in = ok && !in_s, has_out = ok && !in_e;
        valid |= (uint32_t)ok << i;
        enter |= (uint32_t)has_in << i;
        leave |= (uint32_t)has_out << i;
        jin |= (has_in ? (uint32_t)jl : 0u) << (4 * i);
        jout |= (has_out ? (uint32_t)jh : 0u) << (4 * i);
        if (has_in) ev_in |= 1u << jl;
        if (has_out) ev_out |= 1u << jh;
    }
    const uint32_t ev = ev_in | ev_out;
    uint32_t in2;
    if ((ev | valid) == 0u) {
        // no piece, no event: p2 within p1 iff its vertex centroid is (strictly or on
        // an edge line: p2 of positive area keeps its centroid off p1's lines otherwise)
        double mx = 0.0, my = 0.0;
#pragma unroll 1
        for (int j = 0; j < K; ++j) {
            double x, y;
            V.q(j, x, y);
            mx += x;
            my += y;
        }
        mx /= K;
        my /= K;
        bool cin = true;
#pragma unroll 1
        for (int i = 0; i < K; ++i) {
            double vx, vy, v1x, v1y;
            V.p(i, vx, vy);
            V.p((i + 1) & KM, v1x, v1y);
            cin = cin && (v1x - vx) * (my - vy) - (v1y - vy) * (mx - vx) >= 0.0;
        }
        in2 = cin ? KMASK : 0u;
    } else if (ev == 0u) {
        in2 = 0u;
    } else {   // the last event before p2 vertex j along p2 is an exit (clip_intervals)
        uint32_t evd = ev | (ev << K);
        uint32_t st = (ev_out & ~ev_in) | ((ev_out & ~ev_in) << K);
#pragma unroll
        for (int sh = 1; sh < 2 * K; sh <<= 1) {
            st = (st & evd) | ((st << sh) & ~evd);
            evd |= evd << sh;
        }
        in2 = (st >> (K - 1)) & KMASK;
    }
#pragma unroll
    for (int q = 0; q < Seq<K>::NW; ++q) s.w[q] = 0ull;
    int pos = walk_bits<K>(valid, enter, leave, jin, jout, in2, s);
    if (pos == 0 && in2 == KMASK) {   // p2 inside p1: all FromP2, in order
        if (K == 4) s.w[0] = 0x83828180ull;
        else { s.w[0] = 0x8786858483828180ull; s.w[Seq<K>::NW - 1] = 0ull; }
        pos = K;
    }
    m = (pos >= 3 && pos <= 2 * K) ? pos : 0;
    if (m == 0) {
#pragma unroll
        for (int q = 0; q < Seq<K>::NW; ++q) s.w[q] = 0ull;
    }
}

// A thin pair's forward outputs: its record recomputed in double (record_exact), then
// the areas of that record in double (fwd_thin_fix).
template <int K, class VERTS>
__device__ __forceinline__ void fwd_thin_redo(const VERTS &V, Seq<K> &s, int &m, float &iou, AreasX2 *out = nullptr)
{
    record_exact<K>(V, s, m);
    fwd_thin_fix<K>(V, s, m, iou, out);
}

// p1, p2 must already be recentred on o = p1.v0 (p1.x[0] == p1.y[0] == 0).
// THIN (FLAGS only): detect thin pairs, R^2 > kThinRatio A_u (pair_is_thin).  A thin
// pair's float area sum — including the sign test that decides an empty
// intersection — is not accurate enough: out.thin is set and out.seq / out.nx hold
// the walk's record whatever the sign of the float area (when the pair is not
// separated and the walk has 3..2K vertices), so the caller can recompute the areas
// of p1, p2 and of that record in double (areas_exact, dgal_exact.cuh) and decide
// emptiness and the IoU from them (fwd_thin_fix).  The kernels do that after their
// tile loop (rare; keeps the double-precision code out of the hot loop).
template <int K, bool FLAGS, int MODE = (K == 4 ? kP2Pieces : kP2Regs), bool THIN = false, bool WLUT = false>
__device__ __forceinline__ FwdOut<K, FLAGS> iou_fwd(const Poly<K> &P, const Poly<K> &Q,
                                                    QTable qt = QTable{nullptr, nullptr, 0},
                                                    const WalkLut4 *wl = nullptr,
                                                    const WalkLut8 *wl8 = nullptr)
{
    constexpr uint32_t KMASK = (1u << K) - 1u;
    Clip<K> c;
    clip_intervals<K, MODE, false, -1, WLUT>(P, Q, c, qt, wl);
    // (after the clip, which keeps P and Q live to its end anyway: one register through the walk)
    const float R2 = (FLAGS && THIN) ? pair_extent2<K>(P, Q) : 0.f;
    const float *t0 = c.t0, *t1 = c.t1;
    const float A1x2 = c.A1x2, A2x2 = c.A2x2, Aix2 = c.Aix2;
    bool nonempty = c.nonempty;

    FwdOut<K, FLAGS> out;
#pragma unroll
    for (int k = 0; k < Seq<K>::NW; ++k) out.seq.w[k] = 0;
    out.nx = 0;
    out.iou = 0.f;
    out.A1x2 = A1x2;
    out.A2x2 = A2x2;
    out.Aix2 = 0.f;
    out.thin = false;

    if (FLAGS) {
        // p2 vertices inside p1, consistent with the crossings (clip_intervals)
        const uint32_t in2 = c.in2;
        const uint32_t in2dup = in2 | (in2 << K);

        // Walk p1's edges in order: [FromP1(i) | Cross(i, j_in)] [Cross(i, j_out) run of FromP2]
        Seq<K> s;
#pragma unroll
        for (int k = 0; k < Seq<K>::NW; ++k) s.w[k] = 0;
        int pos = 0;
        if (K == 4 && WLUT) {
            // table walk: edge i's group = table bytes + M i | j_in, at the byte offset
            // given by the prefix sum of the counts (all four in one multiply)
            uint32_t glo[4], ghi[4], cnt = 0;
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const uint32_t key = c.key[i];
                const uint4 e = *reinterpret_cast<const uint4 *>(wl->e[(key & 0x1F0u) | in2]);
                glo[i] = (e.x + e.z * (uint32_t)i) | (key >> 16);
                ghi[i] = e.y;
                cnt += e.w << (8 * i);
            }
            const uint32_t off = cnt * 0x08080800u;   // byte i: 8 x (count of edges < i)
            uint64_t w = (uint64_t)ghi[0] << 32 | glo[0];
#pragma unroll
            for (int i = 1; i < 4; ++i)
                w |= shl64((uint64_t)ghi[i] << 32 | glo[i], (off >> (8 * i)) & 0xFFu);
            s.w[0] = w;
            pos = (int)((cnt * 0x01010101u) >> 24);
        } else if (K == 8 && WLUT) {
            // table walk (WalkLut8): run length, then the group's bytes 1.. and count
            const uint8_t *Lrow = wl8->L + (in2 << 3);
#pragma unroll
            for (int i = 0; i < K; ++i) {
                const bool valid = (c.valid >> i) & 1u;
                const bool has_in = (c.enter >> i) & 1u;
                const bool has_out = (c.leave >> i) & 1u;
                const uint32_t jo = (c.jout >> (4 * i)) & 7u;
                const uint32_t L = Lrow[jo];
                const uint32_t idx = has_out ? jo * 9u + L : (valid ? 72u : 73u);
                const uint4 e = *reinterpret_cast<const uint4 *>(wl8->g[idx]);
                const uint32_t b0 = has_in ? (0xC0u | (i << 3) | ((c.jin >> (4 * i)) & 7u))
                                           : (valid ? (0x40u | i) : 0u);
                const uint64_t glo = ((uint64_t)e.y << 32 | e.x) | b0 | (has_out ? (uint32_t)i << 11 : 0u);
                const uint64_t ghi = e.z;
                const uint32_t sh = 8u * (uint32_t)pos;
                s.w[0] |= shl64(glo, sh);
                s.w[Seq<K>::NW - 1] |= (sh >= 64u) ? shl64(glo, sh - 64u) : (shr64(glo, 64u - sh) | shl64(ghi, sh));
                pos += (int)e.w;
            }
        } else {
            pos = walk_bits<K>(c.valid, c.enter, c.leave, c.jin, c.jout, in2, s);
        }
        if (pos == 0 && in2 == KMASK) {  // p2 inside p1: all FromP2, in order
            if (K == 4) s.w[0] = 0x83828180ull;
            else { s.w[0] = 0x8786858483828180ull; s.w[Seq<K>::NW - 1] = 0; }
            pos = K;
        }
        // The walk from p1's edge 0 IS the canonical order (R3: start at the first
        // vertex along p1's boundary from v0; FromP2(0) when p2 lies inside p1).
        const bool cand = !c.sep && pos >= 3 && pos <= 2 * K;
        out.thin = THIN && cand && pair_is_thin(R2, (A1x2 + A2x2) - Aix2);
        nonempty = nonempty && cand;
        if (nonempty || out.thin) {
            out.seq = s;
            out.nx = pos;
        }
    }
    if (nonempty) {
        const float Aux2 = (A1x2 + A2x2) - Aix2;
        out.iou = (Aux2 > 0.f) ? iou_div(Aix2, Aux2) : 0.f;
        out.Aix2 = Aix2;
    }
    return out;
}

// The IoU of a thin pair for the pairwise evaluators (their clip records no flags):
// out of line (rare; the evaluators are at their register budget) — the clip again
// with the flag walk from the raw vertices (px[k], py[k]: p1 = the row, qx, qy: p2 =
// the column; global or shared memory), then the areas of the recorded
// intersection in double (dgal_exact.cuh), as the split forward does.
template <int K>
__device__ __noinline__ float pair_iou_exact(const float *px, const float *py, const float *qx, const float *qy)
{
    Poly<K> P, Q;
    const float ox = px[0], oy = py[0];
#pragma unroll
    for (int k = 0; k < K; ++k) {
        P.x[k] = __fsub_rn(px[k], ox); P.y[k] = __fsub_rn(py[k], oy);
        Q.x[k] = __fsub_rn(qx[k], ox); Q.y[k] = __fsub_rn(qy[k], oy);
    }
    P.x[0] = 0.f;
    P.y[0] = 0.f;
    FwdOut<K, true> r = iou_fwd<K, true, kP2Regs, true>(P, Q);
    if (r.thin || r.nx > 0) fwd_thin_redo<K>(RawPolyVerts{px, py, qx, qy}, r.seq, r.nx, r.iou);
    return r.iou;
}

// ---------------------------------------------------------------------------
// fused IoU forward + backward for a loss whose dL/dIoU is known up front
// (e.g. L = mean(1 - IoU) has dL/dIoU = -1/n)
// ---------------------------------------------------------------------------
// The gradient uses the very intervals the forward computes (no xflags round
// trip, no crossing recomputation): dA_i/dv_i += n_i ∫(1-t)dt, dA_i/dv_i+1 +=
// n_i ∫t dt over each boundary piece, then the S:303 chain.
// p1, p2 recentred on p1.v0.  Returns IoU (identical to the pairwise path).
// need (when given): the float result may miss the tolerance — a nearly parallel
// (p1 edge, p2 edge) pair (crossing parameters conditioned by 1/sin) or a thin pair
// (area sum conditioned by R^2 / A_u) — and the caller must have the pair redone by
// the exact split path (the fused kernels' refine pass).
template <int K, int MODE = kP2Pieces, bool PK = false, int ILLG = -1>
__device__ __forceinline__ float iou_fused(const Poly<K> &P, const Poly<K> &Q, float g, Poly<K> &G1,
                                           Poly<K> &G2, const Extrude ex = flat(), VolCoef *co = nullptr,
                                           QTable qt = QTable{nullptr, nullptr, 0}, bool *need = nullptr,
                                           IllTab it = IllTab{nullptr, 0})
{
#pragma unroll
    for (int k = 0; k < K; ++k) { G1.x[k] = 0.f; G1.y[k] = 0.f; G2.x[k] = 0.f; G2.y[k] = 0.f; }
    if (co) *co = VolCoef{0.f, 0.f, 0.f, 0.f, 0.f};
    if (need) *need = false;
    Clip<K> c;
    if (need) clip_intervals<K, MODE, true, ILLG>(P, Q, c, qt, nullptr, it);
    else clip_intervals<K, MODE, false>(P, Q, c, qt);
    const float R2 = need ? pair_extent2<K>(P, Q) : 0.f;   // (after the clip: not live through it)
    if (!c.nonempty) {
        // a thin pair's float area may be <= 0 although p1 and p2 overlap: the refine
        // pass decides (when the pair is not separated and has a boundary piece)
        if (need) *need = !c.sep && (c.valid | c.in2) != 0u && pair_is_thin(R2, (c.A1x2 + c.A2x2) - c.Aix2);
        return 0.f;
    }
    if (need) *need = c.ill || pair_is_thin(R2, (c.A1x2 + c.A2x2) - c.Aix2);
    // V = A d (2D: d = 1); IoU = V_i / V_u
    const float Vix2 = c.Aix2 * ex.dz;
    const float Vux2 = (c.A1x2 * ex.d1 + c.A2x2 * ex.d2) - Vix2;
    if (!(Vux2 > 0.f) || !(Vix2 > 0.f)) return 0.f;
    const float iou = iou_div(Vix2, Vux2);

    if constexpr (PK && (DGAL_F32X2 & 4)) {
        // the same weights and gradients with (p1, p2) quantities in paired FP32
        const float *ax = c.ax, *ay = c.ay, *bx = c.bx, *by = c.by;
        const uint64_t half2 = f2pack(0.5f, 0.5f);
        uint64_t AL[K], BE[K];
#pragma unroll
        for (int i = 0; i < K; ++i) {
            const float fx = c.fx[i], fy = c.fy[i];
            const float inv = rcp_approx(fmaf(fx, fx, fy * fy));
            const uint64_t dx = f2sub(f2pack(ax[i], bx[i]), f2pack(Q.x[i], Q.x[i]));
            const uint64_t dy = f2sub(f2pack(ay[i], by[i]), f2pack(Q.y[i], Q.y[i]));
            float s0, s1;
            f2unpack(f2mul(f2fma(dx, f2pack(fx, fx), f2mul(dy, f2pack(fy, fy))), f2pack(inv, inv)), s0, s1);
            const uint64_t T0 = f2pack(__saturatef(c.t0[i]), __saturatef(s0));
            const uint64_t T1 = f2pack(__saturatef(c.t1[i]), __saturatef(s1));
            float d1, d2;
            f2unpack(f2sub(T1, T0), d1, d2);
            const uint64_t L = f2pack(fmaxf(d1, 0.f), ((c.on2 >> i) & 1u) ? fmaxf(d2, 0.f) : 0.f);
            BE[i] = f2mul(L, f2mul(f2add(T0, T1), half2));
            AL[i] = f2sub(L, BE[i]);
        }
        const float Vi = 0.5f * Vix2, Vu = 0.5f * Vux2;
    const float inv = rcp_refined(Vu);   // 1 / V_u to ~1 ulp (V_u normal, > 0)
        const float q = Vi * inv;
        const float cvi = g * ((1.f + q) * inv);
        const float cvu = g * (-q * inv);
        const float ci = cvi * ex.dz;
        const float hu1 = (0.5f * cvu) * ex.d1, hu2 = (0.5f * cvu) * ex.d2;
        if (co) *co = VolCoef{cvi, cvu, 0.5f * c.Aix2, 0.5f * c.A1x2, 0.5f * c.A2x2};
        const uint64_t CI = f2pack(ci, ci), HU = f2pack(hu1, hu2);
        uint64_t EY[K], NX[K];
#pragma unroll
        for (int k = 0; k < K; ++k) {
            EY[k] = f2pack(c.gy[k], c.fy[k]);
            NX[k] = f2sub(0ull, f2pack(c.gx[k], c.fx[k]));
        }
#pragma unroll
        for (int k = 0; k < K; ++k) {
            const int km = (k + K - 1) % K;
            const uint64_t WA = f2fma(CI, AL[k], HU), WB = f2fma(CI, BE[km], HU);
            f2unpack(f2fma(WA, EY[k], f2mul(WB, EY[km])), G1.x[k], G2.x[k]);
            f2unpack(f2fma(WA, NX[k], f2mul(WB, NX[km])), G1.y[k], G2.y[k]);
        }
        return iou;
    }
    // piece weights (saturate: dead edges carry arbitrary end points, length 0)
    // p2 pieces: parameters of their end points (the crossing points of the p1
    // side) along the edge (projection; exact 0 at w_j)
    const float *ax = c.ax, *ay = c.ay, *bx = c.bx, *by = c.by;
    float al1[K], be1[K], al2[K], be2[K];
#pragma unroll
    for (int i = 0; i < K; ++i) {
        const float a0 = __saturatef(c.t0[i]), a1 = __saturatef(c.t1[i]);
        const float inv = rcp_approx(fmaf(c.fx[i], c.fx[i], c.fy[i] * c.fy[i]));
        const float b0 = __saturatef(fmaf(ax[i] - Q.x[i], c.fx[i], (ay[i] - Q.y[i]) * c.fy[i]) * inv);
        const float b1 = __saturatef(fmaf(bx[i] - Q.x[i], c.fx[i], (by[i] - Q.y[i]) * c.fy[i]) * inv);
        const float l1 = fmaxf(a1 - a0, 0.f);
        const float l2 = ((c.on2 >> i) & 1u) ? fmaxf(b1 - b0, 0.f) : 0.f;
        const float h1 = 0.5f * (a0 + a1), h2 = 0.5f * (b0 + b1);
        al1[i] = l1 - l1 * h1; be1[i] = l1 * h1;
        al2[i] = l2 - l2 * h2; be2[i] = l2 * h2;
    }
    // dIoU/dV_i = (V_u + V_i)/V_u^2, dIoU/dV_1,2 = -V_i/V_u^2; dV/dA = d
    const float Vi = 0.5f * Vix2, Vu = 0.5f * Vux2;
    const float inv = rcp_refined(Vu);   // 1 / V_u to ~1 ulp (V_u normal, > 0)
    const float q = Vi * inv;
    const float cvi = g * ((1.f + q) * inv);
    const float cvu = g * (-q * inv);
    const float ci = cvi * ex.dz;
    const float hu1 = (0.5f * cvu) * ex.d1, hu2 = (0.5f * cvu) * ex.d2;
    if (co) *co = VolCoef{cvi, cvu, 0.5f * c.Aix2, 0.5f * c.A1x2, 0.5f * c.A2x2};
#pragma unroll
    for (int k = 0; k < K; ++k) {
        const int km = (k + K - 1) % K;
        const float wa1 = fmaf(ci, al1[k], hu1), wb1 = fmaf(ci, be1[km], hu1);
        const float wa2 = fmaf(ci, al2[k], hu2), wb2 = fmaf(ci, be2[km], hu2);
        G1.x[k] = fmaf(wa1, c.gy[k], wb1 * c.gy[km]);
        G1.y[k] = -fmaf(wa1, c.gx[k], wb1 * c.gx[km]);
        G2.x[k] = fmaf(wa2, c.fy[k], wb2 * c.fy[km]);
        G2.y[k] = -fmaf(wa2, c.fx[k], wb2 * c.fx[km]);
    }
    return iou;
}

// ---------------------------------------------------------------------------
// backward: iou_grad through the recorded nx / xflags
// ---------------------------------------------------------------------------
// Flag-byte -> provenance bits, staged in shared memory by the kernel:
//   FromP1(i) -> bit i, FromP2(j) -> bit 8 + j,
//   Cross(i,j) -> bit 16 + i (p1 edge i has a crossing) | bit 24 + j (p2 edge j has one)
// (every other byte, including the 0x00 padding, maps to 0).
struct FlagLut {
    uint32_t v[256];
};

__device__ __forceinline__ void fill_flag_lut(FlagLut &L, int tid, int nthreads)
{
    for (int b = tid; b < 256; b += nthreads) {
        const int tag = b >> 6, i = (b >> 3) & 7, j = b & 7;
        L.v[b] = (tag == 1) ? (1u << j) : (tag == 2) ? (1u << (8 + j))
               : (tag == 3) ? ((1u << (16 + i)) | (1u << (24 + j))) : 0u;
    }
}

// Backward, split in three phases so a warp can share the crossing work:
//   bwd_prologue   (per pair)     default interval end points into the scratch;
//   bwd_crossing   (per Cross)    one recorded Cross(i, j): its two end points;
//   bwd_epilogue   (per pair)     pieces -> A_i -> dL/dv of p1 and p2.
// The scratch is per pair, transposed as [slot][TILE] so dynamic slots never
// conflict on banks: slot i = t0 of p1 edge i, K + i = t1, 2K + j = s0 of p2
// edge j, 3K + j = s1.  Inputs are read raw from shared memory (vertex
// differences of one scene are exact by Sterbenz; the crossing parameters only
// need differences); the epilogue recentres on p1.v0 for the shoelace terms.
template <int K, int TILE>
__device__ __forceinline__ void bwd_prologue(float *scr)
{
#pragma unroll
    for (int k = 0; k < K; ++k) {
        scr[k * TILE] = 0.f;
        scr[(K + k) * TILE] = 1.f;
        scr[(2 * K + k) * TILE] = 0.f;
        scr[(3 * K + k) * TILE] = 1.f;
    }
}

// Cross(i, j) is X = v_i + t g_i = w_j + s f_j.  If p1 edge i enters p2 there the
// boundary piece on p1 edge i starts at t and the piece on p2 edge j ends at s;
// if it exits, the other way round.  s is the projection of the same point X onto
// p2 edge j, so the two pieces meeting at X share it.
//
// Precision: t is conditioned by 1/sin of the crossing angle.  bwd_crossing (float)
// serves well-conditioned crossings — there the entry/exit role is the sign of
// g_i x f_j, which the forward's classification agrees with — and reports the
// others (|sin| < 2^-10).  bwd_crossing_exact recomputes those with the numerators /
// denominators in double (differences and products of the float inputs are exact
// there: ~1e-7 relative accuracy instead of ~6e-8/sin), and takes the role from
// the forward's own float decision values for that (edge, line), recomputed
// bitwise-identically (same recentring, same contraction-free expressions): for
// nearly parallel edges the true sign and the forward's could disagree, and the
// gradient must differentiate the boundary the forward recorded.
constexpr float kRefineSin = 0.0009765625f;   // 2^-10: float t error ~6e-8/sin <= 6e-5 above it
#ifndef DGAL_BWD_REFINE
#define DGAL_BWD_REFINE 1     // exact second pass for ill-conditioned crossings
#endif

template <int K, int TILE>
__device__ __forceinline__ bool bwd_crossing(const float *sPx, const float *sPy, const float *sQx,
                                             const float *sQy, uint32_t b, float *scr,
                                             float refine_sin = kRefineSin)
{
    const int i = (b >> 3) & (K - 1), j = b & (K - 1);
    const int i1 = (i + 1) & (K - 1), j1 = (j + 1) & (K - 1);
    const float vx = sPx[i], vy = sPy[i];
    const float ex = sPx[i1] - vx, ey = sPy[i1] - vy;
    const float wx = sQx[j], wy = sQy[j];
    const float hx = sQx[j1] - wx, hy = sQy[j1] - wy;
    const float Dx = wx - vx, Dy = wy - vy;
    const float den = ex * hy - ey * hx;                       // g_i x f_j
    const float r = rcp_approx(den);
    const float t = __saturatef((Dx * hy - Dy * hx) * r);      // along p1 edge i
    const float hh = fmaf(hx, hx, hy * hy);
    const float s = __saturatef(fmaf(fmaf(t, ex, -Dx), hx, fmaf(t, ey, -Dy) * hy) * rcp_approx(hh));
    const bool enter = den < 0.f;
    DGAL_ASSERT(i >= 0 && i < K && j >= 0 && j < K);
    // ill-conditioned (den^2 < sin^2 |e|^2 |h|^2): left to bwd_crossing_exact
    const bool need = DGAL_BWD_REFINE && (den * den < (refine_sin * refine_sin) * fmaf(ex, ex, ey * ey) * hh);
    if (!need) {
        scr[(enter ? i : K + i) * TILE] = t;
        scr[(enter ? 3 * K + j : 2 * K + j) * TILE] = s;
    }
    return need;
}

// Exact geometry for bwd_crossing_exact: vertices i, i+1 of p1 and j, j+1 of p2 of
// the pair at tile slot pt, in double.  Polygon path: the staged float tile IS
// the input, so its values are exact.
template <int K>
struct TileGeometry {
    static constexpr float kRefine = kRefineSin;   // |sin| below which a crossing is redone in double
    const float *x1, *y1, *x2, *y2;   // tile bases, [pair][k]
    __device__ __forceinline__ void get(int pt, int i, int i1, int j, int j1, double &vx, double &vy,
                                        double &v1x, double &v1y, double &wx, double &wy, double &w1x,
                                        double &w1y) const
    {
        vx = x1[pt * K + i]; vy = y1[pt * K + i]; v1x = x1[pt * K + i1]; v1y = y1[pt * K + i1];
        wx = x2[pt * K + j]; wy = y2[pt * K + j]; w1x = x2[pt * K + j1]; w1y = y2[pt * K + j1];
    }
    // all vertices of the pair, for the exact area of a thin pair (dgal_exact.cuh)
    __device__ __forceinline__ RawPolyVerts verts(int pt) const
    {
        return RawPolyVerts{x1 + pt * K, y1 + pt * K, x2 + pt * K, y2 + pt * K};
    }
};

template <int K, int TILE, class GEO>
__device__ __forceinline__ void bwd_crossing_exact(const float *sPx, const float *sPy, const float *sQx,
                                                   const float *sQy, uint32_t b, float *scr, const GEO &geo,
                                                   int pt)
{
    const int i = (b >> 3) & (K - 1), j = b & (K - 1);
    const int i1 = (i + 1) & (K - 1), j1 = (j + 1) & (K - 1);
    // the forward's class of line j for edge i: the sign of d[i][j] - d[i+1][j]
    // on the recentred coordinates (clip_intervals), bitwise the same floats
    const float ox = sPx[0], oy = sPy[0];
    const float pxi = __fsub_rn(sPx[i], ox), pyi = __fsub_rn(sPy[i], oy);
    const float pxi1 = __fsub_rn(sPx[i1], ox), pyi1 = __fsub_rn(sPy[i1], oy);
    const float qxj = __fsub_rn(sQx[j], ox), qyj = __fsub_rn(sQy[j], oy);
    const float qxj1 = __fsub_rn(sQx[j1], ox), qyj1 = __fsub_rn(sQy[j1], oy);
    const float fxj = qxj1 - qxj, fyj = qyj1 - qyj;
    const float da = __fadd_rn(cross_rn(fxj, fyj, __fsub_rn(i == 0 ? 0.f : pxi, qxj),
                                        __fsub_rn(i == 0 ? 0.f : pyi, qyj)), kTiny);
    const float db = __fadd_rn(cross_rn(fxj, fyj, __fsub_rn(i1 == 0 ? 0.f : pxi1, qxj),
                                        __fsub_rn(i1 == 0 ? 0.f : pyi1, qyj)), kTiny);
    const bool enter = __saturatef(-((da - db) + kTiny) * kBig) > 0.5f;
    // the crossing in double on the exact geometry
    double vx, vy, v1x, v1y, wx, wy, w1x, w1y;
    geo.get(pt, i, i1, j, j1, vx, vy, v1x, v1y, wx, wy, w1x, w1y);
    const double ex = v1x - vx, ey = v1y - vy;
    const double hx = w1x - wx, hy = w1y - wy;
    const double Dx = wx - vx, Dy = wy - vy;
    const double den = ex * hy - ey * hx;
    const double tn = Dx * hy - Dy * hx;
    const float t = __saturatef((float)tn * rcp_approx((float)den));
    const double tt = t;
    const double sn = (tt * ex - Dx) * hx + (tt * ey - Dy) * hy;       // (X - w_j) . f_j
    const double hh = hx * hx + hy * hy;
    const float s = __saturatef((float)sn * rcp_approx((float)hh));
    scr[(enter ? i : K + i) * TILE] = t;
    scr[(enter ? 3 * K + j : 2 * K + j) * TILE] = s;
}

// V = OR of the flag table over the recorded bytes (vertex / crossing provenance).
// Returns whether the pair is thin (pair_is_thin on its float areas): then the
// caller recomputes the intersection's area in double and calls again with twice
// it in *ovr, which replaces the float sum in the S:303 coefficients (the piece
// weights stay the float ones: they need ~1e-7, not 1e-16; so do A_1, A_2, whose
// float sums are accurate to ~eps R^2 / A — only a sliver intersection's is not).
// OVR3: *ovr holds {A_i, A_1, A_2} (twice each), all three replacing the float sums.
template <int K, int TILE, bool PK = false, bool OVR3 = false>
__device__ __forceinline__ bool bwd_epilogue(const float *sPx, const float *sPy, const float *sQx,
                                             const float *sQy, float g, uint32_t V, const float *scr,
                                             Poly<K> &G1, Poly<K> &G2, const Extrude ex = flat(),
                                             VolCoef *co = nullptr, const float *ovr = nullptr)
{
#pragma unroll
    for (int k = 0; k < K; ++k) { G1.x[k] = 0.f; G1.y[k] = 0.f; G2.x[k] = 0.f; G2.y[k] = 0.f; }
    if (co) *co = VolCoef{0.f, 0.f, 0.f, 0.f, 0.f};
    if (V == 0) return false;  // nx == 0: zero subgradient
    bool thin = false;

    if constexpr (PK && (DGAL_F32X2 & 4)) {
    // paired FP32 along (p1, p2): X[k] = (v_k.x, w_k.x), Y[k] = (v_k.y, w_k.y) recentred
    // on v_0; edge vectors EX/EY = (g, f), their negatives NX, shoelace terms C =
    // (C1, C2); every per-edge / per-vertex quantity below is a (p1, p2) pair
    uint64_t X[K], Y[K];
    {
        const float ox = sPx[0], oy = sPy[0];
        const uint64_t o2x = f2pack(ox, ox), o2y = f2pack(oy, oy);
#pragma unroll
        for (int k = 0; k < K; ++k) {
            X[k] = f2sub(f2pack(sPx[k], sQx[k]), o2x);
            Y[k] = f2sub(f2pack(sPy[k], sQy[k]), o2y);
        }
    }
    uint64_t EY[K], NX[K], C[K], A12 = 0ull;
#pragma unroll
    for (int i = 0; i < K; ++i) {
        const int i1 = (i + 1) % K;
        EY[i] = f2sub(Y[i1], Y[i]);
        NX[i] = f2sub(X[i], X[i1]);
        C[i] = f2fma(X[i], Y[i1], f2sub(0ull, f2mul(X[i1], Y[i])));
        A12 = f2add(A12, C[i]);
    }
    float A1x2, A2x2;
    f2unpack(A12, A1x2, A2x2);

    // boundary pieces -> A_i and the edge weights
    //   alpha = ∫ (1-t) dt = l (1 - h),  beta = ∫ t dt = l h,  l = t1 - t0, h = (t0 + t1)/2
    // (edge i on the boundary, as masks: vertex i, vertex i+1 (rotated) or a crossing)
    constexpr uint32_t KMASK = (1u << K) - 1u;
    const uint32_t v1 = V & KMASK, v2 = (V >> 8) & KMASK;
    const uint32_t on1m = v1 | ((v1 >> 1) | (v1 << (K - 1))) | (V >> 16);
    const uint32_t on2m = v2 | ((v2 >> 1) | (v2 << (K - 1))) | (V >> 24);
    uint64_t AL[K], BE[K], AIX = 0ull;
    const uint64_t half2 = f2pack(0.5f, 0.5f);
#pragma unroll
    for (int i = 0; i < K; ++i) {
        const uint64_t T0 = f2pack(scr[i * TILE], scr[(2 * K + i) * TILE]);
        const uint64_t T1 = f2pack(scr[(K + i) * TILE], scr[(3 * K + i) * TILE]);
        float d1, d2;
        f2unpack(f2sub(T1, T0), d1, d2);
        const uint64_t L = f2pack(((on1m >> i) & 1u) ? fmaxf(d1, 0.f) : 0.f, ((on2m >> i) & 1u) ? fmaxf(d2, 0.f) : 0.f);
        const uint64_t H = f2mul(f2add(T0, T1), half2);
        BE[i] = f2mul(L, H);
        AL[i] = f2sub(L, BE[i]);
        AIX = f2fma(L, C[i], AIX);
    }
    float ai1, ai2;
    f2unpack(AIX, ai1, ai2);
    float Aix2 = ai1 + ai2;
    if (ovr) {
        Aix2 = ovr[0];
        if (OVR3) { A1x2 = ovr[1]; A2x2 = ovr[2]; }
    } else if (DGAL_THIN_BWD) {
        // the piece sum's rounding is bounded by ~2 eps sum_k (|v_k|^2 + |w_k|^2)
        // (|x y'| <= (x^2 + y'^2) / 2 for each product of each shoelace term)
        uint64_t S2 = 0ull;
#pragma unroll
        for (int k = 0; k < K; ++k) S2 = f2fma(X[k], X[k], f2fma(Y[k], Y[k], S2));
        float s1_, s2_;
        f2unpack(S2, s1_, s2_);
        thin = pair_is_thin_sum<K>(s1_ + s2_, (A1x2 + A2x2) - Aix2);
    }

    // dIoU/dV_i = (V_u + V_i)/V_u^2, dIoU/dV_1,2 = -V_i/V_u^2; V = A d (2D: d = 1)
    const float Ai = 0.5f * Aix2;
    const float Vi = Ai * ex.dz;
    const float Vu = 0.5f * ((A1x2 * ex.d1 + A2x2 * ex.d2) - Aix2 * ex.dz);
    if (!(Vu > 0.f) || !(Vi > 0.f)) return thin;  // R10 guard
    const float inv = rcp_refined(Vu);   // 1 / V_u to ~1 ulp (V_u normal, > 0)
    const float q = Vi * inv;
    const float cvi = g * ((1.f + q) * inv);
    const float cvu = g * (-q * inv);
    const float ci = cvi * ex.dz;
    // area_grad of p1/p2 is (n_k + n_k-1)/2 per vertex
    const float hu1 = (0.5f * cvu) * ex.d1, hu2 = (0.5f * cvu) * ex.d2;
    if (co) *co = VolCoef{cvi, cvu, Ai, 0.5f * A1x2, 0.5f * A2x2};

    // vertex k collects edge k (as its start, alpha) and edge k-1 (as its end, beta);
    // n = perp(edge) = (e_y, -e_x)
    const uint64_t CI = f2pack(ci, ci), HU = f2pack(hu1, hu2);
#pragma unroll
    for (int k = 0; k < K; ++k) {
        const int km = (k + K - 1) % K;
        const uint64_t WA = f2fma(CI, AL[k], HU), WB = f2fma(CI, BE[km], HU);
        f2unpack(f2fma(WA, EY[k], f2mul(WB, EY[km])), G1.x[k], G2.x[k]);
        f2unpack(f2fma(WA, NX[k], f2mul(WB, NX[km])), G1.y[k], G2.y[k]);
    }
    } else {
    Poly<K> P, Q;
    {
        const float ox = sPx[0], oy = sPy[0];
#pragma unroll
        for (int k = 0; k < K; ++k) {
            P.x[k] = sPx[k] - ox; P.y[k] = sPy[k] - oy;
            Q.x[k] = sQx[k] - ox; Q.y[k] = sQy[k] - oy;
        }
        P.x[0] = 0.f;   // exact for finite input; lets the compiler fold it
        P.y[0] = 0.f;
    }
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

    // boundary pieces -> A_i and the edge weights
    //   alpha = ∫ (1-t) dt = l (1 - h),  beta = ∫ t dt = l h,  l = t1 - t0, h = (t0 + t1)/2
    // p1 edge i is on the boundary iff v_i or v_i+1 is a vertex of p1 ∩ p2 or it is crossed
    // (edge i on the boundary, as masks: vertex i, vertex i+1 (rotated) or a crossing)
    constexpr uint32_t KMASK = (1u << K) - 1u;
    const uint32_t v1 = V & KMASK, v2 = (V >> 8) & KMASK;
    const uint32_t on1m = v1 | ((v1 >> 1) | (v1 << (K - 1))) | (V >> 16);
    const uint32_t on2m = v2 | ((v2 >> 1) | (v2 << (K - 1))) | (V >> 24);
    float al1[K], be1[K], al2[K], be2[K];
    float Aix2 = 0.f;
#pragma unroll
    for (int i = 0; i < K; ++i) {
        const bool on1 = (on1m >> i) & 1u;
        const bool on2 = (on2m >> i) & 1u;
        const float a0 = scr[i * TILE], a1 = scr[(K + i) * TILE];
        const float b0 = scr[(2 * K + i) * TILE], b1 = scr[(3 * K + i) * TILE];
        const float l1 = on1 ? fmaxf(a1 - a0, 0.f) : 0.f;
        const float l2 = on2 ? fmaxf(b1 - b0, 0.f) : 0.f;
        const float h1 = 0.5f * (a0 + a1), h2 = 0.5f * (b0 + b1);
        al1[i] = l1 - l1 * h1; be1[i] = l1 * h1;
        al2[i] = l2 - l2 * h2; be2[i] = l2 * h2;
        Aix2 = fmaf(l1, C1[i], Aix2);
        Aix2 = fmaf(l2, C2[i], Aix2);
    }
    if (ovr) {
        Aix2 = ovr[0];
        if (OVR3) { A1x2 = ovr[1]; A2x2 = ovr[2]; }
    } else if (DGAL_THIN_BWD) {
        float sq = 0.f;
#pragma unroll
        for (int k = 0; k < K; ++k) sq = fmaf(P.x[k], P.x[k], fmaf(P.y[k], P.y[k], fmaf(Q.x[k], Q.x[k], fmaf(Q.y[k], Q.y[k], sq))));
        thin = pair_is_thin_sum<K>(sq, (A1x2 + A2x2) - Aix2);
    }

    // dIoU/dV_i = (V_u + V_i)/V_u^2, dIoU/dV_1,2 = -V_i/V_u^2; V = A d (2D: d = 1)
    const float Ai = 0.5f * Aix2;
    const float Vi = Ai * ex.dz;
    const float Vu = 0.5f * ((A1x2 * ex.d1 + A2x2 * ex.d2) - Aix2 * ex.dz);
    if (!(Vu > 0.f) || !(Vi > 0.f)) return thin;  // R10 guard
    const float inv = rcp_refined(Vu);   // 1 / V_u to ~1 ulp (V_u normal, > 0)
    const float q = Vi * inv;
    const float cvi = g * ((1.f + q) * inv);
    const float cvu = g * (-q * inv);
    const float ci = cvi * ex.dz;
    // area_grad of p1/p2 is (n_k + n_k-1)/2 per vertex
    const float hu1 = (0.5f * cvu) * ex.d1, hu2 = (0.5f * cvu) * ex.d2;
    if (co) *co = VolCoef{cvi, cvu, Ai, 0.5f * A1x2, 0.5f * A2x2};

    // vertex k collects edge k (as its start, alpha) and edge k-1 (as its end, beta);
    // n = perp(edge) = (e_y, -e_x)
#pragma unroll
    for (int k = 0; k < K; ++k) {
        const int km = (k + K - 1) % K;
        const float wa1 = fmaf(ci, al1[k], hu1), wb1 = fmaf(ci, be1[km], hu1);
        const float wa2 = fmaf(ci, al2[k], hu2), wb2 = fmaf(ci, be2[km], hu2);
        G1.x[k] = fmaf(wa1, gy[k], wb1 * gy[km]);
        G1.y[k] = -fmaf(wa1, gx[k], wb1 * gx[km]);
        G2.x[k] = fmaf(wa2, fy[k], wb2 * fy[km]);
        G2.y[k] = -fmaf(wa2, fx[k], wb2 * fx[km]);
    }
    }
    return thin;
}

// The 2D epilogue in double, for a thin pair (bwd_pair_exact): its vertex gradients
// are small differences of the intersection and union terms, each ~g L / A_u (L the
// pair's extent), which float rounds to ~eps g L^2 / A_u — up to 1e-4 absolute at
// aspect 300.  Same formulas as bwd_epilogue, every quantity in double (the interval
// end points are the float ones, exact in double); the areas are the exact ones.
template <int K, int TILE>
__device__ __forceinline__ void bwd_epilogue_exact(const float *sPx, const float *sPy, const float *sQx,
                                                   const float *sQy, float g, uint32_t V, const float *scr,
                                                   const AreasX2 &ar, Poly<K> &G1, Poly<K> &G2)
{
#pragma unroll
    for (int k = 0; k < K; ++k) { G1.x[k] = 0.f; G1.y[k] = 0.f; G2.x[k] = 0.f; G2.y[k] = 0.f; }
    if (V == 0) return;
    constexpr uint32_t KMASK = (1u << K) - 1u;
    const uint32_t v1 = V & KMASK, v2 = (V >> 8) & KMASK;
    const uint32_t on1m = v1 | ((v1 >> 1) | (v1 << (K - 1))) | (V >> 16);
    const uint32_t on2m = v2 | ((v2 >> 1) | (v2 << (K - 1))) | (V >> 24);
    const double Ai = 0.5 * ar.ai, Au = 0.5 * ((ar.a1 + ar.a2) - ar.ai);
    if (!(Au > 0.0) || !(Ai > 0.0)) return;  // R10 guard
    const double inv = 1.0 / Au, q = Ai * inv;
    const double ci = (double)g * ((1.0 + q) * inv);    // dL/dA_i
    const double hu = 0.5 * ((double)g * (-q * inv));  // dL/dA_1,2 times 1/2 (area_grad)
    // piece weights of edge i: alpha = l (1 - h), beta = l h (p1: which = 0, p2: 1),
    // recomputed per use (no arrays: the caller's loop is at its register budget)
    auto wts = [&](int which, int i, double &alpha, double &beta) {
        const double t0 = scr[(2 * K * which + i) * TILE], t1 = scr[(2 * K * which + K + i) * TILE];
        const uint32_t on = which ? on2m : on1m;
        const double l = ((on >> i) & 1u) ? fmax(t1 - t0, 0.0) : 0.0;
        beta = l * (0.5 * (t0 + t1));
        alpha = l - beta;
    };
#pragma unroll 1
    for (int k = 0; k < K; ++k) {
        const int km = (k + K - 1) % K, k1 = (k + 1) % K;
        double al, be, bem, alm;
        // p1 vertex k: edge k (as its start, alpha) and edge k-1 (as its end, beta)
        wts(0, k, al, be);
        wts(0, km, alm, bem);
        const double gxk = (double)sPx[k1] - sPx[k], gyk = (double)sPy[k1] - sPy[k];
        const double gxm = (double)sPx[k] - sPx[km], gym = (double)sPy[k] - sPy[km];
        double wa = ci * al + hu, wb = ci * bem + hu;
        const float g1x = (float)(wa * gyk + wb * gym), g1y = (float)(-(wa * gxk + wb * gxm));
        wts(1, k, al, be);
        wts(1, km, alm, bem);
        const double fxk = (double)sQx[k1] - sQx[k], fyk = (double)sQy[k1] - sQy[k];
        const double fxm = (double)sQx[k] - sQx[km], fym = (double)sQy[k] - sQy[km];
        wa = ci * al + hu;
        wb = ci * bem + hu;
        const float g2x = (float)(wa * fyk + wb * fym), g2y = (float)(-(wa * fxk + wb * fxm));
        // (a dynamic k: write through the unrolled selects of the register arrays)
#pragma unroll
        for (int q = 0; q < K; ++q) {
            if (q == k) { G1.x[q] = g1x; G1.y[q] = g1y; G2.x[q] = g2x; G2.y[q] = g2y; }
        }
    }
}

// One backward tile: thread tid owns pair tid of a tile of TILE pairs whose
// vertices are staged in shared memory as [pair][k] planes.  Decodes the pair's
// flag bytes into provenance bits, queues its Cross bytes in the warp's queue
// (warp prefix sum), evaluates the warp's crossings 32 at a time (full SIMT
// width), then runs the epilogue.  Must be called by all 32 lanes of the warp.
template <int K, int TILE, class GEO = TileGeometry<K>, bool PK = false>
__device__ __forceinline__ bool bwd_tile_pair(const float *tx1, const float *ty1, const float *tx2,
                                              const float *ty2, const Seq<K> &sq, int m, float g, bool live,
                                              float *scr, uint16_t *queue, const FlagLut &lut,
                                              Poly<K> &G1, Poly<K> &G2, const Extrude ex = flat(),
                                              VolCoef *co = nullptr, const GEO *geo = nullptr)
{
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    // the recorded bytes, masked to the first m once (the padding is 0x00 already;
    // the mask keeps a malformed record from reading past nx)
    Seq<K> w;
    int cnt = 0;
#pragma unroll
    for (int q = 0; q < Seq<K>::NW; ++q) {
        const int rem = m - 8 * q;
        const uint64_t keep = (rem >= 8) ? ~0ull : ((rem <= 0) ? 0ull : (shl64(1ull, 8u * (uint32_t)rem) - 1ull));
        w.w[q] = sq.w[q] & keep;
        // Cross bytes: tag bits 7 and 6 both set
        cnt += __popcll(w.w[q] & (w.w[q] << 1) & 0x8080808080808080ull);
    }
    uint32_t V = 0;
#pragma unroll
    for (int p = 0; p < 2 * K; ++p) V |= lut.v[seq_byte<K>(w, p)];

    // warp prefix sum of the counts (0 .. 2K) bit by bit: one ballot per bit, the bits
    // independent (a shuffle scan is a chain of five dependent shuffles: ncu put 8 % of
    // the backward's stall samples on it)
    const unsigned below = (1u << lane) - 1u;
    int at = 0, total = 0;
#pragma unroll
    for (int bit = 0; (1 << bit) <= 2 * K; ++bit) {
        const unsigned bb = __ballot_sync(0xFFFFFFFFu, (cnt >> bit) & 1);
        at += __popc(bb & below) << bit;
        total += __popc(bb) << bit;
    }
#pragma unroll
    for (int p = 0; p < 2 * K; ++p) {
        const uint32_t b = seq_byte<K>(w, p);
        if (b >= 0xC0u) {
            DGAL_ASSERT(at >= 0 && at < 32 * 2 * K);
            queue[at++] = (uint16_t)((lane << 8) | b);
        }
    }
    bwd_prologue<K, TILE>(scr + tid);
    __syncwarp();
    // pass 1 (float) over all crossings; the ill-conditioned ones are compacted in
    // place to the front of the queue (each write lands at or before the writer's
    // own, already consumed, slot)
    int nref = 0;
    for (int base = 0; base < total; base += 32) {   // warp-uniform trip count
        const int e = base + lane;
        bool need = false;
        uint32_t ent = 0;
        if (e < total) {
            DGAL_ASSERT(e < 32 * 2 * K);
            ent = queue[e];
            DGAL_ASSERT((int)(ent >> 8) < 32);
            const int pt = warp * 32 + (int)(ent >> 8);
            need = bwd_crossing<K, TILE>(tx1 + pt * K, ty1 + pt * K, tx2 + pt * K, ty2 + pt * K, ent & 0xFFu,
                                         scr + pt, GEO::kRefine);
        }
        const unsigned bal = __ballot_sync(0xFFFFFFFFu, need);
        if (bal) {
            __syncwarp();
            if (need) queue[nref + __popc(bal & ((1u << lane) - 1u))] = (uint16_t)ent;
            nref += __popc(bal);
            __syncwarp();
        }
    }
    // pass 2: exact recomputation of the compacted ones, 32 at a time
    for (int base = 0; base < nref; base += 32) {
        const int e = base + lane;
        if (e < nref) {
            const uint32_t ent = queue[e];
            const int pt = warp * 32 + (int)(ent >> 8);
            if (geo)
                bwd_crossing_exact<K, TILE, GEO>(tx1 + pt * K, ty1 + pt * K, tx2 + pt * K, ty2 + pt * K,
                                                 ent & 0xFFu, scr + pt, *geo, pt);
            else
                bwd_crossing_exact<K, TILE, TileGeometry<K>>(tx1 + pt * K, ty1 + pt * K, tx2 + pt * K,
                                                             ty2 + pt * K, ent & 0xFFu, scr + pt,
                                                             TileGeometry<K>{tx1, ty1, tx2, ty2}, pt);
        }
    }
    __syncwarp();
    bool thin = false;
    if (live)
        thin = bwd_epilogue<K, TILE, PK>(tx1 + tid * K, ty1 + tid * K, tx2 + tid * K, ty2 + tid * K, g, V, scr + tid,
                                         G1, G2, ex, co);
    return DGAL_THIN_BWD && thin;
}

// the recorded bytes masked to the first m, and their provenance bits (the flag table)
template <int K>
__device__ __forceinline__ uint32_t masked_record(Seq<K> &w, int m, const FlagLut &lut)
{
#pragma unroll
    for (int q = 0; q < Seq<K>::NW; ++q) {
        const int rem = m - 8 * q;
        w.w[q] &= (rem >= 8) ? ~0ull : ((rem <= 0) ? 0ull : (shl64(1ull, 8u * (uint32_t)rem) - 1ull));
    }
    uint32_t V = 0;
#pragma unroll
    for (int p = 0; p < 2 * K; ++p) V |= lut.v[seq_byte<K>(w, p)];
    return V;
}

// The whole backward of ONE pair by its own thread, every crossing in double and the
// intersection's area in double (areas_exact): the thin-pair redo of the per-thread
// backward kernel, run after its tile loop with the pair re-staged at tile slot pt
// (no warp cooperation, so it runs for the thin lanes only).
template <int K, int TILE, bool PK = false>
__device__ __forceinline__ void bwd_pair_exact(const float *tx1, const float *ty1, const float *tx2,
                                               const float *ty2, int pt, Seq<K> w, int m, float g, float *scr,
                                               const FlagLut &lut, Poly<K> &G1, Poly<K> &G2)
{
    const uint32_t V = masked_record<K>(w, m, lut);
    bwd_prologue<K, TILE>(scr + pt);
    const TileGeometry<K> geo{tx1, ty1, tx2, ty2};
#pragma unroll 1
    for (int p = 0; p < m && p < 2 * K; ++p) {
        const uint64_t ww = (K == 8 && p >= 8) ? w.w[Seq<K>::NW - 1] : w.w[0];
        const uint32_t b = (uint32_t)(ww >> (8 * (p & 7))) & 0xFFu;
        if (b >= 0xC0u)
            bwd_crossing_exact<K, TILE, TileGeometry<K>>(tx1 + pt * K, ty1 + pt * K, tx2 + pt * K, ty2 + pt * K, b,
                                                         scr + pt, geo, pt);
    }
    const AreasX2 a = areas_exact<K, true>(geo.verts(pt), w, m);
    bwd_epilogue_exact<K, TILE>(tx1 + pt * K, ty1 + pt * K, tx2 + pt * K, ty2 + pt * K, g, V, scr + pt, a, G1, G2);
}


// A thin pair (bwd_tile_pair returned true; rare): the area of the recorded
// intersection in double (dgal_exact.cuh), then the epilogue again with it.
// Called by the kernels AFTER they stored the first gradients (so those are dead
// here: no register pressure on the common path), before the tile's shared memory
// (vertices, interval scratch) is reused; the record is re-read by the caller
// (sq, m: as given to bwd_tile_pair).  Overwrites G1, G2 (and co).
// The vertices are the tile's floats (for boxes: the float corners; their rounding,
// ~eps L, moves a sliver's area by ~eps L W — relative ~eps; it is the float SUM,
// ~eps R^2, that is not accurate enough).
template <int K, int TILE, bool PK = false>
__device__ __forceinline__ void bwd_thin_redo(const float *tx1, const float *ty1, const float *tx2,
                                              const float *ty2, Seq<K> w, int m, float g, const float *scr,
                                              const FlagLut &lut, Poly<K> &G1, Poly<K> &G2,
                                              const Extrude ex = flat(), VolCoef *co = nullptr)
{
    const int tid = threadIdx.x;
    const uint32_t V = masked_record<K>(w, m, lut);
    const AreasX2 a = areas_exact<K, false>(TileGeometry<K>{tx1, ty1, tx2, ty2}.verts(tid), w, m);
    const float ovr = (float)a.ai;
    bwd_epilogue<K, TILE, PK>(tx1 + tid * K, ty1 + tid * K, tx2 + tid * K, ty2 + tid * K, g, V, scr + tid, G1, G2,
                              ex, co, &ovr);
}

}  // namespace dgal
