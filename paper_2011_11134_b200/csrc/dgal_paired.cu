// dgal_paired.cu — paired forward / backward kernels: one thread per
// pair, polygons and clip state in registers, float4 SoA streaming loads.
#include "dgal_core.cuh"
#include "dgal_internal.h"
#include "dgal_pipe.cuh"
#include "dgal_refine.cuh"

namespace dgal {

template <int K>
__device__ __forceinline__ void recentre(Poly<K> &P, Poly<K> &Q)
{
    // local origin o = p1.v0 (R11): IoU is translation invariant, and float
    // coordinates near 0 keep the decision predicates accurate.
    const float ox = P.x[0], oy = P.y[0];
    // (paired: vertices 2q, 2q+1 per sub.rn.f32x2, bitwise the scalar result)
    const uint64_t o2x = f2pack(ox, ox), o2y = f2pack(oy, oy);
#pragma unroll
    for (int q = 0; q < K / 2; ++q) {
        f2unpack(f2sub(f2pack(Q.x[2 * q], Q.x[2 * q + 1]), o2x), Q.x[2 * q], Q.x[2 * q + 1]);
        f2unpack(f2sub(f2pack(Q.y[2 * q], Q.y[2 * q + 1]), o2y), Q.y[2 * q], Q.y[2 * q + 1]);
        if (q > 0) {
            f2unpack(f2sub(f2pack(P.x[2 * q], P.x[2 * q + 1]), o2x), P.x[2 * q], P.x[2 * q + 1]);
            f2unpack(f2sub(f2pack(P.y[2 * q], P.y[2 * q + 1]), o2y), P.y[2 * q], P.y[2 * q + 1]);
        } else {
            P.x[1] = __fsub_rn(P.x[1], ox);
            P.y[1] = __fsub_rn(P.y[1], oy);
        }
    }
    // x - x == 0 for every finite x: stated as a constant so the compiler folds
    // the products with p1.v0 (fewer instructions and registers)
    P.x[0] = 0.f;
    P.y[0] = 0.f;
}

// Forward, one pair per thread, direct streaming loads.  The kernel is
// issue-bound (ncu: not_selected / math_pipe_throttle), so a persistent
// bulk-copy pipeline (tried: DESIGN.md §4.1) costs more in registers than the
// latency it hides; for K = 8 it also spills.
#ifndef DGAL_FWD4_MINB
#define DGAL_FWD4_MINB 7     // CTAs per SM the K=4 forward is register-budgeted for (72 registers,
                             // 31.5 KB shared: 7 fit; A/B after the events-without-selects diet:
                             // 0.3480 vs 0.3502 ms at 6, outputs bitwise equal)
#endif
#ifndef DGAL_FWD4_THREADS
#define DGAL_FWD4_THREADS 128
#endif
constexpr int kFwd4Threads = DGAL_FWD4_THREADS;

#ifndef DGAL_FWD4_WALKLUT
#define DGAL_FWD4_WALKLUT 1   // K = 4 flag walk + p2 inside mask from shared-memory tables
#endif

#ifndef DGAL_FWD_P2MODE
#define DGAL_FWD_P2MODE kP2Smem   // how the forward forms the p2 side (dgal_core.cuh P2Mode)
#endif

#ifndef DGAL_FWD4_NT
#define DGAL_FWD4_NT 8        // K = 4: consecutive tiles of T pairs per CTA (amortises the table fill)
#endif
#ifndef DGAL_FWD8_THREADS
#define DGAL_FWD8_THREADS 128   // K = 8 (A/B: 256 x 1 CTA 0.50 ms, 128 x 3 0.38 ms)
#endif
#ifndef DGAL_FWD8_MINB
#define DGAL_FWD8_MINB 4   // 128 registers, no spill since the WalkLut8 walk (A/B: 3 CTAs/SM 0.305 ms, 4: 0.301)
#endif
#ifndef DGAL_FWD8_NT
#define DGAL_FWD8_NT 4         // K = 8: 4 tiles per CTA with the cp.async prefetch (A/B: 0.373 -> 0.367 ms)
#endif
#ifndef DGAL_FWD8_WALKLUT
#define DGAL_FWD8_WALKLUT 1   // K = 8: the flag walk from WalkLut8 (dgal_core.cuh)
#endif
#ifndef DGAL_FWD8_PREFETCH
#define DGAL_FWD8_PREFETCH 1
#endif
constexpr int kFwd8Threads = DGAL_FWD8_THREADS;
#ifndef DGAL_FWD4_PREFETCH
#define DGAL_FWD4_PREFETCH 1  // K = 4: tile t+1 copied to shared memory (cp.async) while tile t computes
#endif

template <int K>
__global__ void __launch_bounds__((K == 4) ? kFwd4Threads : kFwd8Threads, (K == 4) ? DGAL_FWD4_MINB : DGAL_FWD8_MINB)
paired_fwd_direct_kernel(int64_t n, const float *__restrict__ x1, const float *__restrict__ y1,
                         const float *__restrict__ x2, const float *__restrict__ y2,
                         float *__restrict__ iou, uint8_t *__restrict__ nx, uint8_t *__restrict__ xflags)
{
    constexpr int T = (K == 4) ? kFwd4Threads : kFwd8Threads;
    constexpr bool WL = (K == 4) && DGAL_FWD4_WALKLUT;
    constexpr bool WL8 = (K == 8) && DGAL_FWD8_WALKLUT;
    constexpr int NT = (K == 4) ? DGAL_FWD4_NT : DGAL_FWD8_NT;
    // per-thread p2 vertex table (DGAL_FWD_P2MODE == kP2Smem, rows as QTable), [thread][slot]:
    // x at slots 0..K+1, y at K+2..2K+3; the zero slots K+1 and 2K+3 are written once.  An
    // odd per-thread stride kQS keeps the warp's accesses conflict-free and an event's
    // address one LEA
    constexpr int kQS = 2 * K + 5;
    __shared__ float sq[kQS * T];
    __shared__ WalkLut4 wlut[1];      // K = 4: the walk tables (DGAL_FWD4_WALKLUT; unused otherwise)
    __shared__ WalkLut8 wlut8[1];     // K = 8: the walk tables (DGAL_FWD8_WALKLUT; unused otherwise)
    constexpr bool PF = (K == 4) ? DGAL_FWD4_PREFETCH : DGAL_FWD8_PREFETCH;
    // PF: 2-stage per-thread ring [stage][plane][thread][K] (each thread copies and
    // reads only its own 64 bytes: no CTA barrier, cp.async groups order it)
    __shared__ __align__(16) float ring[PF ? 2 * 4 * T * K : 4];
    const int64_t k0 = (int64_t)blockIdx.x * (NT * T) + threadIdx.x;
    const int tid = threadIdx.x;
    auto prefetch = [&](int stage, int64_t k) {
        float *r = ring + stage * (4 * T * K) + tid * K;
#pragma unroll
        for (int q = 0; q < K / 4; ++q) {
            cp_async16(r + 4 * q, x1 + k * K + 4 * q);
            cp_async16(r + T * K + 4 * q, y1 + k * K + 4 * q);
            cp_async16(r + 2 * T * K + 4 * q, x2 + k * K + 4 * q);
            cp_async16(r + 3 * T * K + 4 * q, y2 + k * K + 4 * q);
        }
    };
    Poly<K> P, Q;
    if (PF) {
        if (k0 < n) prefetch(0, k0);
        cp_async_commit();
    } else if (k0 < n) {   // the first tile's loads go out before the table fill
        load_poly<K>(x1, y1, k0, P);
        load_poly<K>(x2, y2, k0, Q);
    }
    if (WL) {
        load_walk_lut4(wlut[0], threadIdx.x, T);
        __syncthreads();
    }
    if (WL8) {
        load_walk_lut8(wlut8[0], threadIdx.x, T);
        __syncthreads();
    }
    float *const sqt = sq + threadIdx.x * kQS;
    const QTable qt{sqt, sqt + K + 2, 1};
    sqt[K + 1] = 0.f;
    sqt[2 * K + 3] = 0.f;
    uint32_t thinmask = 0;   // tiles whose pair is thin (R^2 > kThinRatio A_u)
#pragma unroll 1
    for (int t = 0; t < NT; ++t) {
        const int64_t k = k0 + (int64_t)t * T;
        if (k >= n) break;
        if (PF) {
            if (t + 1 < NT && k + T < n) prefetch((t + 1) & 1, k + T);
            cp_async_commit();
            cp_async_wait<1>();   // this thread's copies of tile t have landed
            const float *r = ring + (t & 1) * (4 * T * K) + tid * K;
#pragma unroll
            for (int q = 0; q < K / 4; ++q) {
                const float4 u = *reinterpret_cast<const float4 *>(r + 4 * q);
                const float4 v = *reinterpret_cast<const float4 *>(r + T * K + 4 * q);
                const float4 w = *reinterpret_cast<const float4 *>(r + 2 * T * K + 4 * q);
                const float4 z = *reinterpret_cast<const float4 *>(r + 3 * T * K + 4 * q);
                P.x[4 * q] = u.x; P.x[4 * q + 1] = u.y; P.x[4 * q + 2] = u.z; P.x[4 * q + 3] = u.w;
                P.y[4 * q] = v.x; P.y[4 * q + 1] = v.y; P.y[4 * q + 2] = v.z; P.y[4 * q + 3] = v.w;
                Q.x[4 * q] = w.x; Q.x[4 * q + 1] = w.y; Q.x[4 * q + 2] = w.z; Q.x[4 * q + 3] = w.w;
                Q.y[4 * q] = z.x; Q.y[4 * q + 1] = z.y; Q.y[4 * q + 2] = z.z; Q.y[4 * q + 3] = z.w;
            }
        } else if (t > 0) {
            load_poly<K>(x1, y1, k, P);
            load_poly<K>(x2, y2, k, Q);
        }
        recentre<K>(P, Q);
        if (DGAL_FWD_P2MODE == kP2Smem) {
#pragma unroll
            for (int q = 0; q < K; ++q) { sqt[q] = Q.x[q]; sqt[K + 2 + q] = Q.y[q]; }
            sqt[K] = Q.x[0];
            sqt[2 * K + 2] = Q.y[0];
        }
        const FwdOut<K, true> r = iou_fwd<K, true, DGAL_FWD_P2MODE, DGAL_THIN, WL || WL8>(P, Q, qt, WL ? &wlut[0] : nullptr,
                                                                             WL8 ? &wlut8[0] : nullptr);
        thinmask |= (uint32_t)r.thin << t;   // thin pair: fixed after the loop
        __stcs(iou + k, r.iou);
        nx[k] = (uint8_t)r.nx;
        if (K == 4) {
            __stcs(reinterpret_cast<unsigned long long *>(xflags) + k, (unsigned long long)r.seq.w[0]);
        } else {
            ulonglong2 v;
            v.x = r.seq.w[0];
            v.y = r.seq.w[Seq<K>::NW - 1];
            __stcs(reinterpret_cast<ulonglong2 *>(xflags) + k, v);
        }
    }
    // thin pairs (rare; dgal_exact.cuh): the areas of the record this thread stored, in
    // double from the raw inputs, decide emptiness and the IoU (out of the hot loop)
#ifdef DGAL_THIN_NOPOST
    if (thinmask) iou[k0] = -1.f;
    thinmask = 0;
#endif
#pragma unroll 1
    while (thinmask) {
        const int t = __ffs(thinmask) - 1;
        thinmask &= thinmask - 1u;
        const int64_t k = k0 + (int64_t)t * T;
        Seq<K> sq2;
        int m = nx[k];
        if (K == 4) sq2.w[0] = reinterpret_cast<const unsigned long long *>(xflags)[k];
        else {
            const ulonglong2 v = reinterpret_cast<const ulonglong2 *>(xflags)[k];
            sq2.w[0] = v.x; sq2.w[Seq<K>::NW - 1] = v.y;
        }
        float v;
        fwd_thin_redo<K>(RawPolyVerts{x1 + k * K, y1 + k * K, x2 + k * K, y2 + k * K}, sq2, m, v);
        iou[k] = v;
        nx[k] = (uint8_t)m;
        if (K == 4) reinterpret_cast<unsigned long long *>(xflags)[k] = sq2.w[0];
        else reinterpret_cast<ulonglong2 *>(xflags)[k] = make_ulonglong2(sq2.w[0], sq2.w[Seq<K>::NW - 1]);
    }
}

// ---------------------------------------------------------------------------
// Backward: persistent CTAs, bulk-copy (TMA engine) pipeline of input tiles
// ---------------------------------------------------------------------------
// One tile = kTile consecutive pairs = one contiguous byte range per input
// (x1, y1, x2, y2, grad, xflags, nx).  Thread 0 prefetches tile it+1 into the
// other stage of a 2-deep shared-memory ring while every thread computes tile
// it from shared memory, so the 141 B/pair of HBM traffic overlaps the math at
// any occupancy.  The tail tile (or misaligned inputs) is loaded directly.
// Warps are independent within a tile (own pairs, own crossing queue), so a
// stage is released per warp on an "empty" mbarrier instead of a CTA barrier:
// only the producer waits for all warps before refilling it; the others run on.
#ifndef DGAL_BWD4_TILE
#define DGAL_BWD4_TILE 256
#endif
#ifndef DGAL_BWD8_TILE
#define DGAL_BWD8_TILE 128   // K = 8: smaller tiles so 2+ CTAs fit the shared memory
#endif
#ifndef DGAL_BWD4_MINB
#define DGAL_BWD4_MINB 3
#endif
#ifndef DGAL_BWD8_MINB
#define DGAL_BWD8_MINB 3   // A/B (K = 8): 256 x 1 CTA 0.263 ms, 128 x 2 0.262, 128 x 3 0.235
#endif
template <int K>
struct BwdCfg {
    static constexpr int tile = (K == 4) ? DGAL_BWD4_TILE : DGAL_BWD8_TILE;
    static constexpr int threads = tile + 32;   // + the producer warp
    static constexpr int minb = (K == 4) ? DGAL_BWD4_MINB : DGAL_BWD8_MINB;
};

template <int K>
struct BwdSmem {
    static constexpr int kTile = BwdCfg<K>::tile;
    struct Stage {
        float x1[kTile * K], y1[kTile * K], x2[kTile * K], y2[kTile * K];
        float g[kTile];
        uint64_t xf[kTile * (K / 4)];  // 2K flag bytes per pair
        uint8_t nx[kTile];
    };
    Stage st[2];
    float scr[4 * K * kTile];                       // interval end points, [slot][pair]
    uint16_t queue[kTile / 32][32 * 2 * K];         // per-warp crossing queue: lane << 8 | byte
    FlagLut lut;
    uint64_t bar[2];     // full: the stage's bulk copies landed
    uint64_t empty[2];   // empty: every warp is done with the stage
};

// Warp-specialised: warps 0..7 consume (one pair per thread), warp 8 produces —
// its lane 0 refills a stage with the next tile as soon as all consumer warps have
// released it, so no consumer ever waits on the producer's own bookkeeping.
template <int K>
__global__ void __launch_bounds__(BwdCfg<K>::threads, BwdCfg<K>::minb)
paired_bwd_kernel(int64_t n, const float *__restrict__ x1, const float *__restrict__ y1,
                  const float *__restrict__ x2, const float *__restrict__ y2,
                  const float *__restrict__ grad, const uint8_t *__restrict__ nx,
                  const uint8_t *__restrict__ xflags,
                  float *__restrict__ gx1, float *__restrict__ gy1,
                  float *__restrict__ gx2, float *__restrict__ gy2, int use_bulk)
{
    extern __shared__ __align__(128) unsigned char smem_raw[];
    BwdSmem<K> &S = *reinterpret_cast<BwdSmem<K> *>(smem_raw);
    constexpr int kTile = BwdCfg<K>::tile, kBwdThreads = BwdCfg<K>::threads;
    const int tid = threadIdx.x;
    const int64_t ntiles = (n + kTile - 1) / kTile;
    const int64_t nfull = use_bulk ? n / kTile : 0;  // tiles fed by bulk copies
    constexpr uint32_t kStageBytes = 4u * kTile * K * 4u + kTile * 4u + kTile * 2u * K + kTile;

    fill_flag_lut(S.lut, tid, kBwdThreads);
    if (tid == 0) {
        mbar_init(&S.bar[0], 1);
        mbar_init(&S.bar[1], 1);
        mbar_init(&S.empty[0], kTile / 32);
        mbar_init(&S.empty[1], kTile / 32);
        fence_mbar_init();
    }
    __syncthreads();

    if (tid >= kTile) {   // ---- producer warp ----
        if (tid == kTile) {
            int it = 0;
#pragma unroll 1
            for (int64_t tile = blockIdx.x; tile < nfull; ++it, tile += gridDim.x) {
                const int s = it & 1;
                // stage s last held tile it-2: wait until every consumer warp released it
                if (it >= 2) mbar_wait(&S.empty[s], (uint32_t)((it - 2) >> 1) & 1u);
                const int64_t b = tile * kTile;
                typename BwdSmem<K>::Stage &T = S.st[s];
                mbar_arrive_expect_tx(&S.bar[s], kStageBytes);
                bulk_g2s(T.x1, x1 + b * K, kTile * K * 4, &S.bar[s]);
                bulk_g2s(T.y1, y1 + b * K, kTile * K * 4, &S.bar[s]);
                bulk_g2s(T.x2, x2 + b * K, kTile * K * 4, &S.bar[s]);
                bulk_g2s(T.y2, y2 + b * K, kTile * K * 4, &S.bar[s]);
                bulk_g2s(T.g, grad + b, kTile * 4, &S.bar[s]);
                bulk_g2s(T.xf, xflags + b * 2 * K, kTile * 2 * K, &S.bar[s]);
                bulk_g2s(T.nx, nx + b, kTile, &S.bar[s]);
            }
        }
        return;
    }

    int64_t tile = blockIdx.x;
#pragma unroll 1
    for (int it = 0; tile < ntiles; ++it, tile += gridDim.x) {
        const int s = it & 1;
        typename BwdSmem<K>::Stage &T = S.st[s];
        const int64_t k = tile * kTile + tid;
        DGAL_ASSERT(tile < ntiles && (tile >= nfull || (tile + 1) * kTile <= n));
        if (tile < nfull) {
            mbar_wait(&S.bar[s], (uint32_t)(it >> 1) & 1u);
        } else if (k < n) {  // direct path: this thread stages its own pair (own slots only)
#pragma unroll
            for (int q = 0; q < K; ++q) {
                T.x1[tid * K + q] = x1[k * K + q]; T.y1[tid * K + q] = y1[k * K + q];
                T.x2[tid * K + q] = x2[k * K + q]; T.y2[tid * K + q] = y2[k * K + q];
            }
            T.g[tid] = grad[k];
            T.nx[tid] = nx[k];
#pragma unroll
            for (int q = 0; q < K / 4; ++q)
                T.xf[tid * (K / 4) + q] = reinterpret_cast<const uint64_t *>(xflags)[k * (K / 4) + q];
        }
        // ---- per pair: provenance bits, the warp's crossings, epilogue ----
        const bool live = k < n;
        Seq<K> sq;
#pragma unroll
        for (int q = 0; q < K / 4; ++q) sq.w[q] = live ? T.xf[tid * (K / 4) + q] : 0ull;
        const int m = live ? T.nx[tid] : 0;
        Poly<K> G1, G2;
        const bool thin = bwd_tile_pair<K, kTile>(T.x1, T.y1, T.x2, T.y2, sq, m, live ? T.g[tid] : 0.f, live, S.scr,
                                                  S.queue[tid >> 5], S.lut, G1, G2);
        if (live) {
            store_plane<K>(gx1, k, G1.x);
            store_plane<K>(gy1, k, G1.y);
            store_plane<K>(gx2, k, G2.x);
            store_plane<K>(gy2, k, G2.y);
        }
        if (thin) {   // thin pair: area in double, gradients again (rare); the record re-read
            Seq<K> s2;
#pragma unroll
            for (int q = 0; q < K / 4; ++q) s2.w[q] = T.xf[tid * (K / 4) + q];
            bwd_pair_exact<K, kTile>(T.x1, T.y1, T.x2, T.y2, tid, s2, T.nx[tid], T.g[tid], S.scr, S.lut, G1, G2);
            store_plane<K>(gx1, k, G1.x);
            store_plane<K>(gy1, k, G1.y);
            store_plane<K>(gx2, k, G2.x);
            store_plane<K>(gy2, k, G2.y);
        }
        __syncwarp();                                      // the warp is done with stage s
        if ((tid & 31) == 0) mbar_arrive(&S.empty[s]);
    }
}

// ---------------------------------------------------------------------------
// Backward, per-thread prefetch: no producer warp, no stage barriers.  Every
// thread copies its own pair of the NEXT tile (vertices, g, flag bytes) into a
// 2-stage ring with cp.async while the warp works on the current tile; a warp
// only reads its own 32 pairs (crossing queue), so a __syncwarp after the
// copies complete is the only ordering needed.  CTAs own NT consecutive tiles.
// (The producer-warp kernel above spends ~20 % of its issue slots polling its
// full / empty barriers: ncu source counters.)
#ifndef DGAL_BWD4_PT
#define DGAL_BWD4_PT 1        // K = 4 backward: per-thread prefetch kernel (0: producer-warp kernel)
#endif
#ifndef DGAL_BWD_REV
#define DGAL_BWD_REV 1
#endif
#ifndef DGAL_BWDPT_THREADS
#define DGAL_BWDPT_THREADS 128
#endif
#ifndef DGAL_BWDPT_MINB
#define DGAL_BWDPT_MINB 7     // K = 4: 70 registers, 30 KB shared memory per CTA
#endif
#ifndef DGAL_BWD8_PT
#define DGAL_BWD8_PT 0
#endif
#ifndef DGAL_BWDPT8_MINB
#define DGAL_BWDPT8_MINB 3
#endif
#ifndef DGAL_BWDPT_NT
#define DGAL_BWDPT_NT 8
#endif
constexpr int kBwdPtThreads = DGAL_BWDPT_THREADS;

template <int K>
struct BwdPtSmem {
    static constexpr int T = kBwdPtThreads;
    struct Stage {
        float x1[T * K], y1[T * K], x2[T * K], y2[T * K];
        float g[T];
        uint64_t xf[T * (K / 4)];
    };
    Stage st[2];
    float scr[4 * K * T];
    uint16_t queue[T / 32][32 * 2 * K];
    FlagLut lut;
    uint32_t thinm[T];   // per thread: tiles whose pair is thin (kept here, not in a register: the loop is at 72)
};

// The per-thread backward's thin-pair redo (after its tile loop), out of line: its
// code then does not enter the register allocation of the hot loop.
template <int K>
__device__ __noinline__ void bwd_pt_thin_redo(int64_t n, const float *__restrict__ x1, const float *__restrict__ y1,
                                              const float *__restrict__ x2, const float *__restrict__ y2,
                                              const float *__restrict__ grad, const uint8_t *__restrict__ xflags,
                                              float *__restrict__ gx1, float *__restrict__ gy1,
                                              float *__restrict__ gx2, float *__restrict__ gy2, BwdPtSmem<K> &S)
{
    constexpr int T = kBwdPtThreads, NT = DGAL_BWDPT_NT;
    const int tid = threadIdx.x;
    uint32_t thinmask = S.thinm[tid];
    typename BwdPtSmem<K>::Stage &D = S.st[0];
    const int64_t chunk = DGAL_BWD_REV ? (int64_t)(gridDim.x - 1 - blockIdx.x) : (int64_t)blockIdx.x;
    const int64_t base = chunk * (NT * T);
    const int nv = (int)min((int64_t)NT, (n - base + T - 1) / T);
#pragma unroll 1
    while (thinmask) {
        const int t = __ffs(thinmask) - 1;
        thinmask &= thinmask - 1u;
        const int64_t k = base + (int64_t)(DGAL_BWD_REV ? (nv - 1 - t) : t) * T + tid;
#pragma unroll
        for (int q = 0; q < K; ++q) {
            D.x1[tid * K + q] = x1[k * K + q]; D.y1[tid * K + q] = y1[k * K + q];
            D.x2[tid * K + q] = x2[k * K + q]; D.y2[tid * K + q] = y2[k * K + q];
        }
        Seq<K> sq;
#pragma unroll
        for (int q = 0; q < K / 4; ++q) sq.w[q] = reinterpret_cast<const uint64_t *>(xflags)[k * (K / 4) + q];
        Poly<K> G1, G2;
        bwd_pair_exact<K, T, K == 4>(D.x1, D.y1, D.x2, D.y2, tid, sq, record_len<K>(sq), grad[k], S.scr, S.lut, G1,
                                     G2);
        store_plane<K>(gx1, k, G1.x);
        store_plane<K>(gy1, k, G1.y);
        store_plane<K>(gx2, k, G2.x);
        store_plane<K>(gy2, k, G2.y);
    }
}

template <int K>
__global__ void __launch_bounds__(kBwdPtThreads, (K == 4) ? DGAL_BWDPT_MINB : DGAL_BWDPT8_MINB)
paired_bwd_pt_kernel(int64_t n, const float *__restrict__ x1, const float *__restrict__ y1,
                     const float *__restrict__ x2, const float *__restrict__ y2,
                     const float *__restrict__ grad, const uint8_t *__restrict__ nx,
                     const uint8_t *__restrict__ xflags,
                     float *__restrict__ gx1, float *__restrict__ gy1,
                     float *__restrict__ gx2, float *__restrict__ gy2)
{
    constexpr int T = kBwdPtThreads, NT = DGAL_BWDPT_NT;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    BwdPtSmem<K> &S = *reinterpret_cast<BwdPtSmem<K> *>(smem_raw);
    const int tid = threadIdx.x;
    // DGAL_BWD_REV: chunks and tiles in descending order, so the first tiles the
    // backward reads are the last ones the forward touched (still in L2), and the
    // next forward's first tiles are the last ones this kernel read.
    const int64_t chunk = DGAL_BWD_REV ? (int64_t)(gridDim.x - 1 - blockIdx.x) : (int64_t)blockIdx.x;
    const int64_t base = chunk * (NT * T);
    const int nv = (int)min((int64_t)NT, (n - base + T - 1) / T);   // tiles of this chunk in range
    auto tile_base = [&](int t) { return base + (int64_t)(DGAL_BWD_REV ? (nv - 1 - t) : t) * T; };
    auto prefetch = [&](int stage, int64_t k) {
        typename BwdPtSmem<K>::Stage &D = S.st[stage];
#pragma unroll
        for (int q = 0; q < K / 4; ++q) {
            cp_async16(D.x1 + tid * K + 4 * q, x1 + k * K + 4 * q);
            cp_async16(D.y1 + tid * K + 4 * q, y1 + k * K + 4 * q);
            cp_async16(D.x2 + tid * K + 4 * q, x2 + k * K + 4 * q);
            cp_async16(D.y2 + tid * K + 4 * q, y2 + k * K + 4 * q);
        }
        cp_async4(D.g + tid, grad + k);
        if (K == 4) cp_async8(D.xf + tid, xflags + k * 8);
        else cp_async16(D.xf + 2 * tid, xflags + k * 16);
    };
    // nx is not loaded: a forward record's bytes past nx are the 0x00 padding (R2),
    // which the phases ignore (no flag-table bits, no crossing), so the record is
    // read whole (m = 2K; the thin redo counts its bytes) — one load and one live
    // register less per pair (the loop is at its 72-register budget)
    if (tile_base(0) + tid < n) prefetch(0, tile_base(0) + tid);
    cp_async_commit();
    fill_flag_lut(S.lut, tid, T);
    __syncthreads();
    S.thinm[tid] = 0u;
#pragma unroll 1
    for (int t = 0; t < nv; ++t) {
        const int64_t k = tile_base(t) + tid;
        const bool live = k < n;
        const int m = live ? 2 * K : 0;
        if (t + 1 < nv) {
            const int64_t kn = tile_base(t + 1) + tid;
            if (kn < n) prefetch((t + 1) & 1, kn);
        }
        cp_async_commit();
        cp_async_wait<1>();                      // this thread's copies of tile t landed
        __syncwarp();                            // ... and the other lanes' (crossing queue)
        typename BwdPtSmem<K>::Stage &D = S.st[t & 1];
        Seq<K> sq;
#pragma unroll
        for (int q = 0; q < K / 4; ++q) sq.w[q] = live ? D.xf[tid * (K / 4) + q] : 0ull;
        Poly<K> G1, G2;
        const bool thin = bwd_tile_pair<K, T, TileGeometry<K>, K == 4>(D.x1, D.y1, D.x2, D.y2, sq, m,
                                                                       live ? D.g[tid] : 0.f, live, S.scr,
                                                                       S.queue[tid >> 5], S.lut, G1, G2);
        if (live) {
            store_plane<K>(gx1, k, G1.x);
            store_plane<K>(gy1, k, G1.y);
            store_plane<K>(gx2, k, G2.x);
            store_plane<K>(gy2, k, G2.y);
        }
        if (thin) S.thinm[tid] |= 1u << t;      // thin pair: redone after the loop
        __syncwarp();                            // stage t & 1 is refilled next iteration
    }
    // thin pairs (rare; dgal_exact.cuh), out of the hot loop: each thread redoes its own,
    // re-staged at its slot of stage 0 from global memory, every crossing and the
    // intersection's area in double (bwd_pair_exact; no warp cooperation)
    if (!DGAL_THIN_BWD) return;
#ifdef DGAL_NOPOSTBWD
    return;
#endif
    cp_async_wait<0>();
    if (S.thinm[tid]) bwd_pt_thin_redo<K>(n, x1, y1, x2, y2, grad, xflags, gx1, gy1, gx2, gy2, S);
}

cudaError_t launch_paired_fwd(int K, int64_t n, const float *x1, const float *y1, const float *x2,
                              const float *y2, float *iou, uint8_t *nx, uint8_t *xflags,
                              cudaStream_t st)
{
    if (K == 4) {
        const unsigned grid = (unsigned)((n + DGAL_FWD4_NT * kFwd4Threads - 1) / (DGAL_FWD4_NT * kFwd4Threads));
        paired_fwd_direct_kernel<4><<<grid, kFwd4Threads, 0, st>>>(n, x1, y1, x2, y2, iou, nx, xflags);
    } else {
        const unsigned grid = (unsigned)((n + DGAL_FWD8_NT * kFwd8Threads - 1) / (DGAL_FWD8_NT * kFwd8Threads));
        paired_fwd_direct_kernel<8><<<grid, kFwd8Threads, 0, st>>>(n, x1, y1, x2, y2, iou, nx, xflags);
    }
    return cudaGetLastError();
}

namespace {
template <int K>
cudaError_t launch_bwd_k(int64_t n, const float *x1, const float *y1, const float *x2, const float *y2,
                         const float *grad, const uint8_t *nx, const uint8_t *xflags, float *gx1, float *gy1,
                         float *gx2, float *gy2, cudaStream_t st)
{
    const size_t smem = sizeof(BwdSmem<K>);
    static DeviceCache cache;
    const int limit = cache.get([&](int dev) {
        const int a = set_smem_attr(paired_bwd_kernel<K>, smem);
        if (a <= 0) return a;
        int sms = 0, per = 0;
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, paired_bwd_kernel<K>, BwdCfg<K>::threads, smem);
        return sms * (per > 0 ? per : 1);
    });
    if (limit <= 0) return (cudaError_t)(-limit);
    constexpr int kTile = BwdCfg<K>::tile;
    const int64_t ntiles = (n + kTile - 1) / kTile;
    const unsigned grid = (unsigned)(ntiles < limit ? ntiles : limit);
    auto al16 = [](const void *p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; };
    const int use_bulk = al16(grad) && al16(nx) && al16(xflags);   // planes are 16 B aligned (ABI)
    paired_bwd_kernel<K><<<grid, BwdCfg<K>::threads, smem, st>>>(n, x1, y1, x2, y2, grad, nx, xflags, gx1, gy1, gx2,
                                                           gy2, use_bulk);
    return cudaGetLastError();
}
template <int K>
cudaError_t launch_bwd_pt(int64_t n, const float *x1, const float *y1, const float *x2, const float *y2,
                          const float *grad, const uint8_t *nx, const uint8_t *xflags, float *gx1, float *gy1,
                          float *gx2, float *gy2, cudaStream_t st)
{
    const size_t smem = sizeof(BwdPtSmem<K>);
    static DeviceCache cache;
    const int a = cache.get([&](int) { return set_smem_attr(paired_bwd_pt_kernel<K>, smem); });
    if (a <= 0) return (cudaError_t)(-a);
    constexpr int64_t per = (int64_t)DGAL_BWDPT_NT * kBwdPtThreads;
    paired_bwd_pt_kernel<K><<<(unsigned)((n + per - 1) / per), kBwdPtThreads, smem, st>>>(
        n, x1, y1, x2, y2, grad, nx, xflags, gx1, gy1, gx2, gy2);
    return cudaGetLastError();
}
}  // namespace

cudaError_t launch_paired_bwd(int K, int64_t n, const float *x1, const float *y1, const float *x2,
                              const float *y2, const float *grad, const uint8_t *nx,
                              const uint8_t *xflags, float *gx1, float *gy1, float *gx2, float *gy2,
                              cudaStream_t st)
{
    auto al = [](const void *p, uintptr_t a) { return (reinterpret_cast<uintptr_t>(p) & (a - 1)) == 0; };
    if (K == 4 && DGAL_BWD4_PT && al(grad, 4) && al(xflags, 8))
        return launch_bwd_pt<4>(n, x1, y1, x2, y2, grad, nx, xflags, gx1, gy1, gx2, gy2, st);
    if (K == 8 && DGAL_BWD8_PT && al(grad, 4) && al(xflags, 16))
        return launch_bwd_pt<8>(n, x1, y1, x2, y2, grad, nx, xflags, gx1, gy1, gx2, gy2, st);
    if (K == 4) return launch_bwd_k<4>(n, x1, y1, x2, y2, grad, nx, xflags, gx1, gy1, gx2, gy2, st);
    return launch_bwd_k<8>(n, x1, y1, x2, y2, grad, nx, xflags, gx1, gy1, gx2, gy2, st);
}

// ---------------------------------------------------------------------------
// Fused loss forward + backward, one pair per thread
// ---------------------------------------------------------------------------
// CTA shape and CTAs per SM the fused kernels are register-budgeted for (A/B on
// B200: K = 4 256 x 3 0.519 ms, 128 x 6 0.505 ms; K = 8 256 x 1 0.523 ms, 128 x 3
// 0.361 ms, 128 x 2 0.443 ms)
#ifndef DGAL_FUSED4_MINB
#define DGAL_FUSED4_MINB 6
#endif
#ifndef DGAL_FUSED4_THREADS
#define DGAL_FUSED4_THREADS 128
#endif
#ifndef DGAL_FUSED8_MINB
#define DGAL_FUSED8_MINB 3
#endif
#ifndef DGAL_FUSED8_THREADS
#define DGAL_FUSED8_THREADS 128
#endif
constexpr int kFused4Threads = DGAL_FUSED4_THREADS, kFused8Threads = DGAL_FUSED8_THREADS;

#ifndef DGAL_FUSED_PT_TS
#define DGAL_FUSED_PT_TS 1    // piece table [thread][slot] (1) or [slot][thread] (0)
#endif
#ifndef DGAL_FUSED_NEED
#define DGAL_FUSED_NEED 1     // mark nearly parallel crossings / thin pairs for the refine pass (A/B switch)
#endif
#ifndef DGAL_FUSED_PF
#define DGAL_FUSED_PF 1       // NT consecutive tiles per CTA, tile t+1 copied (cp.async) while tile t computes
#endif
#ifndef DGAL_FUSED4_NT
#define DGAL_FUSED4_NT 8
#endif
#ifndef DGAL_FUSED8_NT
#define DGAL_FUSED8_NT 8
#endif
#ifndef DGAL_FUSED8_PF
#define DGAL_FUSED8_PF 1
#endif

template <int K>
__global__ void __launch_bounds__((K == 4) ? kFused4Threads : kFused8Threads,
                                  (K == 4) ? DGAL_FUSED4_MINB : DGAL_FUSED8_MINB)
paired_fused_kernel(int64_t n, const float *__restrict__ x1, const float *__restrict__ y1,
                    const float *__restrict__ x2, const float *__restrict__ y2,
                    const float *__restrict__ grad, float scale, float *__restrict__ iou,
                    float *__restrict__ gx1, float *__restrict__ gy1,
                    float *__restrict__ gx2, float *__restrict__ gy2, RefineQueue *__restrict__ refine)
{
#ifndef DGAL_FUSED_PK
#define DGAL_FUSED_PK true   // K = 4: gradient part in paired FP32 (K = 8 would spill)
#endif
#ifndef DGAL_FUSED_P2MODE
#define DGAL_FUSED_P2MODE kP2PiecesSmem   // A/B: kP2Pieces 0.571 ms, kP2PiecesSmem 0.526 ms (cfg3)
#endif
    constexpr int T = (K == 4) ? kFused4Threads : kFused8Threads;
    constexpr bool PF = (K == 4) ? DGAL_FUSED_PF : DGAL_FUSED8_PF;
    constexpr int NT = !PF ? 1 : (K == 4) ? DGAL_FUSED4_NT : DGAL_FUSED8_NT;
    // dynamic shared memory (FusedSmem<K>; K = 8 with the ring exceeds 48 KB):
    //   pt     piece table [slot][thread] (kP2PiecesSmem)
    //   ring   PF: 2-stage per-thread ring [stage][plane][thread][K]
    //   gring  PF: [stage][thread] dL/dIoU
    // (each thread copies and reads only its own words: no CTA barrier)
    extern __shared__ __align__(16) float fsm[];
    float *ring = fsm;
    float *gring = ring + (PF ? 2 * 4 * T * K : 0);
    float *pt = gring + (PF ? 2 * T : 0);
    // piece table: [thread][slot] with an odd per-thread stride kPtS (conflict-free; an
    // event's address is one LEA) — x of a_j at j, of b_j at K + j, y at 2K + ...
    constexpr int kPtS = DGAL_FUSED_PT_TS ? 4 * K + 1 : 1;
    uint64_t *illt = reinterpret_cast<uint64_t *>(pt + (DGAL_FUSED_PT_TS ? kPtS * T : 4 * K * T));   // K = 8: ILL factors, [q][thread]
    const int tid = threadIdx.x;
    const int64_t k0 = (int64_t)blockIdx.x * (NT * T) + tid;
    auto prefetch = [&](int stage, int64_t k) {
        float *r = ring + stage * (4 * T * K) + tid * K;
#pragma unroll
        for (int q = 0; q < K / 4; ++q) {
            cp_async16(r + 4 * q, x1 + k * K + 4 * q);
            cp_async16(r + T * K + 4 * q, y1 + k * K + 4 * q);
            cp_async16(r + 2 * T * K + 4 * q, x2 + k * K + 4 * q);
            cp_async16(r + 3 * T * K + 4 * q, y2 + k * K + 4 * q);
        }
        if (grad) cp_async4(gring + stage * T + tid, grad + k);
    };
    if (PF) {
        if (k0 < n) prefetch(0, k0);
        cp_async_commit();
    }
#pragma unroll 1
    for (int t = 0; t < NT; ++t) {
        const int64_t k = k0 + (int64_t)t * T;
        if (k >= n) break;
        Poly<K> P, Q, G1, G2;
        float g = scale;
        if (PF) {
            if (t + 1 < NT && k + T < n) prefetch((t + 1) & 1, k + T);
            cp_async_commit();
            cp_async_wait<1>();   // this thread's copies of tile t have landed
            const float *r = ring + (t & 1) * (4 * T * K) + tid * K;
#pragma unroll
            for (int q = 0; q < K / 4; ++q) {
                const float4 u = *reinterpret_cast<const float4 *>(r + 4 * q);
                const float4 v = *reinterpret_cast<const float4 *>(r + T * K + 4 * q);
                const float4 w = *reinterpret_cast<const float4 *>(r + 2 * T * K + 4 * q);
                const float4 z = *reinterpret_cast<const float4 *>(r + 3 * T * K + 4 * q);
                P.x[4 * q] = u.x; P.x[4 * q + 1] = u.y; P.x[4 * q + 2] = u.z; P.x[4 * q + 3] = u.w;
                P.y[4 * q] = v.x; P.y[4 * q + 1] = v.y; P.y[4 * q + 2] = v.z; P.y[4 * q + 3] = v.w;
                Q.x[4 * q] = w.x; Q.x[4 * q + 1] = w.y; Q.x[4 * q + 2] = w.z; Q.x[4 * q + 3] = w.w;
                Q.y[4 * q] = z.x; Q.y[4 * q + 1] = z.y; Q.y[4 * q + 2] = z.z; Q.y[4 * q + 3] = z.w;
            }
            if (grad) g = gring[(t & 1) * T + tid];
        } else {
            load_poly<K>(x1, y1, k, P);
            load_poly<K>(x2, y2, k, Q);
            if (grad) g = __ldcs(grad + k);
        }
        recentre<K>(P, Q);
        bool need = false;
        const float v = iou_fused<K, DGAL_FUSED_P2MODE, K == 4 && DGAL_FUSED_PK>(
            P, Q, g, G1, G2, flat(), nullptr,
            DGAL_FUSED_PT_TS ? QTable{pt + tid * kPtS, pt + tid * kPtS + 2 * K, 1}
                             : QTable{pt + tid, pt + 2 * K * T + tid, T},
            DGAL_FUSED_NEED ? &need : nullptr, IllTab{illt + tid, T});
        refine_mark(refine, k, need);   // redone exactly by paired_fused_refine_kernel
        if (iou) __stcs(iou + k, v);
        store_plane<K>(gx1, k, G1.x);
        store_plane<K>(gy1, k, G1.y);
        store_plane<K>(gx2, k, G2.x);
        store_plane<K>(gy2, k, G2.y);
    }
}

// ---------------------------------------------------------------------------
// Refine pass of the fused kernel (dgal_refine.cuh): the marked pairs redone with
// the split path's arithmetic — the forward clip with flags (+ the area of the
// recorded intersection in double for a thin pair), then the backward phases
// through those flags (ill-conditioned crossings refined in double).  Each CTA
// gathers a chunk's marked pairs and works on them 128 at a time.
// ---------------------------------------------------------------------------
template <int K>
struct RefineSmem {
    float x1[kRefT * K], y1[kRefT * K], x2[kRefT * K], y2[kRefT * K];   // raw tile, [pair][k]
    float scr[4 * K * kRefT];                               // interval end points, [slot][pair]
    uint16_t queue[kRefT / 32][32 * 2 * K];                 // per-warp crossing queue
    float sq[2 * (K + 2) * kRefT];                          // per-thread p2 vertex table (kP2Smem, QTable rows), [row][thread]
    FlagLut lut;
};

template <int K>
__global__ void __launch_bounds__(kRefT, (K == 4) ? 4 : 2)
paired_fused_refine_kernel(int64_t n, const float *__restrict__ x1, const float *__restrict__ y1,
                           const float *__restrict__ x2, const float *__restrict__ y2,
                           const float *__restrict__ grad, float scale, float *__restrict__ iou,
                           float *__restrict__ gx1, float *__restrict__ gy1, float *__restrict__ gx2,
                           float *__restrict__ gy2, RefineQueue *__restrict__ refine)
{
    extern __shared__ __align__(16) unsigned char smem_raw[];
    RefineSmem<K> &S = *reinterpret_cast<RefineSmem<K> *>(smem_raw);
    const int tid = threadIdx.x;
    const unsigned int total = refine_count(refine);
    if ((unsigned int)blockIdx.x * kRefT < total) {
        fill_flag_lut(S.lut, tid, kRefT);
        __syncthreads();
    }
#pragma unroll 1
    for (unsigned int base = blockIdx.x * kRefT; base < total; base += gridDim.x * kRefT) {
        const unsigned int e = base + tid;
        const bool live = e < total;
        const int64_t k = live ? (int64_t)refine->idx[e] : 0;
        DGAL_ASSERT(!live || k < n);
        Poly<K> P, Q;
        if (live) {
            load_poly<K>(x1, y1, k, P);
            load_poly<K>(x2, y2, k, Q);
        } else {
#pragma unroll
            for (int q = 0; q < K; ++q) { P.x[q] = P.y[q] = Q.x[q] = Q.y[q] = 0.f; }
        }
#pragma unroll
        for (int q = 0; q < K; ++q) {
            S.x1[tid * K + q] = P.x[q]; S.y1[tid * K + q] = P.y[q];
            S.x2[tid * K + q] = Q.x[q]; S.y2[tid * K + q] = Q.y[q];
        }
        recentre<K>(P, Q);
#pragma unroll
        for (int q = 0; q <= K; ++q) {
            S.sq[q * kRefT + tid] = Q.x[q % K];
            S.sq[(K + 2 + q) * kRefT + tid] = Q.y[q % K];
        }
        S.sq[(K + 1) * kRefT + tid] = 0.f;
        S.sq[(2 * K + 3) * kRefT + tid] = 0.f;
        FwdOut<K, true> r = iou_fwd<K, true, kP2Smem, true>(P, Q, QTable{S.sq + tid, S.sq + (K + 2) * kRefT + tid, kRefT});
        if (r.thin)
            fwd_thin_redo<K>(RawPolyVerts{S.x1 + tid * K, S.y1 + tid * K, S.x2 + tid * K, S.y2 + tid * K}, r.seq,
                            r.nx, r.iou);
        if (live && iou) iou[k] = r.iou;
        const float g = live ? (grad ? grad[k] : scale) : 0.f;
        __syncwarp();   // the warp's tile is staged (the crossing queue reads other lanes' pairs)
        Poly<K> G1, G2;
        const bool thin = bwd_tile_pair<K, kRefT, TileGeometry<K>, false>(
            S.x1, S.y1, S.x2, S.y2, r.seq, live ? r.nx : 0, g, live, S.scr, S.queue[tid >> 5], S.lut, G1, G2);
        if (thin) bwd_pair_exact<K, kRefT>(S.x1, S.y1, S.x2, S.y2, tid, r.seq, r.nx, g, S.scr, S.lut, G1, G2);
        if (live) {
            store_plane<K>(gx1, k, G1.x);
            store_plane<K>(gy1, k, G1.y);
            store_plane<K>(gx2, k, G2.x);
            store_plane<K>(gy2, k, G2.y);
        }
        __syncwarp();   // the tile is restaged next round
    }
    __syncthreads();
    if (tid == 0) refine_finish(refine);
}

namespace {
int refine_grid()
{
    static DeviceCache cache;
    const int sms = cache.get([](int dev) {
        int s = 0;
        cudaDeviceGetAttribute(&s, cudaDevAttrMultiProcessorCount, dev);
        return s;
    });
    return (sms > 0 ? sms : 148) * 2;
}
}  // namespace

int refine_grid_for(int64_t) { return refine_grid(); }
size_t refine_workspace_bytes(int64_t n) { return refine_queue_bytes(n); }

namespace {
template <int K>
constexpr size_t fused_smem_bytes()
{
    constexpr int T = (K == 4) ? kFused4Threads : kFused8Threads;
    constexpr bool PF = (K == 4) ? DGAL_FUSED_PF : DGAL_FUSED8_PF;
    return sizeof(float) * ((PF ? 2 * 4 * T * K + 2 * T : 0) + (DGAL_FUSED_PT_TS ? 4 * K + 1 : 4 * K) * T) +
           (K == 8 ? 8 * (K / 2) * T : 0);
}
template <int K>
cudaError_t launch_fused_k(int64_t n, const float *x1, const float *y1, const float *x2, const float *y2,
                           const float *grad, float scale, float *iou, float *gx1, float *gy1, float *gx2,
                           float *gy2, RefineQueue *refine, cudaStream_t st)
{
    constexpr int T = (K == 4) ? kFused4Threads : kFused8Threads;
    constexpr bool PF = (K == 4) ? DGAL_FUSED_PF : DGAL_FUSED8_PF;
    constexpr int64_t per = (int64_t)(PF ? ((K == 4) ? DGAL_FUSED4_NT : DGAL_FUSED8_NT) : 1) * T;
    constexpr size_t smem = fused_smem_bytes<K>();
    static DeviceCache cache, rcache;
    const int a = cache.get([&](int) { return set_smem_attr(paired_fused_kernel<K>, smem); });
    if (a <= 0) return (cudaError_t)(-a);
    const int b = rcache.get([&](int) { return set_smem_attr(paired_fused_refine_kernel<K>, sizeof(RefineSmem<K>)); });
    if (b <= 0) return (cudaError_t)(-b);
    paired_fused_kernel<K><<<(unsigned)((n + per - 1) / per), T, smem, st>>>(n, x1, y1, x2, y2, grad, scale, iou,
                                                                               gx1, gy1, gx2, gy2, refine);
    paired_fused_refine_kernel<K><<<(unsigned)refine_grid(), kRefT, sizeof(RefineSmem<K>), st>>>(
        n, x1, y1, x2, y2, grad, scale, iou, gx1, gy1, gx2, gy2, refine);
    return cudaGetLastError();
}
}  // namespace

cudaError_t launch_paired_fused(int K, int64_t n, const float *x1, const float *y1, const float *x2,
                                const float *y2, const float *grad, float scale, float *iou, float *gx1,
                                float *gy1, float *gx2, float *gy2, void *refine, cudaStream_t st)
{
    RefineQueue *q = static_cast<RefineQueue *>(refine);
    if (K == 4) return launch_fused_k<4>(n, x1, y1, x2, y2, grad, scale, iou, gx1, gy1, gx2, gy2, q, st);
    return launch_fused_k<8>(n, x1, y1, x2, y2, grad, scale, iou, gx1, gy1, gx2, gy2, q, st);
}

}  // namespace dgal
