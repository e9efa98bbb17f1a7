// dgal_pairwise.cu — N x M pairwise IoU + NMS overlap mask (north_star; S:506-513
// "cartesian").  DESIGN.md §4.3.
//
// CTA = 8 warps, a block of 64 rows and a 1024-column tile, both staged in shared
// memory (vertices + bounding circles).  Warp w owns 8 of the rows.  It sweeps
// the tile 128 columns per step, 4 consecutive columns per lane; a lane loads its
// 4 column circles once per step and tests them against the warp's 8 row circles
// (kept in registers), so every shared-memory load feeds 8 rows:
//   * bounding-circle reject (exact: disjoint circles => disjoint polygons),
//   * one float4 streaming zero store per (row, 4 columns) — the output write is
//     the roof of the large matrix,
//   * the 32 (row, column) candidate bits of a lane form one mask; one vote per
//     step; survivors are compacted (warp prefix sum) into a per-warp queue that
//     spans all the warp's rows and is evaluated 32 at a time (full SIMT width),
//   * candidate results overwrite their zero, set a bit in the CTA's shared
//     64 x 1024 bitmap (written out as whole uint64 words at the end) and, for
//     c < row, append to the row's suppressor list.
#include "dgal_core.cuh"
#include "dgal_internal.h"

namespace dgal {

namespace {

constexpr unsigned kFull = 0xFFFFFFFFu;
constexpr int kRowsPerWarp = kPwRowsPerCta / kPwWarps;      // 8
constexpr int kQueue = 32 + kRowsPerWarp * 128;             // <=31 left + one step's worth

template <int K>
__device__ __forceinline__ float4 bounding_circle(const float *x, const float *y)
{
    float cx = 0.f, cy = 0.f;
#pragma unroll
    for (int k = 0; k < K; ++k) { cx += x[k]; cy += y[k]; }
    cx *= (1.f / K);
    cy *= (1.f / K);
    float r2 = 0.f;
#pragma unroll
    for (int k = 0; k < K; ++k) {
        const float dx = x[k] - cx, dy = y[k] - cy;
        r2 = fmaxf(r2, dx * dx + dy * dy);
    }
    // inflate: relative (sqrt/rounding) + absolute (ulp of the scene coordinates)
    const float r = sqrtf(r2) * 1.0001f + 2e-6f * (fabsf(cx) + fabsf(cy)) + 1e-30f;
    return make_float4(cx, cy, r, 0.f);
}

template <int K>
struct PwSmem {
    float cx[kPwTileCols * K], cy[kPwTileCols * K];     // column tile, [col][k]
    float4 ccirc[kPwTileCols];
    float rx[kPwRowsPerCta * K], ry[kPwRowsPerCta * K];  // row block, [row][k]
    uint32_t bits[kPwRowsPerCta][kPwTileCols / 32];
    uint32_t queue[kPwWarps][kQueue];                    // row_local << 16 | col_local
};

}  // namespace

template <int K>
__global__ void __launch_bounds__(kPwThreads)
pairwise_kernel(int64_t n_rows, const float *__restrict__ rxg, const float *__restrict__ ryg, int64_t m,
                const float *__restrict__ cxg, const float *__restrict__ cyg, int64_t row_offset,
                float *__restrict__ iou, float thr, uint64_t *__restrict__ mask, int64_t mask_words,
                int32_t *__restrict__ nbr_count, int32_t *__restrict__ nbr_idx, int32_t cap)
{
    extern __shared__ __align__(16) unsigned char smem_raw[];
    PwSmem<K> &S = *reinterpret_cast<PwSmem<K> *>(smem_raw);
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int64_t c0 = (int64_t)blockIdx.y * kPwTileCols;
    const int64_t r0 = (int64_t)blockIdx.x * kPwRowsPerCta;
    const int ncols = (int)min((int64_t)kPwTileCols, m - c0);
    const int nrows = (int)min((int64_t)kPwRowsPerCta, n_rows - r0);
    const float inf = __int_as_float(0x7f800000);

    // ---- stage the column tile and the row block ----
    for (int t = tid; t < kPwTileCols * K; t += kPwThreads) {
        const bool ok = t < ncols * K;
        S.cx[t] = ok ? __ldg(cxg + c0 * K + t) : 0.f;
        S.cy[t] = ok ? __ldg(cyg + c0 * K + t) : 0.f;
    }
    for (int t = tid; t < kPwRowsPerCta * K; t += kPwThreads) {
        const bool ok = t < nrows * K;
        S.rx[t] = ok ? __ldg(rxg + r0 * K + t) : 0.f;
        S.ry[t] = ok ? __ldg(ryg + r0 * K + t) : 0.f;
    }
    for (int t = tid; t < kPwRowsPerCta * kPwTileCols / 32; t += kPwThreads) (&S.bits[0][0])[t] = 0u;
    __syncthreads();
    for (int t = tid; t < kPwTileCols; t += kPwThreads)
        S.ccirc[t] = (t < ncols) ? bounding_circle<K>(S.cx + t * K, S.cy + t * K)
                                 : make_float4(inf, inf, 0.f, 0.f);
    __syncthreads();

    // ---- this warp's rows: circles in registers ----
    float4 rc[kRowsPerWarp];
#pragma unroll
    for (int q = 0; q < kRowsPerWarp; ++q) {
        const int rl = warp * kRowsPerWarp + q;
        rc[q] = (rl < nrows) ? bounding_circle<K>(S.rx + rl * K, S.ry + rl * K)
                             : make_float4(-inf, -inf, 0.f, 0.f);
    }
    const bool vec_store = iou != nullptr && (m % 4 == 0) && ((reinterpret_cast<uintptr_t>(iou) & 15u) == 0);
    uint32_t *queue = S.queue[warp];

    auto evaluate = [&](uint32_t ent) {
        const int rl = (int)(ent >> 16), cl = (int)(ent & 0xFFFFu);
        DGAL_ASSERT(rl < nrows && cl < ncols);
        const float *px = S.rx + rl * K, *py = S.ry + rl * K;
        const float *qx = S.cx + cl * K, *qy = S.cy + cl * K;
        const float ox = px[0], oy = py[0];
        Poly<K> Pc, Qc;
#pragma unroll
        for (int k = 0; k < K; ++k) {
            Pc.x[k] = __fsub_rn(px[k], ox); Pc.y[k] = __fsub_rn(py[k], oy);
            Qc.x[k] = __fsub_rn(qx[k], ox); Qc.y[k] = __fsub_rn(qy[k], oy);
        }
        Pc.x[0] = 0.f;   // exact for finite input; lets the compiler fold it
        Pc.y[0] = 0.f;
        const FwdOut<K, false> fo = iou_fwd<K, false>(Pc, Qc);
        float v = fo.iou;
        // thin pair (R^2 > kThinRatio A_u): the area of the recorded intersection in double
        if (DGAL_THIN && pair_is_thin(pair_extent2<K>(Pc, Qc), (fo.A1x2 + fo.A2x2) - fo.Aix2))
            v = pair_iou_exact<K>(px, py, qx, qy);
        const int64_t r = r0 + rl, c = c0 + cl;
        if (iou) iou[r * m + c] = v;
        const int64_t grow = row_offset + r;
        if (v > thr && c != grow) {
            if (mask) atomicOr(&S.bits[rl][cl >> 5], 1u << (cl & 31));
            if (nbr_count && c < grow) {
                const int slot = atomicAdd(nbr_count + r, 1);
                if (slot < cap) nbr_idx[r * cap + slot] = (int32_t)c;
            }
        }
    };

    int qn = 0;
#pragma unroll 1
    for (int s = 0; s < kPwTileCols / 128; ++s) {
        const int cb = s * 128 + lane * 4;
        float4 cc[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) cc[u] = S.ccirc[cb + u];
        uint32_t cand = 0;  // bit 4q + u: row q, column cb + u
#pragma unroll
        for (int q = 0; q < kRowsPerWarp; ++q) {
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const float dx = cc[u].x - rc[q].x, dy = cc[u].y - rc[q].y, rs = cc[u].z + rc[q].z;
                cand |= (uint32_t)(dx * dx + dy * dy < rs * rs) << (4 * q + u);
            }
            const int rl = warp * kRowsPerWarp + q;
            if (iou && rl < nrows) {
                float *dst = iou + (r0 + rl) * m + c0 + cb;
                if (vec_store && cb + 3 < ncols) {
                    __stcs(reinterpret_cast<float4 *>(dst), make_float4(0.f, 0.f, 0.f, 0.f));
                } else {
#pragma unroll
                    for (int u = 0; u < 4; ++u)
                        if (cb + u < ncols) __stcs(dst + u, 0.f);
                }
            }
        }
        if (__any_sync(kFull, cand != 0)) {
            // compact this step's candidates into the warp queue (warp prefix sum)
            const int cnt = __popc(cand);
            int incl = cnt;
#pragma unroll
            for (int d = 1; d < 32; d <<= 1) {
                const int v = __shfl_up_sync(kFull, incl, d);
                if (lane >= d) incl += v;
            }
            int at = qn + incl - cnt;
            while (cand) {
                const int bit = __ffs(cand) - 1;
                cand &= cand - 1;
                DGAL_ASSERT(at < kQueue);
                queue[at++] = ((uint32_t)(warp * kRowsPerWarp + (bit >> 2)) << 16) | (uint32_t)(cb + (bit & 3));
            }
            qn += __shfl_sync(kFull, incl, 31);
            __syncwarp();
            while (qn >= 32) {  // warp-uniform
                evaluate(queue[qn - 32 + lane]);
                qn -= 32;
                __syncwarp();
            }
        }
    }
    __syncwarp();
    if (lane < qn) evaluate(queue[lane]);
    __syncthreads();

    // ---- mask rows of the block: whole uint64 words ----
    if (mask) {
        const int nw = (ncols + 63) >> 6;
        const int64_t w0 = c0 >> 6;
        for (int t = tid; t < nrows * nw; t += kPwThreads) {
            const int rl = t / nw, w = t - rl * nw;
            if (w0 + w < mask_words)
                mask[(r0 + rl) * mask_words + w0 + w] =
                    (uint64_t)S.bits[rl][2 * w] | ((uint64_t)S.bits[rl][2 * w + 1] << 32);
        }
    }
}

cudaError_t launch_pairwise(int K, int64_t n_rows, const float *rx, const float *ry, int64_t m,
                            const float *cx, const float *cy, int64_t row_offset, float *iou,
                            float thr, uint64_t *mask, int64_t mask_words, int32_t *nbr_count,
                            int32_t *nbr_idx, int32_t cap, cudaStream_t st)
{
    if (nbr_count) {
        cudaError_t e = cudaMemsetAsync(nbr_count, 0, sizeof(int32_t) * (size_t)n_rows, st);
        if (e != cudaSuccess) return e;
    }
    const dim3 grid((unsigned)((n_rows + kPwRowsPerCta - 1) / kPwRowsPerCta),
                    (unsigned)((m + kPwTileCols - 1) / kPwTileCols));
    if (K == 4) {
        const size_t sm = sizeof(PwSmem<4>);
        static DeviceCache cache;
        const int a = cache.get([&](int) { return set_smem_attr(pairwise_kernel<4>, sm); });
        if (a <= 0) return (cudaError_t)(-a);
        pairwise_kernel<4><<<grid, kPwThreads, sm, st>>>(n_rows, rx, ry, m, cx, cy, row_offset, iou, thr,
                                                         mask, mask_words, nbr_count, nbr_idx, cap);
    } else {
        const size_t sm = sizeof(PwSmem<8>);
        static DeviceCache cache;
        const int a = cache.get([&](int) { return set_smem_attr(pairwise_kernel<8>, sm); });
        if (a <= 0) return (cudaError_t)(-a);
        pairwise_kernel<8><<<grid, kPwThreads, sm, st>>>(n_rows, rx, ry, m, cx, cy, row_offset, iou, thr,
                                                         mask, mask_words, nbr_count, nbr_idx, cap);
    }
    return cudaGetLastError();
}

}  // namespace dgal
