// dgal_pairwise.cu — N x M pairwise IoU + NMS overlap mask (north_star; S:506-513
// "cartesian").  DESIGN.md §4.3.
//
// CTA = 8 warps, one 1024-column tile of p2 polygons staged in shared memory
// (vertices + bounding circles) and reused by the CTA's 64 rows.  A warp owns one
// row at a time and sweeps the tile 128 columns per step, 4 consecutive columns
// per lane:
//   * bounding-circle reject (exact: disjoint circles => disjoint polygons),
//   * a float4 streaming store of zeros for the 4 columns (the output write is
//     the binding roof of the large matrix),
//   * survivors are compacted with __ballot_sync/__popc into a per-warp shared
//     queue and evaluated 32 at a time, one per lane, so the clip runs with full
//     SIMT efficiency however rare candidates are;
//   * candidate results overwrite their zero, set their mask bit in a per-warp
//     shared bitmap (atomicOr on shared), and (c < row) append to the row's
//     suppressor list; the bitmap goes out as whole uint64 words at row end.
#include "dgal_core.cuh"
#include "dgal_internal.h"

namespace dgal {

namespace {

constexpr unsigned kFull = 0xFFFFFFFFu;

template <int K>
__device__ __forceinline__ float4 bounding_circle(const Poly<K> &p)
{
    float cx = 0.f, cy = 0.f;
#pragma unroll
    for (int k = 0; k < K; ++k) { cx += p.x[k]; cy += p.y[k]; }
    cx *= (1.f / K);
    cy *= (1.f / K);
    float r2 = 0.f;
#pragma unroll
    for (int k = 0; k < K; ++k) {
        const float dx = p.x[k] - cx, dy = p.y[k] - cy;
        r2 = fmaxf(r2, dx * dx + dy * dy);
    }
    // inflate: relative (sqrt/rounding) + absolute (ulp of the scene coordinates)
    const float r = sqrtf(r2) * 1.0001f + 2e-6f * (fabsf(cx) + fabsf(cy)) + 1e-30f;
    return make_float4(cx, cy, r, 0.f);
}

template <int K>
__device__ __forceinline__ void load_poly_cached(const float *__restrict__ X, const float *__restrict__ Y,
                                                 int64_t n, Poly<K> &p)
{
    const float4 *x4 = reinterpret_cast<const float4 *>(X + n * K);
    const float4 *y4 = reinterpret_cast<const float4 *>(Y + n * K);
#pragma unroll
    for (int q = 0; q < K / 4; ++q) {
        float4 a = __ldg(x4 + q), b = __ldg(y4 + q);
        p.x[4 * q + 0] = a.x; p.x[4 * q + 1] = a.y; p.x[4 * q + 2] = a.z; p.x[4 * q + 3] = a.w;
        p.y[4 * q + 0] = b.x; p.y[4 * q + 1] = b.y; p.y[4 * q + 2] = b.z; p.y[4 * q + 3] = b.w;
    }
}

template <int K>
struct PwSmem {
    float x[kPwTileCols * K];
    float y[kPwTileCols * K];
    float4 circ[kPwTileCols];
    int queue[kPwWarps][kPwQueueCap];
    uint32_t bits[kPwWarps][kPwTileCols / 32];
};

}  // namespace

template <int K>
__global__ void __launch_bounds__(kPwThreads)
pairwise_kernel(int64_t n_rows, const float *__restrict__ rx, const float *__restrict__ ry, int64_t m,
                const float *__restrict__ cx, const float *__restrict__ cy, int64_t row_offset,
                float *__restrict__ iou, float thr, uint64_t *__restrict__ mask, int64_t mask_words,
                int32_t *__restrict__ nbr_count, int32_t *__restrict__ nbr_idx, int32_t cap)
{
    extern __shared__ __align__(16) unsigned char smem_raw[];
    PwSmem<K> &S = *reinterpret_cast<PwSmem<K> *>(smem_raw);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t c0 = (int64_t)blockIdx.y * kPwTileCols;
    const int ncols = (int)min((int64_t)kPwTileCols, m - c0);

    // ---- stage the column tile: vertices + bounding circles ----
    for (int t = threadIdx.x; t < kPwTileCols; t += kPwThreads) {
        if (t < ncols) {
            Poly<K> q;
            load_poly_cached<K>(cx, cy, c0 + t, q);
#pragma unroll
            for (int k = 0; k < K; ++k) { S.x[t * K + k] = q.x[k]; S.y[t * K + k] = q.y[k]; }
            S.circ[t] = bounding_circle<K>(q);
        } else {
            S.circ[t] = make_float4(__int_as_float(0x7f800000), __int_as_float(0x7f800000), 0.f, 0.f);
        }
    }
    for (int t = lane; t < kPwTileCols / 32; t += 32) S.bits[warp][t] = 0u;
    __syncthreads();

    const bool vec_store = iou != nullptr && (m % 4 == 0) &&
                           ((reinterpret_cast<uintptr_t>(iou) & 15u) == 0);
    const unsigned lt_mask = (1u << lane) - 1u;
    int *queue = S.queue[warp];
    uint32_t *bits = S.bits[warp];

    const int64_t r_end = min(n_rows, (int64_t)(blockIdx.x + 1) * kPwRowsPerCta);
    for (int64_t r = (int64_t)blockIdx.x * kPwRowsPerCta + warp; r < r_end; r += kPwWarps) {
        Poly<K> P;
        load_poly_cached<K>(rx, ry, r, P);  // warp-uniform row: broadcast loads
        const float4 rc = bounding_circle<K>(P);
        const float ox = P.x[0], oy = P.y[0];
        Poly<K> Pc;
#pragma unroll
        for (int k = 0; k < K; ++k) { Pc.x[k] = __fsub_rn(P.x[k], ox); Pc.y[k] = __fsub_rn(P.y[k], oy); }
        const int64_t grow = row_offset + r;
        float *iou_row = iou ? iou + r * m + c0 : nullptr;

        auto evaluate = [&](int e) {
            Poly<K> Qc;
#pragma unroll
            for (int k = 0; k < K; ++k) {
                Qc.x[k] = __fsub_rn(S.x[e * K + k], ox);
                Qc.y[k] = __fsub_rn(S.y[e * K + k], oy);
            }
            const float v = iou_fwd<K, false>(Pc, Qc).iou;
            if (iou_row) iou_row[e] = v;
            const int64_t c = c0 + e;
            if (v > thr && c != grow) {
                if (mask) atomicOr(&bits[e >> 5], 1u << (e & 31));
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
            bool cand[4];
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const float4 cc = S.circ[cb + q];
                const float dx = cc.x - rc.x, dy = cc.y - rc.y, rs = cc.z + rc.z;
                cand[q] = dx * dx + dy * dy < rs * rs;
            }
            if (iou_row) {
                if (vec_store && cb + 3 < ncols) {
                    __stcs(reinterpret_cast<float4 *>(iou_row + cb), make_float4(0.f, 0.f, 0.f, 0.f));
                } else {
#pragma unroll
                    for (int q = 0; q < 4; ++q)
                        if (cb + q < ncols) __stcs(iou_row + cb + q, 0.f);
                }
            }
            if (__any_sync(kFull, cand[0] | cand[1] | cand[2] | cand[3])) {
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    const unsigned bal = __ballot_sync(kFull, cand[q]);
                    if (cand[q]) queue[qn + __popc(bal & lt_mask)] = cb + q;
                    qn += __popc(bal);
                }
                __syncwarp();
                while (qn >= 32) {           // warp-uniform
                    evaluate(queue[qn - 32 + lane]);
                    qn -= 32;
                    __syncwarp();
                }
            }
        }
        __syncwarp();
        if (lane < qn) evaluate(queue[lane]);
        __syncwarp();
        if (mask) {
            const int nw = (ncols + 63) >> 6;
            const int64_t w0 = c0 >> 6;
            for (int w = lane; w < nw; w += 32) {
                if (w0 + w < mask_words) {
                    const uint64_t word = (uint64_t)bits[2 * w] | ((uint64_t)bits[2 * w + 1] << 32);
                    mask[r * mask_words + w0 + w] = word;
                }
                bits[2 * w] = 0u;
                bits[2 * w + 1] = 0u;
            }
            __syncwarp();
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
        static bool attr4 = false;
        if (!attr4) {
            cudaFuncSetAttribute(pairwise_kernel<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
            attr4 = true;
        }
        pairwise_kernel<4><<<grid, kPwThreads, sm, st>>>(n_rows, rx, ry, m, cx, cy, row_offset, iou, thr,
                                                         mask, mask_words, nbr_count, nbr_idx, cap);
    } else {
        const size_t sm = sizeof(PwSmem<8>);
        static bool attr8 = false;
        if (!attr8) {
            cudaFuncSetAttribute(pairwise_kernel<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
            attr8 = true;
        }
        pairwise_kernel<8><<<grid, kPwThreads, sm, st>>>(n_rows, rx, ry, m, cx, cy, row_offset, iou, thr,
                                                         mask, mask_words, nbr_count, nbr_idx, cap);
    }
    return cudaGetLastError();
}

}  // namespace dgal
