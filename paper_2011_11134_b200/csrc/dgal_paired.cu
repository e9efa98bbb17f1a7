// dgal_paired.cu — paired forward / backward kernels: one thread per
// pair, polygons and clip state in registers, float4 SoA streaming loads.
#include "dgal_core.cuh"
#include "dgal_internal.h"

namespace dgal {

template <int K>
__device__ __forceinline__ void recentre(Poly<K> &P, Poly<K> &Q)
{
    // local origin o = p1.v0 (R11): IoU is translation invariant, and float
    // coordinates near 0 keep the decision predicates accurate.
    const float ox = P.x[0], oy = P.y[0];
#pragma unroll
    for (int k = 0; k < K; ++k) {
        P.x[k] = __fsub_rn(P.x[k], ox); P.y[k] = __fsub_rn(P.y[k], oy);
        Q.x[k] = __fsub_rn(Q.x[k], ox); Q.y[k] = __fsub_rn(Q.y[k], oy);
    }
}

template <int K>
__global__ void __launch_bounds__(kPairedThreads)
paired_fwd_kernel(int64_t n, const float *__restrict__ x1, const float *__restrict__ y1,
                  const float *__restrict__ x2, const float *__restrict__ y2,
                  float *__restrict__ iou, uint8_t *__restrict__ nx, uint8_t *__restrict__ xflags)
{
    const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= n) return;
    Poly<K> P, Q;
    load_poly<K>(x1, y1, k, P);
    load_poly<K>(x2, y2, k, Q);
    recentre<K>(P, Q);
    const FwdOut<K, true> r = iou_fwd<K, true>(P, Q);
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

// K=4: cap registers at 80 so 3 CTAs (24 warps) fit per SM — the backward moves
// 141 B/pair and was latency-bound (long_scoreboard) at 2 CTAs/SM.
template <int K>
__global__ void __launch_bounds__(kPairedThreads, (K == 4) ? 3 : 1)
paired_bwd_kernel(int64_t n, const float *__restrict__ x1, const float *__restrict__ y1,
                  const float *__restrict__ x2, const float *__restrict__ y2,
                  const float *__restrict__ grad, const uint8_t *__restrict__ nx,
                  const uint8_t *__restrict__ xflags,
                  float *__restrict__ gx1, float *__restrict__ gy1,
                  float *__restrict__ gx2, float *__restrict__ gy2)
{
    __shared__ FlagLut lut;
    fill_flag_lut(lut, threadIdx.x, blockDim.x);
    __syncthreads();
    const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= n) return;
    Poly<K> P, Q, G1, G2;
    load_poly<K>(x1, y1, k, P);
    load_poly<K>(x2, y2, k, Q);
    const float g = __ldcs(grad + k);
    const int m = nx[k];
    Seq<K> s;
    if (K == 4) {
        s.w[0] = __ldcs(reinterpret_cast<const unsigned long long *>(xflags) + k);
    } else {
        const ulonglong2 v = __ldcs(reinterpret_cast<const ulonglong2 *>(xflags) + k);
        s.w[0] = v.x;
        s.w[Seq<K>::NW - 1] = v.y;
    }
    recentre<K>(P, Q);
    iou_bwd<K>(P, Q, g, m, s, lut, G1, G2);
    store_plane<K>(gx1, k, G1.x);
    store_plane<K>(gy1, k, G1.y);
    store_plane<K>(gx2, k, G2.x);
    store_plane<K>(gy2, k, G2.y);
}

static inline unsigned grid_for(int64_t n) { return (unsigned)((n + kPairedThreads - 1) / kPairedThreads); }

cudaError_t launch_paired_fwd(int K, int64_t n, const float *x1, const float *y1, const float *x2,
                              const float *y2, float *iou, uint8_t *nx, uint8_t *xflags,
                              cudaStream_t st)
{
    if (K == 4)
        paired_fwd_kernel<4><<<grid_for(n), kPairedThreads, 0, st>>>(n, x1, y1, x2, y2, iou, nx, xflags);
    else
        paired_fwd_kernel<8><<<grid_for(n), kPairedThreads, 0, st>>>(n, x1, y1, x2, y2, iou, nx, xflags);
    return cudaGetLastError();
}

cudaError_t launch_paired_bwd(int K, int64_t n, const float *x1, const float *y1, const float *x2,
                              const float *y2, const float *grad, const uint8_t *nx,
                              const uint8_t *xflags, float *gx1, float *gy1, float *gx2, float *gy2,
                              cudaStream_t st)
{
    if (K == 4)
        paired_bwd_kernel<4><<<grid_for(n), kPairedThreads, 0, st>>>(n, x1, y1, x2, y2, grad, nx, xflags,
                                                                     gx1, gy1, gx2, gy2);
    else
        paired_bwd_kernel<8><<<grid_for(n), kPairedThreads, 0, st>>>(n, x1, y1, x2, y2, grad, nx, xflags,
                                                                     gx1, gy1, gx2, gy2);
    return cudaGetLastError();
}

}  // namespace dgal
