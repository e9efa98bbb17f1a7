// dgal_refine.cuh — the fused kernels' refine pass.
//
// The fused loss kernels compute the IoU and the vertex gradients from float clip
// intervals in one pass.  Two kinds of pair can miss the north_star tolerances
// there: a nearly parallel crossing (a p1 edge crossing a p2 line at |sin| below a
// threshold: float crossing parameters are conditioned by 1/sin; Clip::ill) and a
// thin pair (R^2 > kThinRatio A_u: the float area sum is conditioned by R^2 / A_u).
// Both are rare on the benchmark workloads (cfg3: ~0.01 % and 0.004 % of the
// pairs) and both are exact on the split path (the backward refines
// ill-conditioned crossings in double, dgal_exact.cuh redoes thin areas), so the
// fused kernel only queues them and a second kernel, enqueued right after it,
// redoes the queued pairs with the split path's arithmetic — 32 queued pairs per
// warp, wherever they sit in the batch.
//
// The queue lives in a caller-owned workspace: {count, done, -, -, idx[n]}.  A
// fused-kernel warp appends its marked pairs with one atomicAdd (warp-aggregated);
// the refine kernel reads count, works through idx[0 .. count), and its last CTA
// resets count and done to 0 — so the workspace is all-zero between calls (the
// caller zero-fills it once, include/dgal.h).
#pragma once

#include <cstdint>

namespace dgal {

constexpr int kRefT = 128;   // refine CTA: 128 threads (4 warps)

struct RefineQueue {
    unsigned int count;   // queued pairs
    unsigned int done;    // refine CTAs finished (the last one resets both)
    unsigned int pad[2];
    unsigned int idx[1];  // [n] pair indices
};

// bytes of the workspace for n pairs (16-byte multiple)
inline size_t refine_queue_bytes(int64_t n) { return (size_t)((16 + 4 * (n < 0 ? 0 : n) + 15) / 16) * 16; }

// Queue the warp's marked pairs.  Called by every active lane of the warp.
__device__ __forceinline__ void refine_mark(RefineQueue *__restrict__ q, int64_t k, bool need)
{
    const unsigned act = __activemask();
    const unsigned bal = __ballot_sync(act, need);
    if (bal == 0u) return;
    const int lane = (int)(threadIdx.x & 31), leader = __ffs(bal) - 1;
    unsigned int base = 0;
    if (lane == leader) base = atomicAdd(&q->count, (unsigned int)__popc(bal));
    base = __shfl_sync(act, base, leader);
    if (need) q->idx[base + __popc(bal & ((1u << lane) - 1u))] = (unsigned int)k;
}

// The refine kernel's bookkeeping: the number of queued pairs (read once per CTA,
// before any CTA can reset it) ...
__device__ __forceinline__ unsigned int refine_count(const RefineQueue *q)
{
    return *reinterpret_cast<const volatile unsigned int *>(&q->count);
}

// ... and, by one thread per CTA after the CTA's last read of the queue: the last
// CTA to finish resets the queue for the next call.
__device__ __forceinline__ void refine_finish(RefineQueue *q)
{
    __threadfence();
    if (atomicAdd(&q->done, 1u) == gridDim.x - 1u) {
        q->count = 0u;
        q->done = 0u;
        __threadfence();
    }
}

}  // namespace dgal
