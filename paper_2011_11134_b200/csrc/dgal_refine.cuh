// dgal_refine.cuh — the fused kernels' refine pass.
//
// The fused loss kernels compute the IoU and the vertex gradients from float clip
// intervals in one pass.  Two kinds of pair can miss the north_star tolerances
// there: a nearly parallel (p1 edge, p2 edge) pair, whose crossing parameters are
// conditioned by 1/sin (Clip::ill), and a thin pair, whose area sum is conditioned
// by R^2 / A_u (pair_is_thin).  Both are rare on the benchmark workloads (cfg3:
// ~1.5 % and 0.004 %) and both are exact on the split path (the backward refines
// ill-conditioned crossings in double, dgal_exact.cuh redoes thin areas), so the
// fused kernel only marks them — one bit per pair in a caller-owned refine mask —
// and a second kernel redoes the marked pairs with the split path's arithmetic,
// compacted so each warp works on 32 marked pairs:
//
//   mask word w covers pairs 32w .. 32w+31 (bit = pair & 31).  A fused-kernel warp
//   owns exactly one word (its 32 consecutive pairs) and stores it, whole, only
//   when a bit is set; the refine pass reads every word, clears the non-zero ones
//   and queues their pairs in shared memory.  The mask is therefore all-zero
//   between calls (the caller zero-fills it once, include/dgal.h).
#pragma once

#include <cstdint>

namespace dgal {

constexpr int kRefT = 128;                            // refine CTA: 128 threads (4 warps)
constexpr int kRefWordsPerThread = 2;                 // one 8-byte load per thread per chunk
constexpr int kRefChunkWords = kRefT * kRefWordsPerThread;   // 256 words = 8192 pairs per chunk
constexpr int kRefChunkPairs = kRefChunkWords * 32;

__host__ __device__ inline int64_t refine_words(int64_t n) { return (n + 31) / 32; }
// bytes of the refine mask for n pairs: whole 8-byte vectors (the pass loads uint2)
inline size_t refine_mask_bytes(int64_t n) { return (size_t)((refine_words(n) + 1) / 2) * 8; }

// A warp's marks: lanes map to consecutive pairs k = 32w + lane (all fused kernels
// lay pairs out that way).  Called by every active lane of the warp.
__device__ __forceinline__ void refine_mark(uint32_t *__restrict__ mask, int64_t k, bool need)
{
    const unsigned act = __activemask();
    const unsigned bal = __ballot_sync(act, need);
    if (bal != 0u && (int)(threadIdx.x & 31) == __ffs(bal) - 1) mask[k >> 5] = bal;
}

// Gather the marked pairs of chunk c into q[0 .. *qn) as offsets from the chunk's
// first pair, clearing their words.  All threads of the CTA; the caller syncs.
__device__ __forceinline__ void refine_gather(uint32_t *__restrict__ mask, int64_t nwords, int64_t c,
                                              uint16_t *q, int *qn)
{
    const int64_t w0 = c * kRefChunkWords + (int64_t)threadIdx.x * kRefWordsPerThread;
    if (w0 >= nwords) return;
    const uint2 v = *reinterpret_cast<const uint2 *>(mask + w0);   // words past nwords are 0 (padding)
    const uint32_t wv[2] = {v.x, v.y};
    if ((v.x | v.y) == 0u) return;
    *reinterpret_cast<uint2 *>(mask + w0) = make_uint2(0u, 0u);
#pragma unroll
    for (int u = 0; u < kRefWordsPerThread; ++u) {
        uint32_t b = wv[u];
        if (!b) continue;
        int at = atomicAdd(qn, __popc(b));
        const int off = (threadIdx.x * kRefWordsPerThread + u) * 32;
        while (b) {
            const int bit = __ffs(b) - 1;
            b &= b - 1u;
            q[at++] = (uint16_t)(off + bit);
        }
    }
}

}  // namespace dgal
