// dgal_nms.cu — greedy rotated-NMS keep decision by parallel rounds.
//
// Greedy NMS (boxes sorted by score; keep i iff no KEPT k < i has IoU(i,k) > thr)
// is the unique solution of keep(i) = not exists k < i: keep(k) and S(k, i).
// Rounds: an undecided box with a kept suppressor is removed; one whose
// suppressors are all removed is kept.  Every decision is final and correct by
// induction on the index, and the smallest undecided box always decides, so the
// rounds terminate with exactly the greedy result; in practice the number of
// rounds is the length of the longest suppression chain (a handful).
// Status bytes: 0 undecided, 1 kept, 2 removed.
#include <cooperative_groups.h>

#include "dgal_internal.h"

namespace dgal {

__device__ __forceinline__ int decide(int64_t r, int64_t i, const uint64_t *__restrict__ mask,
                                      int64_t mask_words, const int32_t *__restrict__ nbr_count,
                                      const int32_t *__restrict__ nbr_idx, int32_t cap,
                                      const volatile uint8_t *status)
{
    bool any_kept = false, all_removed = true;
    const int cnt = nbr_count ? nbr_count[r] : -1;
    if (cnt >= 0 && cnt <= cap) {
        const int32_t *lst = nbr_idx + r * cap;
        for (int k = 0; k < cnt; ++k) {
            DGAL_ASSERT(lst[k] >= 0 && lst[k] < i);
            const uint8_t s = status[lst[k]];
            any_kept |= (s == 1);
            all_removed &= (s == 2);
        }
    } else {
        // overflowed (or absent) list: scan the lower part of the mask row
        const uint64_t *row = mask + r * mask_words;
        const int64_t last = i >> 6;
        for (int64_t w = 0; w <= last; ++w) {
            uint64_t b = row[w];
            if (w == last) b &= (i & 63) ? ((1ull << (i & 63)) - 1ull) : 0ull;  // columns < i only
            while (b) {
                const int j = __ffsll((long long)b) - 1;
                b &= b - 1;
                const uint8_t s = status[(w << 6) + j];
                any_kept |= (s == 1);
                all_removed &= (s == 2);
            }
        }
    }
    return any_kept ? 2 : (all_removed ? 1 : 0);
}

__global__ void __launch_bounds__(kNmsRoundThreads)
nms_round_kernel(int64_t n_rows, int64_t row_offset, const uint64_t *__restrict__ mask,
                 int64_t mask_words, const int32_t *__restrict__ nbr_count,
                 const int32_t *__restrict__ nbr_idx, int32_t cap, uint8_t *status, int32_t *undecided)
{
    const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    int still = 0;
    if (r < n_rows) {
        const int64_t i = row_offset + r;
        volatile uint8_t *vs = status;
        if (vs[i] == 0) {
            const int d = decide(r, i, mask, mask_words, nbr_count, nbr_idx, cap, vs);
            if (d) vs[i] = (uint8_t)d;
            else still = 1;
        }
    }
    // one atomic per warp
    const unsigned b = __ballot_sync(0xFFFFFFFFu, still);
    if ((threadIdx.x & 31) == 0 && b) atomicAdd(undecided, __popc(b));
}

__global__ void __launch_bounds__(kNmsKeepThreads)
nms_keep_kernel(int64_t n, const uint64_t *__restrict__ mask, int64_t mask_words,
                const int32_t *__restrict__ nbr_count, const int32_t *__restrict__ nbr_idx,
                int32_t cap, uint8_t *status, uint8_t *__restrict__ keep)
{
    __shared__ int s_undecided;
    volatile uint8_t *vs = status;
    for (int64_t i = threadIdx.x; i < n; i += blockDim.x) vs[i] = 0;
    __syncthreads();
    for (;;) {
        if (threadIdx.x == 0) s_undecided = 0;
        __syncthreads();
        int still = 0;
        for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
            if (vs[i] != 0) continue;
            const int d = decide(i, i, mask, mask_words, nbr_count, nbr_idx, cap, vs);
            if (d) vs[i] = (uint8_t)d;
            else ++still;
        }
        if (still) atomicAdd(&s_undecided, still);
        __syncthreads();
        const int u = s_undecided;
        __syncthreads();
        if (u == 0) break;
    }
    for (int64_t i = threadIdx.x; i < n; i += blockDim.x) keep[i] = (vs[i] == 1) ? 1 : 0;
}

// A round to the rank-local fixed point (dgal_nms_round with scratch): passes over
// the rank's rows, grid barriers between them, until a pass decides nothing new
// (the other ranks' entries of status are constant during the round).  Within
// one rank every suppression chain resolves in this one round; only chains that
// cross ranks need further rounds (exchanges).  Progress of pass p goes to
// cnt[p & 1]; the last pass (no progress) counts the undecided rows.
__global__ void __launch_bounds__(kNmsRoundThreads)
nms_round_grid_kernel(int64_t n_rows, int64_t row_offset, const uint64_t *__restrict__ mask, int64_t mask_words,
                      const int32_t *__restrict__ nbr_count, const int32_t *__restrict__ nbr_idx, int32_t cap,
                      uint8_t *status, int32_t *undecided, int32_t *cnt)
{
    namespace cg = cooperative_groups;
    cg::grid_group grid = cg::this_grid();
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    const int64_t t0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    volatile uint8_t *vs = status;
    if (t0 == 0) { cnt[0] = 0; cnt[1] = 0; }
    grid.sync();
    for (int p = 0;; ++p) {
        volatile int32_t *c = cnt + (p & 1);
        if (t0 == 0) cnt[(p + 1) & 1] = 0;
        int prog = 0, still = 0;
        for (int64_t r = t0; r < n_rows; r += stride) {
            const int64_t i = row_offset + r;
            if (vs[i] != 0) continue;
            const int d = decide(r, i, mask, mask_words, nbr_count, nbr_idx, cap, vs);
            if (d) { vs[i] = (uint8_t)d; ++prog; }
            else ++still;
        }
#pragma unroll
        for (int d = 16; d > 0; d >>= 1) {
            prog += __shfl_down_sync(0xFFFFFFFFu, prog, d);
            still += __shfl_down_sync(0xFFFFFFFFu, still, d);
        }
        if ((threadIdx.x & 31) == 0 && prog) atomicAdd((int32_t *)c, prog);
        grid.sync();
        if (*c == 0) {           // the same value for every thread (read after the barrier)
            if ((threadIdx.x & 31) == 0 && still) atomicAdd(undecided, still);
            break;
        }
        grid.sync();             // everyone has read c before it is cleared again (pass p + 2)
    }
}

cudaError_t launch_nms_round(int64_t n_total, int64_t n_rows, int64_t row_offset,
                             const uint64_t *mask, int64_t mask_words, const int32_t *nbr_count,
                             const int32_t *nbr_idx, int32_t cap, uint8_t *status, int32_t *undecided,
                             int32_t *scratch, cudaStream_t st)
{
    (void)n_total;
    if (scratch) {
        static DeviceCache cache;   // co-resident grid size (-1: no cooperative launch)
        const int limit = cache.get([&](int dev) {
            int sms = 0, per = 0, coop = 0;
            cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
            cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, dev);
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, nms_round_grid_kernel, kNmsRoundThreads, 0);
            return coop ? sms * (per > 0 ? per : 1) : -1;
        });
        if (limit > 0) {
            const int64_t need = (n_rows + kNmsRoundThreads - 1) / kNmsRoundThreads;
            unsigned grid = (unsigned)(need < limit ? need : limit);
            void *args[] = {&n_rows, &row_offset, (void *)&mask, &mask_words, (void *)&nbr_count,
                            (void *)&nbr_idx, &cap, &status, &undecided, &scratch};
            return cudaLaunchCooperativeKernel((const void *)nms_round_grid_kernel, dim3(grid),
                                               dim3(kNmsRoundThreads), args, 0, st);
        }
    }
    const unsigned grid = (unsigned)((n_rows + kNmsRoundThreads - 1) / kNmsRoundThreads);
    nms_round_kernel<<<grid, kNmsRoundThreads, 0, st>>>(n_rows, row_offset, mask, mask_words, nbr_count,
                                                        nbr_idx, cap, status, undecided);
    return cudaGetLastError();
}

// All rounds grid-wide: a cooperative launch (every CTA resident), one box per
// thread per round, grid barriers between rounds.  The undecided count of round r
// goes to cnt[r & 1]; cnt[(r + 1) & 1] is cleared during round r, before anyone
// can add to it (round r + 1 starts after the barrier).
__global__ void __launch_bounds__(kNmsRoundThreads)
nms_keep_grid_kernel(int64_t n, const uint64_t *__restrict__ mask, int64_t mask_words,
                     const int32_t *__restrict__ nbr_count, const int32_t *__restrict__ nbr_idx, int32_t cap,
                     uint8_t *status, uint8_t *__restrict__ keep, int32_t *cnt)
{
    namespace cg = cooperative_groups;
    cg::grid_group grid = cg::this_grid();
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    const int64_t t0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    volatile uint8_t *vs = status;
    for (int64_t i = t0; i < n; i += stride) vs[i] = 0;
    if (t0 == 0) { cnt[0] = 0; cnt[1] = 0; }
    grid.sync();
    for (int r = 0;; ++r) {
        volatile int32_t *c = cnt + (r & 1);
        if (t0 == 0) cnt[(r + 1) & 1] = 0;
        int still = 0;
        for (int64_t i = t0; i < n; i += stride) {
            DGAL_ASSERT(i >= 0 && i < n);
            if (vs[i] != 0) continue;
            const int d = decide(i, i, mask, mask_words, nbr_count, nbr_idx, cap, vs);
            if (d) vs[i] = (uint8_t)d;
            else ++still;
        }
        const unsigned b = __ballot_sync(0xFFFFFFFFu, still != 0);
        if (b) {
            // warp sum of the (small) counts
            int v = still;
#pragma unroll
            for (int d = 16; d > 0; d >>= 1) v += __shfl_down_sync(0xFFFFFFFFu, v, d);
            if ((threadIdx.x & 31) == 0) atomicAdd((int32_t *)c, v);
        }
        grid.sync();
        if (*c == 0) break;      // the same value for every thread (read after the barrier)
        grid.sync();             // everyone has read c before it is cleared again (round r + 2)
    }
    for (int64_t i = t0; i < n; i += stride) keep[i] = (vs[i] == 1) ? 1 : 0;
}

cudaError_t launch_nms_keep(int64_t n, const uint64_t *mask, int64_t mask_words,
                            const int32_t *nbr_count, const int32_t *nbr_idx, int32_t cap,
                            uint8_t *status, uint8_t *keep, int32_t *scratch, cudaStream_t st)
{
    if (scratch) {
        static DeviceCache cache;   // co-resident grid size (-1: no cooperative launch)
        const int limit = cache.get([&](int dev) {
            int sms = 0, per = 0, coop = 0;
            cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
            cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, dev);
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, nms_keep_grid_kernel, kNmsRoundThreads, 0);
            return coop ? sms * (per > 0 ? per : 1) : -1;
        });
        if (limit > 0) {
            const int64_t need = (n + kNmsRoundThreads - 1) / kNmsRoundThreads;
            unsigned grid = (unsigned)(need < limit ? need : limit);
            void *args[] = {&n, (void *)&mask, &mask_words, (void *)&nbr_count, (void *)&nbr_idx, &cap, &status,
                            &keep, &scratch};
            return cudaLaunchCooperativeKernel((const void *)nms_keep_grid_kernel, dim3(grid),
                                               dim3(kNmsRoundThreads), args, 0, st);
        }
    }
    nms_keep_kernel<<<1, kNmsKeepThreads, 0, st>>>(n, mask, mask_words, nbr_count, nbr_idx, cap, status,
                                                   keep);
    return cudaGetLastError();
}

}  // namespace dgal
