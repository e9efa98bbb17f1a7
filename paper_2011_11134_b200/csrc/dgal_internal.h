// dgal_internal.h — launch configuration and launcher prototypes shared by the
// .cu translation units of libdgal.so (not part of the public ABI).
#pragma once

#include <atomic>
#include <cassert>
#include <cstdint>
#include <cuda_runtime.h>

// Checked build (-DDGAL_CHECKED, libdgal_checked.so): device-side bounds asserts on
// every dynamic shared / global index (compute-sanitizer is not available on the
// GPU pool).  Compiled out of the release library.
#ifdef DGAL_CHECKED
#define DGAL_ASSERT(x) assert(x)
#else
#define DGAL_ASSERT(x) ((void)0)
#endif

namespace dgal {

// Per-device, per-launcher cache of a launch-configuration value (a kernel's
// dynamic-shared-memory attribute having been set, a co-resident grid size).
// The value is a pure function of (device, kernel), so racing first calls just
// compute it twice; each device has its own slot (one process may drive several
// GPUs from several threads).  0 = not yet known; a failed computation (<= 0) is
// not cached.  This is the only state the library keeps.
constexpr int kMaxDevices = 64;
struct DeviceCache {
    std::atomic<int> v[kMaxDevices];
    template <class F>
    int get(F compute)
    {
        int dev = 0;
        if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= kMaxDevices) return compute(dev);
        int x = v[dev].load(std::memory_order_relaxed);
        if (x <= 0) {
            x = compute(dev);
            if (x > 0) v[dev].store(x, std::memory_order_relaxed);
        }
        return x;
    }
};
// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) once per device: 1, or -error
template <class K>
int set_smem_attr(K kernel, size_t bytes)
{
    const cudaError_t e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
    return e == cudaSuccess ? 1 : -(int)e;
}

constexpr int kPairedThreads = 256;     // paired kernels: one pair per thread

// pairwise kernel geometry
constexpr int kPwThreads = 256;         // 8 warps
constexpr int kPwWarps = kPwThreads / 32;
constexpr int kPwTileCols = 1024;       // column tile staged in shared memory
constexpr int kPwRowsPerCta = 64;       // row block per CTA (8 rows per warp)
// (the per-warp candidate queue is sized in dgal_pairwise.cu)

constexpr int kNmsKeepThreads = 1024;   // single-CTA keep kernel
constexpr int kNmsRoundThreads = 256;

cudaError_t launch_paired_fwd(int K, int64_t n, const float *x1, const float *y1, const float *x2,
                              const float *y2, float *iou, uint8_t *nx, uint8_t *xflags,
                              cudaStream_t st);
cudaError_t launch_paired_bwd(int K, int64_t n, const float *x1, const float *y1, const float *x2,
                              const float *y2, const float *grad, const uint8_t *nx,
                              const uint8_t *xflags, float *gx1, float *gy1, float *gx2, float *gy2,
                              cudaStream_t st);
cudaError_t launch_paired_fused(int K, int64_t n, const float *x1, const float *y1, const float *x2,
                                const float *y2, const float *grad, float scale, float *iou, float *gx1,
                                float *gy1, float *gx2, float *gy2, void *refine, cudaStream_t st);
int refine_grid_for(int64_t n);   // grid of the fused kernels' refine pass (dgal_refine.cuh)
constexpr int64_t kMaxFusedPairs = 0xFFFFFFFFll;   // queue entries are 32-bit pair indices
size_t refine_workspace_bytes(int64_t n);
cudaError_t launch_box_fwd(int dims, int layout, int64_t n, const float *b1, const float *b2, float *iou,
                           uint8_t *nx, uint8_t *xflags, cudaStream_t st);
cudaError_t launch_box_bwd(int dims, int layout, int64_t n, const float *b1, const float *b2, const float *grad,
                           const uint8_t *nx, const uint8_t *xflags, float *gb1, float *gb2, cudaStream_t st);
cudaError_t launch_box_fused(int dims, int layout, int64_t n, const float *b1, const float *b2, const float *grad,
                             float scale, float *iou, float *gb1, float *gb2, void *refine, cudaStream_t st);
cudaError_t launch_pairwise(int K, int64_t n_rows, const float *rx, const float *ry, int64_t m,
                            const float *cx, const float *cy, int64_t row_offset, float *iou,
                            float thr, uint64_t *mask, int64_t mask_words, int32_t *nbr_count,
                            int32_t *nbr_idx, int32_t cap, cudaStream_t st);
size_t pairwise_workspace_bytes(int64_t m);
cudaError_t launch_pairwise_indexed(int K, int64_t n_rows, const float *rx, const float *ry, int64_t m,
                                    const float *cx, const float *cy, int64_t row_offset, float *iou,
                                    float thr, uint64_t *mask, int64_t mask_words, int32_t *nbr_count,
                                    int32_t *nbr_idx, int32_t cap, void *workspace, cudaStream_t st);
cudaError_t launch_nms_round(int64_t n_total, int64_t n_rows, int64_t row_offset,
                             const uint64_t *mask, int64_t mask_words, const int32_t *nbr_count,
                             const int32_t *nbr_idx, int32_t cap, uint8_t *status, int32_t *undecided,
                             int32_t *scratch, cudaStream_t st);
cudaError_t launch_nms_keep(int64_t n, const uint64_t *mask, int64_t mask_words,
                            const int32_t *nbr_count, const int32_t *nbr_idx, int32_t cap,
                            uint8_t *status, uint8_t *keep, int32_t *scratch, cudaStream_t st);

}  // namespace dgal
