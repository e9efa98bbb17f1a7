// dgal_api.cu — the extern "C" boundary of libdgal.so (include/dgal.h): host-side
// argument validation, K dispatch, launch on the caller's stream.  No memory
// allocation, no host synchronisation; the only global state is the host-buffer
// call's per-device streams and events.
#include <climits>
#include <cstdint>
#include <mutex>

#include "../../include/dgal.h"
#include "dgal_internal.h"

#ifndef DGAL_VERSION
#define DGAL_VERSION "0.1.0"
#endif

namespace {

inline bool aligned(const void *p, uintptr_t a) { return (reinterpret_cast<uintptr_t>(p) & (a - 1)) == 0; }

inline dgal_status from_cuda(cudaError_t e) { return e == cudaSuccess ? DGAL_OK : DGAL_ERR_CUDA; }

inline cudaStream_t as_cuda(dgal_stream s) { return reinterpret_cast<cudaStream_t>(s); }

// dgal_iou_paired_host: one staging slot per pipeline stream, carved from the
// caller's device workspace (256-byte aligned pieces)
constexpr int kHostStreams = 3;
inline size_t a256(size_t b) { return (b + 255) & ~(size_t)255; }

struct HostSlot {
    float *x1, *y1, *x2, *y2, *g, *iou, *gx1, *gy1, *gx2, *gy2;
    uint8_t *nx, *xf;
};

inline size_t host_slot_bytes(int K, int64_t chunk)
{
    const size_t c = (size_t)chunk;
    return 8 * a256(sizeof(float) * c * K) + 2 * a256(sizeof(float) * c) + a256(c) + a256(c * 2 * K);
}

inline HostSlot host_slot(void *ws, int K, int64_t chunk, int s)
{
    const size_t c = (size_t)chunk;
    char *p = static_cast<char *>(ws) + (size_t)s * host_slot_bytes(K, chunk);
    auto take = [&](size_t b) { char *q = p; p += a256(b); return q; };
    HostSlot h;
    float **planes[8] = {&h.x1, &h.y1, &h.x2, &h.y2, &h.gx1, &h.gy1, &h.gx2, &h.gy2};
    for (float **q : planes) *q = reinterpret_cast<float *>(take(sizeof(float) * c * K));
    h.g = reinterpret_cast<float *>(take(sizeof(float) * c));
    h.iou = reinterpret_cast<float *>(take(sizeof(float) * c));
    h.nx = reinterpret_cast<uint8_t *>(take(c));
    h.xf = reinterpret_cast<uint8_t *>(take(c * 2 * K));
    return h;
}

struct HostPipe {
    std::mutex mu;
    bool init = false;
    cudaStream_t s[kHostStreams] = {};
    cudaEvent_t fork = nullptr, join[kHostStreams] = {};
};
HostPipe g_host_pipe[64];

}  // namespace

extern "C" {

dgal_status dgal_iou_paired_fwd(int K, int64_t n, const float *x1, const float *y1, const float *x2,
                                const float *y2, float *iou, uint8_t *nx, uint8_t *xflags,
                                dgal_stream stream)
{
    if (K != 4 && K != 8) return DGAL_ERR_UNSUPPORTED_K;
    if (n < 0) return DGAL_ERR_INVALID_ARG;
    if (n == 0) return DGAL_OK;
    if (!x1 || !y1 || !x2 || !y2 || !iou || !nx || !xflags) return DGAL_ERR_INVALID_ARG;
    if (!aligned(x1, 16) || !aligned(y1, 16) || !aligned(x2, 16) || !aligned(y2, 16) ||
        !aligned(xflags, (uintptr_t)(2 * K)))
        return DGAL_ERR_MISALIGNED;
    return from_cuda(dgal::launch_paired_fwd(K, n, x1, y1, x2, y2, iou, nx, xflags, as_cuda(stream)));
}

dgal_status dgal_iou_paired_bwd(int K, int64_t n, const float *x1, const float *y1, const float *x2,
                                const float *y2, const float *grad_iou, const uint8_t *nx,
                                const uint8_t *xflags, float *gx1, float *gy1, float *gx2, float *gy2,
                                dgal_stream stream)
{
    if (K != 4 && K != 8) return DGAL_ERR_UNSUPPORTED_K;
    if (n < 0) return DGAL_ERR_INVALID_ARG;
    if (n == 0) return DGAL_OK;
    if (!x1 || !y1 || !x2 || !y2 || !grad_iou || !nx || !xflags || !gx1 || !gy1 || !gx2 || !gy2)
        return DGAL_ERR_INVALID_ARG;
    if (!aligned(x1, 16) || !aligned(y1, 16) || !aligned(x2, 16) || !aligned(y2, 16) ||
        !aligned(gx1, 16) || !aligned(gy1, 16) || !aligned(gx2, 16) || !aligned(gy2, 16) ||
        !aligned(xflags, (uintptr_t)(2 * K)))
        return DGAL_ERR_MISALIGNED;
    return from_cuda(dgal::launch_paired_bwd(K, n, x1, y1, x2, y2, grad_iou, nx, xflags, gx1, gy1, gx2,
                                             gy2, as_cuda(stream)));
}

size_t dgal_paired_host_workspace_bytes(int K, int64_t chunk)
{
    if ((K != 4 && K != 8) || chunk <= 0) return 0;
    return kHostStreams * host_slot_bytes(K, chunk);
}

dgal_status dgal_iou_paired_host(int K, int64_t n, const float *x1, const float *y1, const float *x2,
                                 const float *y2, const float *grad_iou, float *iou, float *gx1, float *gy1,
                                 float *gx2, float *gy2, int64_t chunk, void *workspace,
                                 size_t workspace_bytes, dgal_stream stream)
{
    if (K != 4 && K != 8) return DGAL_ERR_UNSUPPORTED_K;
    if (n < 0 || chunk <= 0 || (chunk & 3)) return DGAL_ERR_INVALID_ARG;
    if (n == 0) return DGAL_OK;
    if (!x1 || !y1 || !x2 || !y2 || !grad_iou || !iou || !gx1 || !gy1 || !gx2 || !gy2 || !workspace)
        return DGAL_ERR_INVALID_ARG;
    if (workspace_bytes < dgal_paired_host_workspace_bytes(K, chunk)) return DGAL_ERR_INVALID_ARG;
    if (!aligned(workspace, 256)) return DGAL_ERR_MISALIGNED;
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return DGAL_ERR_CUDA;
    HostPipe &hp = g_host_pipe[dev];
    std::lock_guard<std::mutex> lock(hp.mu);
    if (!hp.init) {
        for (int i = 0; i < kHostStreams; ++i) {
            if (cudaStreamCreateWithFlags(&hp.s[i], cudaStreamNonBlocking) != cudaSuccess ||
                cudaEventCreateWithFlags(&hp.join[i], cudaEventDisableTiming) != cudaSuccess)
                return DGAL_ERR_CUDA;
        }
        if (cudaEventCreateWithFlags(&hp.fork, cudaEventDisableTiming) != cudaSuccess) return DGAL_ERR_CUDA;
        hp.init = true;
    }
    const cudaStream_t cs = as_cuda(stream);
    cudaError_t e = cudaEventRecord(hp.fork, cs);
    for (int i = 0; i < kHostStreams && e == cudaSuccess; ++i) e = cudaStreamWaitEvent(hp.s[i], hp.fork, 0);
    dgal_status st = from_cuda(e);
    const cudaMemcpyKind H2D = cudaMemcpyHostToDevice, D2H = cudaMemcpyDeviceToHost;
    int64_t c = 0;
    for (int64_t off = 0; off < n && st == DGAL_OK; off += chunk, ++c) {
        const int64_t m = (n - off < chunk) ? n - off : chunk;
        const int si = (int)(c % kHostStreams);
        const cudaStream_t s = hp.s[si];
        const HostSlot h = host_slot(workspace, K, chunk, si);
        const size_t pb = sizeof(float) * (size_t)m * K, o = (size_t)off * K;
        // (a stage reuses its slot after the stage kHostStreams chunks earlier: same stream)
        e = cudaMemcpyAsync(h.x1, x1 + o, pb, H2D, s);
        if (e == cudaSuccess) e = cudaMemcpyAsync(h.y1, y1 + o, pb, H2D, s);
        if (e == cudaSuccess) e = cudaMemcpyAsync(h.x2, x2 + o, pb, H2D, s);
        if (e == cudaSuccess) e = cudaMemcpyAsync(h.y2, y2 + o, pb, H2D, s);
        if (e == cudaSuccess) e = cudaMemcpyAsync(h.g, grad_iou + off, sizeof(float) * (size_t)m, H2D, s);
        st = from_cuda(e);
        if (st == DGAL_OK)
            st = from_cuda(dgal::launch_paired_fwd(K, m, h.x1, h.y1, h.x2, h.y2, h.iou, h.nx, h.xf, s));
        if (st == DGAL_OK)
            st = from_cuda(dgal::launch_paired_bwd(K, m, h.x1, h.y1, h.x2, h.y2, h.g, h.nx, h.xf, h.gx1, h.gy1,
                                                   h.gx2, h.gy2, s));
        if (st == DGAL_OK) {
            e = cudaMemcpyAsync(iou + off, h.iou, sizeof(float) * (size_t)m, D2H, s);
            if (e == cudaSuccess) e = cudaMemcpyAsync(gx1 + o, h.gx1, pb, D2H, s);
            if (e == cudaSuccess) e = cudaMemcpyAsync(gy1 + o, h.gy1, pb, D2H, s);
            if (e == cudaSuccess) e = cudaMemcpyAsync(gx2 + o, h.gx2, pb, D2H, s);
            if (e == cudaSuccess) e = cudaMemcpyAsync(gy2 + o, h.gy2, pb, D2H, s);
            st = from_cuda(e);
        }
    }
    // join (also after an error: the caller's stream never runs ahead of enqueued work)
    for (int i = 0; i < kHostStreams; ++i) {
        const cudaError_t e1 = cudaEventRecord(hp.join[i], hp.s[i]);
        const cudaError_t e2 = (e1 == cudaSuccess) ? cudaStreamWaitEvent(cs, hp.join[i], 0) : e1;
        if (st == DGAL_OK && e2 != cudaSuccess) st = DGAL_ERR_CUDA;
    }
    return st;
}

size_t dgal_fused_workspace_bytes(int64_t n)
{
    return dgal::refine_workspace_bytes(n < 0 ? 0 : n);
}

dgal_status dgal_iou_paired_fused(int K, int64_t n, const float *x1, const float *y1, const float *x2,
                                  const float *y2, const float *grad_iou, float grad_scale, float *iou,
                                  float *gx1, float *gy1, float *gx2, float *gy2, void *workspace,
                                  size_t workspace_bytes, dgal_stream stream)
{
    if (K != 4 && K != 8) return DGAL_ERR_UNSUPPORTED_K;
    if (n < 0) return DGAL_ERR_INVALID_ARG;
    if (n == 0) return DGAL_OK;
    if (!x1 || !y1 || !x2 || !y2 || !gx1 || !gy1 || !gx2 || !gy2) return DGAL_ERR_INVALID_ARG;
    if (!workspace || workspace_bytes < dgal::refine_workspace_bytes(n)) return DGAL_ERR_INVALID_ARG;
    if (n > dgal::kMaxFusedPairs) return DGAL_ERR_INVALID_ARG;
    if (!aligned(x1, 16) || !aligned(y1, 16) || !aligned(x2, 16) || !aligned(y2, 16) ||
        !aligned(gx1, 16) || !aligned(gy1, 16) || !aligned(gx2, 16) || !aligned(gy2, 16) ||
        (grad_iou && !aligned(grad_iou, 4)) || (iou && !aligned(iou, 4)) || !aligned(workspace, 16))
        return DGAL_ERR_MISALIGNED;
    return from_cuda(dgal::launch_paired_fused(K, n, x1, y1, x2, y2, grad_iou, grad_scale, iou, gx1, gy1, gx2,
                                               gy2, workspace, as_cuda(stream)));
}

namespace {
inline dgal_status box_check(int dims, int layout, int64_t n, const float *b1, const float *b2)
{
    if (dims != 2 && dims != 3) return DGAL_ERR_INVALID_ARG;
    if (layout != DGAL_BOX_PLANES && layout != DGAL_BOX_ROWS) return DGAL_ERR_INVALID_ARG;
    if (n < 0) return DGAL_ERR_INVALID_ARG;
    if (n > 0 && (!b1 || !b2)) return DGAL_ERR_INVALID_ARG;
    if (n > 0 && (!aligned(b1, 4) || !aligned(b2, 4))) return DGAL_ERR_MISALIGNED;
    return DGAL_OK;
}
}  // namespace

dgal_status dgal_box_iou_paired_fwd(int dims, int layout, int64_t n, const float *b1, const float *b2, float *iou,
                                    uint8_t *nx, uint8_t *xflags, dgal_stream stream)
{
    const dgal_status c = box_check(dims, layout, n, b1, b2);
    if (c != DGAL_OK || n == 0) return c;
    if (!iou || !nx || !xflags) return DGAL_ERR_INVALID_ARG;
    if (!aligned(iou, 4) || !aligned(xflags, 8)) return DGAL_ERR_MISALIGNED;
    return from_cuda(dgal::launch_box_fwd(dims, layout, n, b1, b2, iou, nx, xflags, as_cuda(stream)));
}

dgal_status dgal_box_iou_paired_bwd(int dims, int layout, int64_t n, const float *b1, const float *b2,
                                    const float *grad_iou, const uint8_t *nx, const uint8_t *xflags, float *grad_b1,
                                    float *grad_b2, dgal_stream stream)
{
    const dgal_status c = box_check(dims, layout, n, b1, b2);
    if (c != DGAL_OK || n == 0) return c;
    if (!grad_iou || !nx || !xflags || !grad_b1 || !grad_b2) return DGAL_ERR_INVALID_ARG;
    if (!aligned(grad_iou, 4) || !aligned(xflags, 8) || !aligned(grad_b1, 4) || !aligned(grad_b2, 4))
        return DGAL_ERR_MISALIGNED;
    return from_cuda(dgal::launch_box_bwd(dims, layout, n, b1, b2, grad_iou, nx, xflags, grad_b1, grad_b2,
                                          as_cuda(stream)));
}

dgal_status dgal_box_iou_paired_fused(int dims, int layout, int64_t n, const float *b1, const float *b2,
                                      const float *grad_iou, float grad_scale, float *iou, float *grad_b1,
                                      float *grad_b2, void *workspace, size_t workspace_bytes, dgal_stream stream)
{
    const dgal_status c = box_check(dims, layout, n, b1, b2);
    if (c != DGAL_OK || n == 0) return c;
    if (!grad_b1 || !grad_b2) return DGAL_ERR_INVALID_ARG;
    if (!workspace || workspace_bytes < dgal::refine_workspace_bytes(n)) return DGAL_ERR_INVALID_ARG;
    if (n > dgal::kMaxFusedPairs) return DGAL_ERR_INVALID_ARG;
    if ((grad_iou && !aligned(grad_iou, 4)) || (iou && !aligned(iou, 4)) || !aligned(grad_b1, 4) ||
        !aligned(grad_b2, 4) || !aligned(workspace, 16))
        return DGAL_ERR_MISALIGNED;
    return from_cuda(dgal::launch_box_fused(dims, layout, n, b1, b2, grad_iou, grad_scale, iou, grad_b1, grad_b2,
                                            workspace, as_cuda(stream)));
}

dgal_status dgal_iou_pairwise(int K, int64_t n_rows, const float *row_x, const float *row_y, int64_t m,
                              const float *col_x, const float *col_y, int64_t row_offset, float *iou,
                              float nms_thresh, uint64_t *mask, int64_t mask_words, int32_t *nbr_count,
                              int32_t *nbr_idx, int32_t nbr_cap, void *workspace, size_t workspace_bytes,
                              dgal_stream stream)
{
    if (K != 4 && K != 8) return DGAL_ERR_UNSUPPORTED_K;
    if (n_rows < 0 || m < 0 || row_offset < 0) return DGAL_ERR_INVALID_ARG;
    if (n_rows == 0) return DGAL_OK;
    if (m == 0) {   // no columns: every row has zero suppressors (nbr_count is an output)
        if ((nbr_count == nullptr) != (nbr_idx == nullptr)) return DGAL_ERR_INVALID_ARG;
        if (!nbr_count) return DGAL_OK;
        return from_cuda(cudaMemsetAsync(nbr_count, 0, sizeof(int32_t) * (size_t)n_rows, as_cuda(stream)));
    }
    if (!row_x || !row_y || !col_x || !col_y) return DGAL_ERR_INVALID_ARG;
    if (!iou && !mask) return DGAL_ERR_INVALID_ARG;                 // nothing to compute
    if (m > (int64_t)65535 * dgal::kPwTileCols) return DGAL_ERR_INVALID_ARG;
    if (mask) {
        if (!(nms_thresh >= 0.f)) return DGAL_ERR_INVALID_ARG;    // also rejects NaN
        if (mask_words < (m + 63) / 64) return DGAL_ERR_INVALID_ARG;
        if (!aligned(mask, 8)) return DGAL_ERR_MISALIGNED;
    }
    if ((nbr_count == nullptr) != (nbr_idx == nullptr)) return DGAL_ERR_INVALID_ARG;
    if (nbr_count && (!mask || nbr_cap < 0)) return DGAL_ERR_INVALID_ARG;
    if (!aligned(row_x, 16) || !aligned(row_y, 16) || !aligned(col_x, 16) || !aligned(col_y, 16) ||
        (iou && !aligned(iou, 4)))
        return DGAL_ERR_MISALIGNED;
    if (workspace && workspace_bytes >= dgal::pairwise_workspace_bytes(m)) {
        if (!aligned(workspace, 256)) return DGAL_ERR_MISALIGNED;
        if (m > (int64_t)INT32_MAX) return DGAL_ERR_INVALID_ARG;
        return from_cuda(dgal::launch_pairwise_indexed(K, n_rows, row_x, row_y, m, col_x, col_y, row_offset, iou,
                                                       nms_thresh, mask, mask_words, nbr_count, nbr_idx,
                                                       nbr_cap, workspace, as_cuda(stream)));
    }
    if (workspace) return DGAL_ERR_INVALID_ARG;  // too small
    return from_cuda(dgal::launch_pairwise(K, n_rows, row_x, row_y, m, col_x, col_y, row_offset, iou,
                                           nms_thresh, mask, mask_words, nbr_count, nbr_idx, nbr_cap,
                                           as_cuda(stream)));
}

size_t dgal_pairwise_workspace_bytes(int64_t m)
{
    return dgal::pairwise_workspace_bytes(m < 0 ? 0 : m);
}

dgal_status dgal_nms_round(int64_t n_total, int64_t n_rows, int64_t row_offset, const uint64_t *mask,
                           int64_t mask_words, const int32_t *nbr_count, const int32_t *nbr_idx,
                           int32_t nbr_cap, uint8_t *status, int32_t *undecided, int32_t *scratch,
                           dgal_stream stream)
{
    if (n_total < 0 || n_rows < 0 || row_offset < 0 || row_offset + n_rows > n_total)
        return DGAL_ERR_INVALID_ARG;
    if (n_rows == 0) return DGAL_OK;
    if (!mask || !status || !undecided || mask_words < (n_total + 63) / 64) return DGAL_ERR_INVALID_ARG;
    if ((nbr_count == nullptr) != (nbr_idx == nullptr) || nbr_cap < 0) return DGAL_ERR_INVALID_ARG;
    if (!aligned(mask, 8) || !aligned(undecided, 4) || (scratch && !aligned(scratch, 4)))
        return DGAL_ERR_MISALIGNED;
    return from_cuda(dgal::launch_nms_round(n_total, n_rows, row_offset, mask, mask_words, nbr_count,
                                            nbr_idx, nbr_cap, status, undecided, scratch, as_cuda(stream)));
}

dgal_status dgal_nms_keep(int64_t n, const uint64_t *mask, int64_t mask_words, const int32_t *nbr_count,
                          const int32_t *nbr_idx, int32_t nbr_cap, uint8_t *status, uint8_t *keep,
                          int32_t *scratch, dgal_stream stream)
{
    if (n < 0) return DGAL_ERR_INVALID_ARG;
    if (n == 0) return DGAL_OK;
    if (!mask || !status || !keep || mask_words < (n + 63) / 64) return DGAL_ERR_INVALID_ARG;
    if ((nbr_count == nullptr) != (nbr_idx == nullptr) || nbr_cap < 0) return DGAL_ERR_INVALID_ARG;
    if (!aligned(mask, 8) || (scratch && !aligned(scratch, 4))) return DGAL_ERR_MISALIGNED;
    return from_cuda(dgal::launch_nms_keep(n, mask, mask_words, nbr_count, nbr_idx, nbr_cap, status, keep,
                                           scratch, as_cuda(stream)));
}

const char *dgal_status_string(dgal_status s)
{
    switch (s) {
    case DGAL_OK: return "DGAL_OK";
    case DGAL_ERR_INVALID_ARG: return "DGAL_ERR_INVALID_ARG";
    case DGAL_ERR_UNSUPPORTED_K: return "DGAL_ERR_UNSUPPORTED_K";
    case DGAL_ERR_MISALIGNED: return "DGAL_ERR_MISALIGNED";
    case DGAL_ERR_CUDA: return "DGAL_ERR_CUDA";
    }
    return "DGAL_ERR_UNKNOWN";
}

const char *dgal_build_info(void)
{
#define DGAL_STR2(x) #x
#define DGAL_STR(x) DGAL_STR2(x)
    return "libdgal " DGAL_VERSION " sm_100a nvcc " DGAL_STR(__CUDACC_VER_MAJOR__) "." DGAL_STR(
        __CUDACC_VER_MINOR__) "." DGAL_STR(__CUDACC_VER_BUILD__);
}

}  // extern "C"
