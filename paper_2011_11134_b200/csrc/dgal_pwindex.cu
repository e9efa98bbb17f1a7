// dgal_pwindex.cu — indexed pairwise path: for large, sparse
// N x M problems the matrix is (1) zero-filled by a streaming kernel at HBM write
// speed and (2) only the pairs whose bounding circles intersect are evaluated,
// found through a uniform grid over the column circles (counting sort built on
// the device in a caller-provided workspace).  Exactness: disjoint bounding
// circles => disjoint polygons => IoU 0, which the zero-fill already wrote.
#include <mutex>

#include "dgal_core.cuh"
#include "dgal_internal.h"

namespace dgal {

namespace {

constexpr unsigned kFull = 0xFFFFFFFFu;
constexpr int kGridMaxCells = 1 << 16;  // <= 256 x 256 cells
constexpr int kThreads = 256;
#ifndef DGAL_PW_U
#define DGAL_PW_U 4      // circle loads in flight per lane in the flattened sweep (A/B cfg5: 1 / 2 / 4: 6.07 / 6.00 / 5.95 ms)
#endif
constexpr int kU = DGAL_PW_U;

#ifndef DGAL_PW_CELL
#define DGAL_PW_CELL 0.5f   // grid cell size in units of the largest column radius (A/B cfg5: 2 -> 0.5: -0.05 ms)
#endif

struct GridHeader {
    float xmin, ymin, xmax, ymax;  // extent of the column circle centres
    float rmax;                    // largest column radius
    float cell;                    // cell size (>= 2 rmax)
    int nx, ny;                    // grid dims
};

// Per-call state of the candidate pass (workspace): warps claim rows in order.
struct PwState {
    unsigned long long next_row;   // next unclaimed row
    unsigned long long pad[3];
};

struct Workspace {
    GridHeader *hdr;
    PwState *state;
    float4 *circ;       // [m] column circles
    int32_t *cell_of;   // [m]
    int32_t *sorted;    // [m] column ids grouped by cell (unused by the search; kept for tests)
    float4 *csorted;    // [m] circles grouped by cell, .w = column id (int bits)
    int32_t *start;     // [kGridMaxCells + 1] exclusive prefix of the counts
    int32_t *fill;      // [kGridMaxCells]
};

__host__ __device__ inline size_t align256(size_t b) { return (b + 255) & ~(size_t)255; }

__host__ __device__ inline Workspace carve(void *ws, int64_t m)
{
    char *p = static_cast<char *>(ws);
    Workspace w;
    w.hdr = reinterpret_cast<GridHeader *>(p);
    p += align256(sizeof(GridHeader));
    w.state = reinterpret_cast<PwState *>(p);
    p += align256(sizeof(PwState));
    w.circ = reinterpret_cast<float4 *>(p);
    p += align256(sizeof(float4) * (size_t)m);
    w.cell_of = reinterpret_cast<int32_t *>(p);
    p += align256(sizeof(int32_t) * (size_t)m);
    w.sorted = reinterpret_cast<int32_t *>(p);
    p += align256(sizeof(int32_t) * (size_t)m);
    w.csorted = reinterpret_cast<float4 *>(p);
    p += align256(sizeof(float4) * (size_t)m);
    w.start = reinterpret_cast<int32_t *>(p);
    p += align256(sizeof(int32_t) * (kGridMaxCells + 1));
    w.fill = reinterpret_cast<int32_t *>(p);
    return w;
}

__device__ __forceinline__ void atomic_min_f(float *a, float v)
{
    int *ai = reinterpret_cast<int *>(a);
    int old = *ai;
    while (v < __int_as_float(old)) {
        const int prev = atomicCAS(ai, old, __float_as_int(v));
        if (prev == old) break;
        old = prev;
    }
}
__device__ __forceinline__ void atomic_max_f(float *a, float v)
{
    int *ai = reinterpret_cast<int *>(a);
    int old = *ai;
    while (v > __int_as_float(old)) {
        const int prev = atomicCAS(ai, old, __float_as_int(v));
        if (prev == old) break;
        old = prev;
    }
}

template <int K>
__device__ __forceinline__ float4 circle_of(const float *__restrict__ X, const float *__restrict__ Y, int64_t c)
{
    float x[K], y[K];
#pragma unroll
    for (int k = 0; k < K; ++k) { x[k] = __ldg(X + c * K + k); y[k] = __ldg(Y + c * K + k); }
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
    const float r = sqrtf(r2) * 1.0001f + 2e-6f * (fabsf(cx) + fabsf(cy)) + 1e-30f;
    return make_float4(cx, cy, r, 0.f);
}

__global__ void pw_init(Workspace w)
{
    w.state->next_row = 0;
    GridHeader &h = *w.hdr;
    h.xmin = h.ymin = __int_as_float(0x7f800000);
    h.xmax = h.ymax = -__int_as_float(0x7f800000);
    h.rmax = 0.f;
}

template <int K>
__global__ void __launch_bounds__(kThreads) pw_circles(int64_t m, const float *__restrict__ cx,
                                                       const float *__restrict__ cy, Workspace w)
{
    __shared__ float red[5][kThreads / 32];
    const int64_t c = (int64_t)blockIdx.x * kThreads + threadIdx.x;
    float x0 = __int_as_float(0x7f800000), y0 = x0, x1 = -x0, y1 = -x0, r = 0.f;
    if (c < m) {
        const float4 q = circle_of<K>(cx, cy, c);
        w.circ[c] = q;
        x0 = x1 = q.x;
        y0 = y1 = q.y;
        r = q.z;
    }
#pragma unroll
    for (int d = 16; d; d >>= 1) {
        x0 = fminf(x0, __shfl_xor_sync(kFull, x0, d));
        y0 = fminf(y0, __shfl_xor_sync(kFull, y0, d));
        x1 = fmaxf(x1, __shfl_xor_sync(kFull, x1, d));
        y1 = fmaxf(y1, __shfl_xor_sync(kFull, y1, d));
        r = fmaxf(r, __shfl_xor_sync(kFull, r, d));
    }
    const int wp = threadIdx.x >> 5;
    if ((threadIdx.x & 31) == 0) {
        red[0][wp] = x0; red[1][wp] = y0; red[2][wp] = x1; red[3][wp] = y1; red[4][wp] = r;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int i = 1; i < kThreads / 32; ++i) {
            x0 = fminf(x0, red[0][i]); y0 = fminf(y0, red[1][i]);
            x1 = fmaxf(x1, red[2][i]); y1 = fmaxf(y1, red[3][i]); r = fmaxf(r, red[4][i]);
        }
        GridHeader &h = *w.hdr;
        atomic_min_f(&h.xmin, x0);
        atomic_min_f(&h.ymin, y0);
        atomic_max_f(&h.xmax, x1);
        atomic_max_f(&h.ymax, y1);
        atomic_max_f(&h.rmax, r);
    }
}

// grid geometry from the header: cells of size DGAL_PW_CELL x rmax, at most
// 256 x 256 cells.  Any size is exact: a row scans every cell within its reach
// (its radius + rmax) of its centre; smaller cells scan fewer circles per row
// in more (flattened) ranges.
__device__ __forceinline__ void grid_dims(const GridHeader &h, float &cell, int &nx, int &ny)
{
    const float ex = fmaxf(h.xmax - h.xmin, 0.f), ey = fmaxf(h.ymax - h.ymin, 0.f);
    cell = fmaxf(fmaxf(DGAL_PW_CELL * h.rmax, fmaxf(ex, ey) * (1.f / 255.f)), 1e-20f);
    nx = min(256, (int)(ex / cell) + 1);
    ny = min(256, (int)(ey / cell) + 1);
}

__device__ __forceinline__ int cell_coord(float v, float lo, float cell, int n)
{
    return min(n - 1, max(0, (int)floorf((v - lo) / cell)));
}

__global__ void __launch_bounds__(kThreads) pw_count(int64_t m, Workspace w)
{
    const int64_t c = (int64_t)blockIdx.x * kThreads + threadIdx.x;
    if (c >= m) return;
    float cell;
    int nx, ny;
    const GridHeader h = *w.hdr;
    grid_dims(h, cell, nx, ny);
    const float4 q = w.circ[c];
    const int id = cell_coord(q.y, h.ymin, cell, ny) * nx + cell_coord(q.x, h.xmin, cell, nx);
    w.cell_of[c] = id;
    atomicAdd(w.start + id + 1, 1);
    if (c == 0) {
        w.hdr->cell = cell;
        w.hdr->nx = nx;
        w.hdr->ny = ny;
    }
}

// exclusive scan of the nx*ny (<= 65536) cell counts, one CTA: start[1 + j]
// becomes the number of columns in cells < j (the first slot of cell j)
__global__ void __launch_bounds__(1024) pw_scan(Workspace w)
{
    __shared__ int32_t part[1024];
    const int ncells = w.hdr->nx * w.hdr->ny;
    const int per = (ncells + 1023) / 1024;
    const int t = threadIdx.x;
    const int lo = min(ncells, t * per), hi = min(ncells, lo + per);
    int32_t *v = w.start + 1;
    int32_t s = 0;
    for (int i = lo; i < hi; ++i) s += v[i];
    part[t] = s;
    __syncthreads();
    for (int d = 1; d < 1024; d <<= 1) {
        const int32_t add = (t >= d) ? part[t - d] : 0;
        __syncthreads();
        part[t] += add;
        __syncthreads();
    }
    int32_t run = part[t] - s;
    for (int i = lo; i < hi; ++i) {
        const int32_t c = v[i];
        v[i] = run;
        run += c;
    }
    if (t == 0) w.start[0] = 0;
}

__global__ void __launch_bounds__(kThreads) pw_scatter(int64_t m, Workspace w)
{
    const int64_t c = (int64_t)blockIdx.x * kThreads + threadIdx.x;
    if (c >= m) return;
    const int id = w.cell_of[c];
    const int pos = w.start[id + 1] + atomicAdd(w.fill + id, 1);
    DGAL_ASSERT(id >= 0 && id < kGridMaxCells && pos >= 0 && pos < m);
    w.sorted[pos] = (int32_t)c;
    const float4 q = w.circ[c];
    w.csorted[pos] = make_float4(q.x, q.y, q.z, __int_as_float((int)c));
}

// streaming zero fill of a byte range: every block clears one contiguous
// 16 KB chunk (256 threads x 4 x 16 B), blocks in address order — measured at
// 7.6 TB/s on B200 for 40 GB (a grid-stride loop reaches 6.8, cudaMemset 7.4;
// tools/probes/zero_bw.cu)
constexpr int kZeroU = 4;
__global__ void __launch_bounds__(kThreads) pw_zero(char *p, size_t bytes)
{
    const uintptr_t a = reinterpret_cast<uintptr_t>(p);
    size_t head = (16 - (a & 15)) & 15;
    head = head < bytes ? head : bytes;
    const size_t nvec = (bytes - head) / 16;
    const size_t tail = bytes - head - nvec * 16;
    const size_t base = (size_t)blockIdx.x * kThreads * kZeroU + threadIdx.x;
    int4 *v = reinterpret_cast<int4 *>(p + head);
#pragma unroll
    for (int u = 0; u < kZeroU; ++u) {
        const size_t i = base + (size_t)u * kThreads;
        if (i < nvec) __stcs(v + i, make_int4(0, 0, 0, 0));
    }
    if (blockIdx.x == 0) {
        if (threadIdx.x < head) p[threadIdx.x] = 0;
        if (threadIdx.x < tail) p[head + nvec * 16 + threadIdx.x] = 0;
    }
}

inline void launch_zero(void *p, size_t bytes, cudaStream_t st)
{
    const size_t chunk = (size_t)kThreads * kZeroU * 16;
    const size_t grid = (bytes + chunk - 1) / chunk;
    if (grid) pw_zero<<<(unsigned)grid, kThreads, 0, st>>>(static_cast<char *>(p), bytes);
}

struct PwArgs {
    int64_t n_rows;
    const float *rx, *ry;
    int64_t m;
    const float *cx, *cy;
    int64_t row_offset;
    float *iou;
    float thr;
    uint64_t *mask;
    int64_t mask_words;
    int32_t *nbr_count, *nbr_idx;
    int32_t cap;
};

// Evaluate candidate pair (row rr, column c): IoU, mask bit, suppressor list.
template <int K>
__device__ __forceinline__ void pw_eval(const PwArgs &a, int64_t rr, int32_t c)
{
    Poly<K> P, Q;
    // 16-byte loads (planes are 16-byte aligned, include/dgal.h): K/4 per plane;
    // (cached loads: a row's polygon serves all its candidates, a column's its neighbours)
    DGAL_ASSERT(rr >= 0 && rr < a.n_rows && c >= 0 && c < a.m);
#pragma unroll
    for (int q = 0; q < K / 4; ++q) {
        const float4 u0 = __ldg(reinterpret_cast<const float4 *>(a.rx + rr * K) + q);
        const float4 u1 = __ldg(reinterpret_cast<const float4 *>(a.ry + rr * K) + q);
        const float4 u2 = __ldg(reinterpret_cast<const float4 *>(a.cx + (int64_t)c * K) + q);
        const float4 u3 = __ldg(reinterpret_cast<const float4 *>(a.cy + (int64_t)c * K) + q);
        P.x[4 * q] = u0.x; P.x[4 * q + 1] = u0.y; P.x[4 * q + 2] = u0.z; P.x[4 * q + 3] = u0.w;
        P.y[4 * q] = u1.x; P.y[4 * q + 1] = u1.y; P.y[4 * q + 2] = u1.z; P.y[4 * q + 3] = u1.w;
        Q.x[4 * q] = u2.x; Q.x[4 * q + 1] = u2.y; Q.x[4 * q + 2] = u2.z; Q.x[4 * q + 3] = u2.w;
        Q.y[4 * q] = u3.x; Q.y[4 * q + 1] = u3.y; Q.y[4 * q + 2] = u3.z; Q.y[4 * q + 3] = u3.w;
    }
    const float ox = P.x[0], oy = P.y[0];
#pragma unroll
    for (int k = 0; k < K; ++k) {
        P.x[k] = __fsub_rn(P.x[k], ox); P.y[k] = __fsub_rn(P.y[k], oy);
        Q.x[k] = __fsub_rn(Q.x[k], ox); Q.y[k] = __fsub_rn(Q.y[k], oy);
    }
    P.x[0] = 0.f;   // exact for finite input; lets the compiler fold it
    P.y[0] = 0.f;
    const FwdOut<K, false> fo = iou_fwd<K, false>(P, Q);
    float v = fo.iou;
    // thin pair (R^2 > kThinRatio A_u): the area of the recorded intersection in double
    if (DGAL_THIN && pair_is_thin(pair_extent2<K>(P, Q), (fo.A1x2 + fo.A2x2) - fo.Aix2))
        v = pair_iou_exact<K>(a.rx + rr * K, a.ry + rr * K, a.cx + (int64_t)c * K, a.cy + (int64_t)c * K);
    if (a.iou && v != 0.f) a.iou[rr * a.m + c] = v;
    const int64_t grow = a.row_offset + rr;
    if (v > a.thr && c != grow) {
        if (a.mask) atomicOr(reinterpret_cast<unsigned long long *>(a.mask + rr * a.mask_words + (c >> 6)),
                             1ull << (c & 63));
        if (a.nbr_count && c < grow) {
            const int slot = atomicAdd(a.nbr_count + rr, 1);
            if (slot < a.cap) a.nbr_idx[rr * a.cap + slot] = c;
        }
    }
}

// The next unclaimed row (warp-uniform); its suppressor count starts at 0 (no
// separate memset of nbr_count).
__device__ __forceinline__ int64_t claim_row(const PwArgs &a, PwState *s, int lane)
{
    unsigned long long r = 0;
    if (lane == 0) {
        r = atomicAdd(&s->next_row, 1ull);
        if (a.nbr_count && r < (unsigned long long)a.n_rows) a.nbr_count[r] = 0;
    }
    __syncwarp();
    return (int64_t)__shfl_sync(kFull, r, 0);
}

// Sweep of row r (one warp).  The cells of one grid row are consecutive in the
// cell-sorted circle array, so the row's neighbourhood is one contiguous range
// per grid row gy (cells cx0..cx1); up to 32 ranges at a time, lane g holding
// range g, swept as ONE index space (no padding per range) with kU coalesced
// 16 B loads in flight per lane.  push(hit, c, bal) takes each ballot of
// circle-overlapping columns, drain() runs after each kU of them.
template <int K, class Push, class Drain>
__device__ __forceinline__ void sweep_row(const PwArgs &a, const Workspace &w, const GridHeader &h, int ncells,
                                          int64_t r, int lane, Push &&push, Drain &&drain)
{
    const float4 rc = circle_of<K>(a.rx, a.ry, r);               // warp-uniform
    const float reach = rc.z + h.rmax;
    const int cx0 = cell_coord(rc.x - reach, h.xmin, h.cell, h.nx);
    const int cx1 = cell_coord(rc.x + reach, h.xmin, h.cell, h.nx);
    const int cy0 = cell_coord(rc.y - reach, h.ymin, h.cell, h.ny);
    const int cy1 = cell_coord(rc.y + reach, h.ymin, h.cell, h.ny);
    for (int gy0 = cy0; gy0 <= cy1; gy0 += 32) {
        const int G = min(32, cy1 - gy0 + 1);
        int rlo = 0, rlen = 0;
        if (lane < G) {
            const int gy = gy0 + lane;
            const int id0 = gy * h.nx + cx0, id1 = gy * h.nx + cx1;
            rlo = w.start[1 + id0];
            rlen = ((id1 + 1 < ncells) ? w.start[2 + id1] : (int)a.m) - rlo;
        }
        int incl = rlen;   // inclusive prefix of the range lengths
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const int v = __shfl_up_sync(kFull, incl, d);
            if (lane >= d) incl += v;
        }
        const int total = __shfl_sync(kFull, incl, 31);
        const int delta = rlo - (incl - rlen);   // pos = k + delta of the range holding k
        for (int k0 = 0; k0 < total; k0 += 32 * kU) {           // warp-uniform
            float4 q[kU];
#pragma unroll
            for (int u = 0; u < kU; ++u) {
                const int k = k0 + u * 32 + lane;
                int dl = __shfl_sync(kFull, delta, 0);     // (all lanes: shuffles)
                for (int g = 1; g < G; ++g) {
                    const int e = __shfl_sync(kFull, incl, g - 1);
                    const int dg = __shfl_sync(kFull, delta, g);
                    dl = (k >= e) ? dg : dl;
                }
                q[u] = make_float4(0.f, 0.f, -1.f, 0.f);
                if (k < total) {
                    DGAL_ASSERT(k + dl >= 0 && k + dl < a.m);
                    q[u] = w.csorted[k + dl];
                }
            }
#pragma unroll
            for (int u = 0; u < kU; ++u) {
                const float dx = q[u].x - rc.x, dy = q[u].y - rc.y, rs = q[u].z + rc.z;
                const bool hit = q[u].z >= 0.f && dx * dx + dy * dy < rs * rs;
                const int32_t c = __float_as_int(q[u].w);
                push(hit, c, __ballot_sync(kFull, hit));
            }
            __syncwarp();
            drain();
        }
    }
}

// Candidate pass: one WARP per claimed row (persistent grid, rows claimed in
// order); the warp queues the row's circle-overlapping columns and evaluates the
// queue 32 entries at a time.  (A split into a low-register sweep writing a pair
// list and a full-occupancy evaluator was measured slower: DESIGN.md §4.3.)
template <int K>
__global__ void __launch_bounds__(kThreads, K == 4 ? 2 : 1)   // K = 8: the whole register file (no spill)
pw_candidates(PwArgs a, Workspace w)
{
    constexpr int kQ = 32 * (kU + 1);
    __shared__ int64_t qrow[kThreads / 32][kQ];
    __shared__ int32_t qcol[kThreads / 32][kQ];
    const int lane = threadIdx.x & 31, wp = threadIdx.x >> 5;
    const GridHeader h = *w.hdr;
    const int ncells = h.nx * h.ny;
    int qn = 0;
    for (;;) {
        const int64_t r = claim_row(a, w.state, lane);
        if (r >= a.n_rows) break;
        sweep_row<K>(a, w, h, ncells, r, lane,
                     [&](bool hit, int32_t c, unsigned bal) {
                         if (hit) {
                             const int at = qn + __popc(bal & ((1u << lane) - 1u));
                             DGAL_ASSERT(at < kQ && c >= 0 && c < a.m);
                             qrow[wp][at] = r;
                             qcol[wp][at] = c;
                         }
                         qn += __popc(bal);
                     },
                     [&]() {
                         while (qn >= 32) {   // one call site: the evaluator's code once in the loop
                             pw_eval<K>(a, qrow[wp][qn - 32 + lane], qcol[wp][qn - 32 + lane]);
                             qn -= 32;
                             __syncwarp();
                         }
                     });
    }
    __syncwarp();
    if (lane < qn) pw_eval<K>(a, qrow[wp][lane], qcol[wp][lane]);
}

}  // namespace

namespace {
// The grid build (two memsets and five small kernels, ~0.05 ms of launches and latency)
// runs on a per-device, high-priority side stream, overlapping the output zero fill of the
// caller's stream: fork / join events, so it stays ordered with the caller's stream and
// capturable into a CUDA graph; the lock keeps one call's fork / join pairs together.
struct SideStream {
    std::mutex mu;
    bool init = false;
    cudaStream_t s = nullptr;
    cudaEvent_t fork = nullptr, join = nullptr;
};
SideStream g_side[kMaxDevices];
}  // namespace

size_t pairwise_workspace_bytes(int64_t m)
{
    return align256(sizeof(GridHeader)) + align256(sizeof(PwState)) + 2 * align256(sizeof(float4) * (size_t)m) +
           2 * align256(sizeof(int32_t) * (size_t)m) + align256(sizeof(int32_t) * (kGridMaxCells + 1)) +
           align256(sizeof(int32_t) * kGridMaxCells);
}

cudaError_t launch_pairwise_indexed(int K, int64_t n_rows, const float *rx, const float *ry, int64_t m,
                                    const float *cx, const float *cy, int64_t row_offset, float *iou,
                                    float thr, uint64_t *mask, int64_t mask_words, int32_t *nbr_count,
                                    int32_t *nbr_idx, int32_t cap, void *workspace, cudaStream_t st)
{
    const Workspace w = carve(workspace, m);
    const PwArgs a{n_rows, rx, ry, m, cx, cy, row_offset, iou, thr, mask, mask_words, nbr_count, nbr_idx, cap};
    cudaError_t e;
    int dev = 0, sms = 0;
    if ((e = cudaGetDevice(&dev))) return e;
    if (dev < 0 || dev >= kMaxDevices) return cudaErrorInvalidDevice;
    SideStream &ss = g_side[dev];
    std::lock_guard<std::mutex> lock(ss.mu);
    if (!ss.init) {
        int lo = 0, hi = 0;
        if ((e = cudaDeviceGetStreamPriorityRange(&lo, &hi))) return e;
        if ((e = cudaStreamCreateWithPriority(&ss.s, cudaStreamNonBlocking, hi))) return e;
        if ((e = cudaEventCreateWithFlags(&ss.fork, cudaEventDisableTiming))) return e;
        if ((e = cudaEventCreateWithFlags(&ss.join, cudaEventDisableTiming))) return e;
        ss.init = true;
    }
    // (2, side stream) grid index of the column circles, after everything before the call
    if ((e = cudaEventRecord(ss.fork, st))) return e;
    if ((e = cudaStreamWaitEvent(ss.s, ss.fork, 0))) return e;
    const cudaStream_t gs = ss.s;
    if ((e = cudaMemsetAsync(w.start, 0, sizeof(int32_t) * (kGridMaxCells + 1), gs))) return e;
    if ((e = cudaMemsetAsync(w.fill, 0, sizeof(int32_t) * kGridMaxCells, gs))) return e;
    pw_init<<<1, 1, 0, gs>>>(w);
    const unsigned mg = (unsigned)((m + kThreads - 1) / kThreads);
    if (K == 4) pw_circles<4><<<mg, kThreads, 0, gs>>>(m, cx, cy, w);
    else pw_circles<8><<<mg, kThreads, 0, gs>>>(m, cx, cy, w);
    pw_count<<<mg, kThreads, 0, gs>>>(m, w);
    pw_scan<<<1, 1024, 0, gs>>>(w);
    pw_scatter<<<mg, kThreads, 0, gs>>>(m, w);
    if ((e = cudaGetLastError())) return e;
    if ((e = cudaEventRecord(ss.join, gs))) return e;
    // (1) meanwhile, zero-fill the outputs at streaming-write speed (nbr_count: zeroed as
    // each row is claimed, claim_row)
    if (iou) launch_zero(iou, sizeof(float) * (size_t)n_rows * m, st);
    if (mask) launch_zero(mask, sizeof(uint64_t) * (size_t)n_rows * mask_words, st);
    if ((e = cudaStreamWaitEvent(st, ss.join, 0))) return e;
    // (3) candidates: a persistent grid, warps claiming rows in order
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (K == 4) pw_candidates<4><<<(unsigned)sms * 2, kThreads, 0, st>>>(a, w);
    else pw_candidates<8><<<(unsigned)sms, kThreads, 0, st>>>(a, w);
    return cudaGetLastError();
}

}  // namespace dgal
