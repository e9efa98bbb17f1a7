/*
 * include/dgal.h — C ABI of libdgal.so: batched differentiable IoU of convex
 * polygons on NVIDIA B200 (sm_100a).  From-scratch implementation of the data-
 * parallel hot path of DGAL (arXiv 2011.11134).
 *
 * Citations: "P:n" = PAPER.md line n; "S:n" = SPEC.md line n; "R#" = reading in
 * DESIGN.md §3 (the paper is silent or ambiguous there).
 *
 * Conventions common to every call
 * --------------------------------
 *  - Poly2<float,K> batches (P:39 `typedef Poly2<float, 4> Quad2`; "stored in a
 *    fixed size point array ... in counter-clockwise order"): structure of arrays.
 *    Vertex k of polygon n is (x[n*K + k], y[n*K + k]).  Exactly K vertices per
 *    polygon, convex, counter-clockwise.  K is 4 or 8.
 *  - ALL pointers are DEVICE pointers owned by the caller (the one exception,
 *    dgal_iou_paired_host, takes host buffers); the library never allocates
 *    memory, never frees and never synchronises the host ("fix-size
 *    allocated memory"); its only state is a per-device cache of launch
 *    attributes (set once per kernel and device, thread-safe, idempotent),
 *    the host-buffer call's three streams and four events, and the indexed
 *    pairwise call's side stream and two events (its grid build overlaps the
 *    zero fill; fork / join with `stream`, capturable).
 *    Work is enqueued on `stream`
 *    (a cudaStream_t; NULL = legacy default stream).
 *  - Inputs are trusted: no CCW/convexity check on the device.
 *    Invalid polygons give unspecified but finite results.
 *  - Alignment: every x/y plane and gradient plane must be 16-byte aligned
 *    (float4 loads/stores); xflags must be 2K-byte aligned (8 B for K=4, 16 B
 *    for K=8); uint64 masks 8-byte aligned.  Violations -> DGAL_ERR_MISALIGNED.
 *  - n == 0 (or m == 0) is a no-op returning DGAL_OK; the one exception is
 *    dgal_iou_pairwise with n_rows > 0 and m == 0, which still zeroes
 *    nbr_count (when given): no row has a suppressor.
 *  - Errors are detected on the host before launch (nothing is enqueued); a
 *    launch failure (cudaGetLastError) returns DGAL_ERR_CUDA.  Asynchronous
 *    device faults surface at the caller's next synchronisation.
 *  - Results are bitwise deterministic: a pair's outputs depend only on that
 *    pair, whatever the batch size, launch shape or GPU count.
 *
 * Flag bytes xflags (R2, following S:102-103): FromP1(i) = 0x40|i, FromP2(j) =
 * 0x80|j, Cross(i,j) = 0xC0|i<<3|j (p1 edge i x p2 edge j), padding 0x00.  The
 * nx valid bytes list the intersection's vertices counter-clockwise,
 * starting at the first vertex met when walking p1's boundary counter-clockwise
 * from p1's vertex 0 (R3): a vertex on p1 edge i sits at boundary position
 * i + t (t in [0, 1) its parameter along that edge; FromP1(i) is t = 0), and the
 * sequence starts at the smallest position.  When no vertex of the intersection
 * lies on p1's boundary (p2 strictly inside p1) it is FromP2(0), FromP2(1), ...
 * Example (offset unit squares p1 = [0,1]^2, p2 = p1 + (0.5, 0.5)):
 * C8 42 D3 80 = Cross(1,0) FromP1(2) Cross(2,3) FromP2(0) — NOT sorted by byte
 * value.  nx == 0 <=> empty intersection (IoU 0).
 * Thin pairs (R^2 > 8 A_u, R the pair's extent about p1's vertex 0, A_u the union
 * area: the float decisions and area sum are conditioned by R^2 / A_u) get their
 * nx / xflags recomputed in double (the same rules) and their areas from that
 * record in double, in every entry point below.
 */
#ifndef DGAL_H_
#define DGAL_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    DGAL_OK = 0,
    DGAL_ERR_INVALID_ARG = 1,    /* negative size, NULL required pointer, bad cap */
    DGAL_ERR_UNSUPPORTED_K = 2,  /* K not in {4, 8} */
    DGAL_ERR_MISALIGNED = 3,     /* alignment rule above violated */
    DGAL_ERR_CUDA = 4            /* kernel launch failed */
} dgal_status;

/* Same type as cudaStream_t / CUstream. */
typedef struct CUstream_st *dgal_stream;

/*
 * Forward IoU of n independent pairs (the listing's `iou`):
 *   intersection = intersect(p1, p2, xflags); nx = intersection.nvertices;
 *   iou = area(intersection) / (area(p1) + area(p2) - area(intersection)).
 * p1 is the subject, p2 the clipper (R4).
 *   iou    [n]       float, overwritten
 *   nx     [n]       uint8, overwritten (0 or 3..2K)
 *   xflags [n * 2K]  uint8, overwritten (see flag bytes above)
 *
 * Polygons with m < K vertices (triangles in K = 4, 5..7-gons in K = 8): repeat the
 * last vertex K - m times; the result is the IoU of the m-gon, and the gradient of
 * that vertex is the SUM over its copies (tests/test_gpu_paired.py::test_padded_polygons).
 */
dgal_status dgal_iou_paired_fwd(int K, int64_t n,
                                const float *x1, const float *y1,
                                const float *x2, const float *y2,
                                float *iou, uint8_t *nx, uint8_t *xflags,
                                dgal_stream stream);

/*
 * Backward (the listing's `iou_backward` -> `iou_grad(p1, p2, grad, nx,
 * xflags, grad1, grad2)`): propagates grad_iou[k] = dL/dIoU_k to every vertex of
 * both polygons through the recorded nx/xflags of dgal_iou_paired_fwd on the
 * same inputs.  Outputs are OVERWRITTEN (not accumulated; P:52 declares fresh
 * grad1, grad2) in the input SoA layout (the polygon type holds the
 * gradient).  nx == 0 -> zero gradient (S:303 subgradient).
 *   grad_iou [n]; gx1, gy1, gx2, gy2 [n * K] float.
 */
dgal_status dgal_iou_paired_bwd(int K, int64_t n,
                                const float *x1, const float *y1,
                                const float *x2, const float *y2,
                                const float *grad_iou,
                                const uint8_t *nx, const uint8_t *xflags,
                                float *gx1, float *gy1, float *gx2, float *gy2,
                                dgal_stream stream);

/*
 * Forward + backward on HOST buffers (the end-to-end path of the north_star
 * metric: inputs arrive from and results return to host memory).  The same
 * computation as dgal_iou_paired_fwd then dgal_iou_paired_bwd — bitwise the same
 * iou and gradients — pipelined in chunks of `chunk` pairs over three library
 * streams: chunk c's host->device copies, forward, backward and device->host
 * copies run on stream c % 3, so PCIe traffic in both directions overlaps the
 * kernels of the other chunks.  nx / xflags stay on the device (workspace).
 *   x1, y1, x2, y2 [n * K], grad_iou [n]: HOST memory, read;
 *   iou [n], gx1, gy1, gx2, gy2 [n * K]: HOST memory, written.
 *   Page-locked (cudaHostAlloc / cudaHostRegister) host buffers give full PCIe
 *   speed; pageable ones work but the driver stages every copy.
 *   chunk     pairs per pipeline stage, > 0 and a multiple of 4 (2^21 is the
 *             measured optimum on B200).
 *   workspace >= dgal_paired_host_workspace_bytes(K, chunk) bytes of DEVICE
 *             memory (three staging slots), 256-byte aligned; no initialisation.
 * Ordering: the work starts after everything enqueued on `stream` before the
 * call and everything enqueued on `stream` after the call waits for it (event
 * fork / join).  Asynchronous like every call: the host buffers must stay valid
 * (inputs unmodified, outputs unread) until `stream` is synchronised; one call
 * at a time per workspace.  State: the first call on a device creates the three
 * streams and four events (kept for the process's lifetime; calls from several
 * host threads serialise on a lock while they enqueue).
 */
size_t dgal_paired_host_workspace_bytes(int K, int64_t chunk);

dgal_status dgal_iou_paired_host(int K, int64_t n,
                                 const float *x1, const float *y1,
                                 const float *x2, const float *y2,
                                 const float *grad_iou,
                                 float *iou,
                                 float *gx1, float *gy1, float *gx2, float *gy2,
                                 int64_t chunk, void *workspace, size_t workspace_bytes,
                                 dgal_stream stream);

/*
 * Fused forward + backward for an IoU loss whose upstream gradient is known
 * before the forward (e.g. L = mean(1 - IoU): dL/dIoU = -1/n).
 * One pass per pair computes the IoU and dL/d(vertices) from the same clip
 * intervals — no nx/xflags round trip through memory (the split API above is
 * the paper's; this is its fusion).  dL/dIoU of pair k is grad_iou[k] when
 * grad_iou != NULL, else grad_scale.  iou [n] nullable; gx1, gy1, gx2, gy2
 * [n * K] overwritten.  Alignment: planes and gradient planes 16 B, grad_iou
 * and iou 4 B, workspace 16 B (DGAL_ERR_MISALIGNED otherwise).
 *
 * Exactness (north_star tolerances on every input, like the split path): the
 * one-pass float arithmetic is not accurate enough for two rare kinds of pair —
 * a nearly parallel crossing (a p1 edge crossing a p2 edge's line at |sin| <
 * 2^-9, 2^-7 for boxes: float crossing parameters are conditioned by 1/sin) and
 * a thin pair (R^2 > 8 A_u, R the pair's extent: the float area sum is
 * conditioned by R^2 / A_u).  The first kernel queues them in `workspace` and a
 * second kernel, enqueued right after it, recomputes exactly those pairs with
 * the split path's arithmetic (dgal_iou_paired_fwd + _bwd: crossings refined in
 * double, thin records and areas in double), overwriting their iou and gradients.  Unqueued
 * pairs: IoU bit-identical to dgal_iou_pairwise, gradients equal to the split
 * path's up to rounding.
 *   workspace        >= dgal_fused_workspace_bytes(n) bytes of device memory
 *                    (a queue: {count, done, pad[2], idx[n]} of uint32),
 *                    ZERO-FILLED by the caller before its first use; every call
 *                    leaves it zero-filled again (the refine kernel resets the
 *                    counters), so it is reused across calls without clearing.
 *                    One workspace per stream: calls that may run concurrently
 *                    need separate workspaces.  NULL or too small ->
 *                    DGAL_ERR_INVALID_ARG.  n < 2^32 (32-bit queue entries).
 */
size_t dgal_fused_workspace_bytes(int64_t n);   /* 16 + 4 n, rounded up to 16 */

dgal_status dgal_iou_paired_fused(int K, int64_t n,
                                  const float *x1, const float *y1,
                                  const float *x2, const float *y2,
                                  const float *grad_iou, float grad_scale,
                                  float *iou,
                                  float *gx1, float *gy1, float *gx2, float *gy2,
                                  void *workspace, size_t workspace_bytes,
                                  dgal_stream stream);

/*
 * Rotated-box front end (SPEC metrics-boxes S:336-418;
 * P:73, "2D IoU Loss and 3D IoU Loss for rotated bounding boxes").
 * Boxes are given as parameters and converted to Poly2<float,4> inside the
 * kernels by box_to_polygon: corners c + R(theta)(+-w/2, +-h/2), CCW,
 * starting at (-w/2, -h/2) — so nx / xflags are those of dgal_iou_paired_fwd
 * on these corners (K = 4, 8 flag bytes per pair).
 *   dims 2: RotatedBox2 (cx, cy, w, h, theta)          P = 5 parameters
 *   dims 3: yaw-only Box3 (cx, cy, cz, w, h, d, theta)  P = 7 parameters;
 *           IoU = V_i / (V_1 + V_2 - V_i), V_i = A_i dz, dz = overlap of the
 *           z extents [cz - d/2, cz + d/2]; dz == 0 -> IoU 0, nx 0.
 * theta is in radians, unbounded (cos / sin to ~1e-7 rad at any |theta| up to ~1e4:
 * float(theta/pi) plus a first-order correction by the part it misses); w, h, d > 0 (inputs
 * are trusted).
 * layout DGAL_BOX_PLANES: parameter p of box k at b[p * n + k] (a [P, n] tensor,
 *        coalesced: the fast layout); DGAL_BOX_ROWS: at b[k * P + p] ([n, P]).
 * Gradients use the layout of the inputs and are OVERWRITTEN; they are the
 * chain of the polygon backward with box_to_polygon_grad and, in 3D,
 * the product rule through dz (+-1/0 subgradient of min/max; ties -> box 1)
 * and V = A d.  Pointers: 4-byte aligned floats; xflags 8-byte aligned.
 * Errors: dims not 2/3 or bad layout -> DGAL_ERR_INVALID_ARG; the rest as above.
 */
typedef enum { DGAL_BOX_PLANES = 0, DGAL_BOX_ROWS = 1 } dgal_box_layout;

dgal_status dgal_box_iou_paired_fwd(int dims, int layout, int64_t n,
                                    const float *b1, const float *b2,
                                    float *iou /*[n]*/, uint8_t *nx /*[n]*/,
                                    uint8_t *xflags /*[n * 8]*/,
                                    dgal_stream stream);

dgal_status dgal_box_iou_paired_bwd(int dims, int layout, int64_t n,
                                    const float *b1, const float *b2,
                                    const float *grad_iou /*[n]*/,
                                    const uint8_t *nx, const uint8_t *xflags,
                                    float *grad_b1, float *grad_b2 /*like b1, b2*/,
                                    dgal_stream stream);

/* fused forward + backward (f2 on boxes): dL/dIoU = grad_iou[k], or grad_scale
 * when grad_iou == NULL; iou nullable; workspace: the refine queue as for
 * dgal_iou_paired_fused (dgal_fused_workspace_bytes(n), zero-filled once; the
 * queued pairs are redone with the box split path's arithmetic). */
dgal_status dgal_box_iou_paired_fused(int dims, int layout, int64_t n,
                                      const float *b1, const float *b2,
                                      const float *grad_iou, float grad_scale,
                                      float *iou,
                                      float *grad_b1, float *grad_b2,
                                      void *workspace, size_t workspace_bytes,
                                      dgal_stream stream);

/*
 * Pairwise IoU of a row block against all columns ("cartesian";
 * north_star "full N x M pairwise matrices (detection/NMS)"), forward only.
 * Rows play p1, columns p2 (R4).  Row r has global index row_offset + r; column c
 * has global index c (for NMS pass the same score-sorted boxes as columns and
 * the caller's row block as rows).
 *   iou   [n_rows * m] float, row-major (ld = m), nullable.
 *   mask  [n_rows * mask_words] uint64, nullable, mask_words >= ceil(m/64):
 *         bit c of row r  <=>  c != row_offset + r  and  IoU(r, c) > nms_thresh
 *         (strict, R14).  Bits c > row_offset + r form the classic NMS
 *         suppression row; bits c < row_offset + r are the boxes that can
 *         suppress box row_offset + r.  Words beyond ceil(m/64) are untouched
 *         by the tiled path and zeroed by the indexed path.
 *   nbr_count [n_rows], nbr_idx [n_rows * nbr_cap] int32, nullable (both or
 *         neither; requires mask):  the list of columns c < row_offset + r with
 *         IoU > nms_thresh, in no particular order; nbr_count[r] is the true
 *         count (it may exceed nbr_cap, then only nbr_cap entries are stored).
 *         The library zeroes nbr_count itself (cudaMemsetAsync on `stream`).
 *   workspace, workspace_bytes: nullable.  With a device workspace of at least
 *         dgal_pairwise_workspace_bytes(m) bytes the INDEXED path runs: the
 *         outputs are zero-filled at streaming-write speed and only pairs whose
 *         bounding circles intersect are evaluated, found through a uniform grid
 *         over the column circles built in the workspace (best for large sparse
 *         problems, e.g. 1e5 x 1e5).  Without one the TILED path sweeps every
 *         pair through shared-memory column tiles.  Both give the same outputs
 *         (mask/list bit-identical; IoU identical pair by pair).
 */
size_t dgal_pairwise_workspace_bytes(int64_t m);

dgal_status dgal_iou_pairwise(int K, int64_t n_rows,
                              const float *row_x, const float *row_y,
                              int64_t m,
                              const float *col_x, const float *col_y,
                              int64_t row_offset,
                              float *iou,
                              float nms_thresh,
                              uint64_t *mask, int64_t mask_words,
                              int32_t *nbr_count, int32_t *nbr_idx, int32_t nbr_cap,
                              void *workspace, size_t workspace_bytes,
                              dgal_stream stream);

/*
 * Greedy rotated NMS keep decision (north_star "rotated-NMS keep mask"; textbook
 * greedy order, R14): boxes sorted by descending score; box i is kept iff no KEPT
 * box k < i has IoU(i, k) > thr.  Computed as the unique fixed point of that
 * recursion by parallel rounds: a box whose suppressors are all
 * removed is kept, a box with a kept suppressor is removed.
 *
 * dgal_nms_round: ONE round over the rows [row_offset, row_offset + n_rows) of an
 *   n_total-box problem (one rank's row block).  Reads the global status vector
 *   `status` [n_total] (0 undecided, 1 kept, 2 removed), updates the entries of
 *   its own rows in place, and atomically adds the number of its rows still
 *   undecided to *undecided (device int32; the caller zeroes it).  Uses nbr lists
 *   when nbr_count[r] <= nbr_cap, else scans the lower part of mask row r.
 *   scratch (nullable, >= 2 int32, 4-byte aligned, device): with it the round
 *   runs to the rank-local fixed point — passes over the rows, grid-wide barriers
 *   between them (a cooperative launch), until a pass decides nothing new, so
 *   only suppression chains that cross row blocks need further rounds; without
 *   it, one pass.  Either way the rounds converge to the same keep vector.
 * dgal_nms_keep: all rounds for a single-GPU problem (rows = all n boxes,
 *   row_offset = 0) in one kernel (no host round trips); writes keep[i] in {0,1}.
 *   status [n] is caller-provided scratch.  scratch (nullable, >= 2 int32, 4-byte
 *   aligned, device): with it the rounds run grid-wide (a cooperative launch, one
 *   box per thread, grid-wide barriers between rounds); without it, in a single
 *   1024-thread CTA (same result).
 * mask / nbr_* are exactly the outputs of dgal_iou_pairwise with the same thr.
 */
dgal_status dgal_nms_round(int64_t n_total, int64_t n_rows, int64_t row_offset,
                           const uint64_t *mask, int64_t mask_words,
                           const int32_t *nbr_count, const int32_t *nbr_idx, int32_t nbr_cap,
                           uint8_t *status, int32_t *undecided, int32_t *scratch,
                           dgal_stream stream);

dgal_status dgal_nms_keep(int64_t n,
                          const uint64_t *mask, int64_t mask_words,
                          const int32_t *nbr_count, const int32_t *nbr_idx, int32_t nbr_cap,
                          uint8_t *status, uint8_t *keep, int32_t *scratch,
                          dgal_stream stream);

/* Human-readable name of a status code (static storage). */
const char *dgal_status_string(dgal_status s);

/* Build description: "libdgal <version> sm_100a nvcc <ver>" (static storage). */
const char *dgal_build_info(void);

#ifdef __cplusplus
}
#endif

#endif /* DGAL_H_ */
