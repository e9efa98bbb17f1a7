"""paper_2011_11134_b200 — batched differentiable IoU of convex polygons on B200.

Thin Python binding of libdgal.so (include/dgal.h), argument marshalling only:
every step of the method runs in the CUDA kernels behind the C ABI.  PyTorch
supplies device memory and the current CUDA stream.  There is no CPU path.

Polygon batches are two float32 CUDA tensors (x, y) of shape [n, K] (or flat
[n*K]), K in {4, 8}, vertices counter-clockwise.

    iou, nx, xflags = iou_paired_fwd(x1, y1, x2, y2)
    gx1, gy1, gx2, gy2 = iou_paired_bwd(x1, y1, x2, y2, g, nx, xflags)
    iou, mask, cnt, idx = iou_pairwise(rx, ry, cx, cy, ...)    # N x M + NMS mask
    keep = nms_keep(mask, cnt, idx)                           # greedy rotated NMS
    loss-side autograd: PolyIoU.apply(x1, y1, x2, y2)
"""
from __future__ import annotations

import torch

from ._lib import DgalError, call, lib  # noqa: F401

__all__ = ["iou_paired_fwd", "iou_paired_bwd", "iou_paired_fused", "iou_paired", "iou_paired_backward", "PolyIoULoss",
           "box_iou_paired_fwd", "box_iou_paired_bwd", "box_iou_paired_fused", "BoxIoU", "BoxIoULoss", "iou_pairwise", "pairwise_workspace", "fused_workspace", "iou_paired_host", "nms_round", "nms_keep",
           "nms", "PolyIoU", "DgalError", "build_info"]


def build_info() -> str:
    return lib().dgal_build_info().decode()


def _stream(device) -> int:
    return torch.cuda.current_stream(device).cuda_stream


def _plane(t: torch.Tensor, name: str, dtype=torch.float32, numel: int | None = None,
           device=None) -> torch.Tensor:
    """Validate one tensor handed to the C ABI: a contiguous CUDA tensor of `dtype`
    (on `device`, with `numel` elements when given).  The ABI receives raw pointers
    and cannot check sizes, so a short buffer here would be an out-of-bounds device
    access, not an error: every input and out= tensor goes through this."""
    if not isinstance(t, torch.Tensor) or not t.is_cuda:
        raise TypeError(f"{name}: expected a CUDA tensor (there is no CPU path)")
    if t.dtype != dtype:
        raise TypeError(f"{name}: expected {dtype}, got {t.dtype}")
    if not t.is_contiguous():
        raise ValueError(f"{name}: must be contiguous")
    if device is not None and t.device != device:
        raise ValueError(f"{name}: on {t.device}, expected {device} (all tensors of a call share one device)")
    if numel is not None and t.numel() != numel:
        raise ValueError(f"{name}: {t.numel()} elements, expected {numel}")
    return t


def _planes(K, n, dev, **ts):
    for nm, t in ts.items():
        _plane(t, nm, numel=n * K, device=dev)


def _K_n(x: torch.Tensor, K: int | None):
    if K is None:
        if x.dim() != 2:
            raise ValueError("pass K= for flat coordinate planes")
        K = x.shape[-1]
    n = x.numel() // K
    if n * K != x.numel():
        raise ValueError("plane size is not a multiple of K")
    return K, n


def _ptr(t):
    return None if t is None else t.data_ptr()


_FUSED_WS = {}


def fused_workspace(n: int, device=None, stream=None) -> torch.Tensor:
    """Refine queue of the fused kernels (dgal_fused_workspace_bytes(n) bytes, zero-filled
    once; every call leaves it zero-filled).  Cached per (device, stream) — one
    workspace per stream, as include/dgal.h requires — and grown on demand."""
    dev = torch.device(device or "cuda")
    if dev.index is None:
        dev = torch.device("cuda", torch.cuda.current_device())
    st = stream if stream is not None else _stream(dev)
    need = int(lib().dgal_fused_workspace_bytes(int(n)))
    ws = _FUSED_WS.get((dev, st))
    if ws is None or ws.numel() < need:
        ws = torch.zeros(max(need, 16), dtype=torch.uint8, device=dev)
        _FUSED_WS[(dev, st)] = ws
    return ws


def iou_paired_fwd(x1, y1, x2, y2, K: int | None = None, out=None):
    """Forward IoU of n pairs (dgal_iou_paired_fwd).  Returns (iou f32[n], nx u8[n],
    xflags u8[n, 2K]); `out` may supply those three tensors."""
    _plane(x1, "x1")
    K, n = _K_n(x1, K)
    dev = x1.device
    _planes(K, n, dev, x1=x1, y1=y1, x2=x2, y2=y2)
    if out is None:
        iou = torch.empty(n, dtype=torch.float32, device=dev)
        nx = torch.empty(n, dtype=torch.uint8, device=dev)
        xf = torch.empty((n, 2 * K), dtype=torch.uint8, device=dev)
    else:
        iou, nx, xf = out
        _plane(iou, "iou", numel=n, device=dev)
        _plane(nx, "nx", torch.uint8, n, dev)
        _plane(xf, "xflags", torch.uint8, 2 * K * n, dev)
    call("dgal_iou_paired_fwd", K, n, _ptr(x1), _ptr(y1), _ptr(x2), _ptr(y2), _ptr(iou), _ptr(nx),
         _ptr(xf), _stream(dev))
    return iou, nx, xf


def iou_paired_bwd(x1, y1, x2, y2, grad_iou, nx, xflags, K: int | None = None, out=None):
    """iou_grad (dgal_iou_paired_bwd): returns (gx1, gy1, gx2, gy2), each shaped like x1."""
    _plane(x1, "x1")
    K, n = _K_n(x1, K)
    dev = x1.device
    _planes(K, n, dev, x1=x1, y1=y1, x2=x2, y2=y2)
    _plane(grad_iou, "grad_iou", numel=n, device=dev)
    _plane(nx, "nx", torch.uint8, n, dev)
    _plane(xflags, "xflags", torch.uint8, 2 * K * n, dev)
    if out is None:
        out = tuple(torch.empty_like(x1) for _ in range(4))
    gx1, gy1, gx2, gy2 = out
    _planes(K, n, dev, gx1=gx1, gy1=gy1, gx2=gx2, gy2=gy2)
    call("dgal_iou_paired_bwd", K, n, _ptr(x1), _ptr(y1), _ptr(x2), _ptr(y2), _ptr(grad_iou), _ptr(nx),
         _ptr(xflags), _ptr(gx1), _ptr(gy1), _ptr(gx2), _ptr(gy2), _stream(x1.device))
    return gx1, gy1, gx2, gy2


def _host_plane(t, name, numel):
    """A host buffer handed to dgal_iou_paired_host: contiguous CPU float32 of
    `numel` elements (pinned memory gives full PCIe speed)."""
    if not isinstance(t, torch.Tensor) or t.is_cuda:
        raise TypeError(f"{name}: expected a CPU (host) tensor")
    if t.dtype != torch.float32 or not t.is_contiguous() or t.numel() != numel:
        raise ValueError(f"{name}: expected a contiguous float32 tensor of {numel} elements")
    return t


_HOST_WS = {}


def iou_paired_host(x1, y1, x2, y2, grad_iou, K: int | None = None, out=None, chunk: int = 1 << 21,
                    device=None, workspace: torch.Tensor | None = None):
    """Forward + backward on HOST tensors (dgal_iou_paired_host): the chunked
    three-stream pipeline of host->device copies, forward, backward and
    device->host copies runs inside the library.  Inputs and `out` = (iou, gx1,
    gy1, gx2, gy2) are CPU tensors (pin them for full PCIe speed).  Asynchronous
    on the current stream of `device`: synchronise before reading the outputs."""
    K, n = _K_n(x1, K)
    for nm, t in (("x1", x1), ("y1", y1), ("x2", x2), ("y2", y2)):
        _host_plane(t, nm, n * K)
    _host_plane(grad_iou, "grad_iou", n)
    if out is None:
        pin = x1.is_pinned()
        out = (torch.empty(n, dtype=torch.float32, pin_memory=pin),
               *(torch.empty(tuple(x1.shape), dtype=torch.float32, pin_memory=pin) for _ in range(4)))
    iou, gx1, gy1, gx2, gy2 = out
    _host_plane(iou, "iou", n)
    for nm, t in (("gx1", gx1), ("gy1", gy1), ("gx2", gx2), ("gy2", gy2)):
        _host_plane(t, nm, n * K)
    dev = torch.device(device or "cuda")
    if dev.index is None:
        dev = torch.device("cuda", torch.cuda.current_device())
    need = int(lib().dgal_paired_host_workspace_bytes(K, int(chunk)))
    if workspace is None:
        workspace = _HOST_WS.get((dev, K, chunk))
        if workspace is None:
            workspace = torch.empty(max(need, 256), dtype=torch.uint8, device=dev)
            _HOST_WS[(dev, K, chunk)] = workspace
    _plane(workspace, "workspace", torch.uint8, device=dev)
    with torch.cuda.device(dev):
        call("dgal_iou_paired_host", K, n, _ptr(x1), _ptr(y1), _ptr(x2), _ptr(y2), _ptr(grad_iou), _ptr(iou),
             _ptr(gx1), _ptr(gy1), _ptr(gx2), _ptr(gy2), int(chunk), _ptr(workspace), workspace.numel(),
             _stream(dev))
    return out


def iou_paired_fused(x1, y1, x2, y2, grad=None, scale: float = 1.0, K: int | None = None, out=None,
                     want_iou: bool = True, workspace: torch.Tensor | None = None):
    """Fused loss forward + backward (dgal_iou_paired_fused): dL/dIoU = grad[k] (a
    CUDA float tensor [n]) or the scalar `scale`.  Returns (iou | None, gx1, gy1, gx2, gy2).
    workspace: the refine queue (fused_workspace(n), cached per stream when omitted)."""
    _plane(x1, "x1")
    K, n = _K_n(x1, K)
    dev = x1.device
    _planes(K, n, dev, x1=x1, y1=y1, x2=x2, y2=y2)
    if grad is not None:
        _plane(grad, "grad", numel=n, device=dev)
    if out is None:
        iou = torch.empty(n, dtype=torch.float32, device=dev) if want_iou else None
        g4 = tuple(torch.empty_like(x1) for _ in range(4))
    else:
        iou, g4 = out[0], out[1:]
    if iou is not None:
        _plane(iou, "iou", numel=n, device=dev)
    _planes(K, n, dev, gx1=g4[0], gy1=g4[1], gx2=g4[2], gy2=g4[3])
    ws = fused_workspace(n, dev) if workspace is None else _plane(workspace, "workspace", torch.uint8, device=dev)
    call("dgal_iou_paired_fused", K, n, _ptr(x1), _ptr(y1), _ptr(x2), _ptr(y2), _ptr(grad), float(scale),
         _ptr(iou), *[_ptr(t) for t in g4], _ptr(ws), ws.numel(), _stream(dev))
    return (iou, *g4)


class PolyIoULoss(torch.autograd.Function):
    """L = mean(1 - IoU) over the pairs, forward and backward in ONE kernel pass
    (dgal_iou_paired_fused with dL/dIoU = -1/n; the backward scales the stored
    vertex gradients by the incoming dL — exact, the kernel is linear in it)."""

    @staticmethod
    def forward(ctx, x1, y1, x2, y2):
        x1, y1, x2, y2 = (t.contiguous() for t in (x1, y1, x2, y2))
        n = x1.shape[0]
        iou, g1x, g1y, g2x, g2y = iou_paired_fused(x1, y1, x2, y2, scale=-1.0 / max(n, 1))
        ctx.save_for_backward(g1x, g1y, g2x, g2y)
        return (1.0 - iou).mean()

    @staticmethod
    def backward(ctx, dl):
        return tuple(g * dl for g in ctx.saved_tensors)


# ---------------------------------------------------------------------------
# rotated boxes: dims 2 -> (cx, cy, w, h, theta), dims 3 ->
# (cx, cy, cz, w, h, d, theta).  layout "planes": a [P, n] tensor (coalesced, the
# fast layout); "rows": an [n, P] tensor.
# ---------------------------------------------------------------------------
_LAYOUT = {"planes": 0, "rows": 1}


def _box_args(b1, b2, layout):
    if layout not in _LAYOUT:
        raise ValueError("layout must be 'planes' or 'rows'")
    _plane(b1, "b1")
    _plane(b2, "b2", device=b1.device)
    if b1.dim() != 2 or b1.shape != b2.shape:
        raise ValueError("b1, b2 must be 2-D tensors of the same shape")
    P, n = (b1.shape[0], b1.shape[1]) if layout == "planes" else (b1.shape[1], b1.shape[0])
    if P not in (5, 7):
        raise ValueError(f"{P} box parameters: expected 5 (2D) or 7 (3D) for layout {layout!r}")
    return (3 if P == 7 else 2), _LAYOUT[layout], n


def box_iou_paired_fwd(b1, b2, layout: str = "planes", out=None):
    """IoU of n box pairs (dgal_box_iou_paired_fwd).  Returns (iou f32[n], nx u8[n],
    xflags u8[n, 8]) — nx / xflags of the BEV corner polygons (K = 4)."""
    dims, lay, n = _box_args(b1, b2, layout)
    if out is None:
        dev = b1.device
        out = (torch.empty(n, dtype=torch.float32, device=dev), torch.empty(n, dtype=torch.uint8, device=dev),
               torch.empty(n, 8, dtype=torch.uint8, device=dev))
    iou, nx, xf = out
    dev = b1.device
    _plane(iou, "iou", numel=n, device=dev)
    _plane(nx, "nx", torch.uint8, n, dev)
    _plane(xf, "xflags", torch.uint8, 8 * n, dev)
    call("dgal_box_iou_paired_fwd", dims, lay, n, _ptr(b1), _ptr(b2), _ptr(iou), _ptr(nx), _ptr(xf),
         _stream(b1.device))
    return iou, nx, xf


def box_iou_paired_bwd(b1, b2, grad_iou, nx, xflags, layout: str = "planes", out=None):
    """dL/d(box parameters) from dL/dIoU through the recorded nx / xflags
    (dgal_box_iou_paired_bwd).  Returns (grad_b1, grad_b2) shaped like b1, b2."""
    dims, lay, n = _box_args(b1, b2, layout)
    dev = b1.device
    _plane(grad_iou, "grad_iou", numel=n, device=dev)
    _plane(nx, "nx", torch.uint8, n, dev)
    _plane(xflags, "xflags", torch.uint8, 8 * n, dev)
    if out is None:
        out = (torch.empty_like(b1), torch.empty_like(b2))
    _plane(out[0], "grad_b1", numel=b1.numel(), device=dev)
    _plane(out[1], "grad_b2", numel=b1.numel(), device=dev)
    call("dgal_box_iou_paired_bwd", dims, lay, n, _ptr(b1), _ptr(b2), _ptr(grad_iou), _ptr(nx), _ptr(xflags),
         _ptr(out[0]), _ptr(out[1]), _stream(b1.device))
    return out


def box_iou_paired_fused(b1, b2, grad=None, scale: float = 1.0, layout: str = "planes", out=None,
                         want_iou: bool = True, workspace: torch.Tensor | None = None):
    """Fused forward + backward on boxes (dgal_box_iou_paired_fused).  Returns
    (iou | None, grad_b1, grad_b2); workspace as for iou_paired_fused."""
    dims, lay, n = _box_args(b1, b2, layout)
    dev = b1.device
    if grad is not None:
        _plane(grad, "grad", numel=n, device=dev)
    if out is None:
        iou = torch.empty(n, dtype=torch.float32, device=dev) if want_iou else None
        out = (iou, torch.empty_like(b1), torch.empty_like(b2))
    iou, g1, g2 = out
    if iou is not None:
        _plane(iou, "iou", numel=n, device=dev)
    _plane(g1, "grad_b1", numel=b1.numel(), device=dev)
    _plane(g2, "grad_b2", numel=b1.numel(), device=dev)
    ws = fused_workspace(n, dev) if workspace is None else _plane(workspace, "workspace", torch.uint8, device=dev)
    call("dgal_box_iou_paired_fused", dims, lay, n, _ptr(b1), _ptr(b2), _ptr(grad), float(scale), _ptr(iou),
         _ptr(g1), _ptr(g2), _ptr(ws), ws.numel(), _stream(dev))
    return iou, g1, g2


class BoxIoU(torch.autograd.Function):
    """Differentiable rotated-box IoU (2D or yaw-only 3D): forward =
    dgal_box_iou_paired_fwd, backward = dgal_box_iou_paired_bwd."""

    @staticmethod
    def forward(ctx, b1, b2, layout="planes"):
        b1, b2 = b1.contiguous(), b2.contiguous()
        iou, nx, xf = box_iou_paired_fwd(b1, b2, layout)
        ctx.layout = layout
        ctx.save_for_backward(b1, b2, nx, xf)
        return iou

    @staticmethod
    def backward(ctx, g):
        b1, b2, nx, xf = ctx.saved_tensors
        g1, g2 = box_iou_paired_bwd(b1, b2, g.contiguous().float(), nx, xf, ctx.layout)
        return g1, g2, None


class BoxIoULoss(torch.autograd.Function):
    """L = mean(1 - IoU) over box pairs in one fused kernel pass (dL/dIoU = -1/n)."""

    @staticmethod
    def forward(ctx, b1, b2, layout="planes"):
        b1, b2 = b1.contiguous(), b2.contiguous()
        n = b1.shape[1] if layout == "planes" else b1.shape[0]
        iou, g1, g2 = box_iou_paired_fused(b1, b2, scale=-1.0 / max(n, 1), layout=layout)
        ctx.save_for_backward(g1, g2)
        return (1.0 - iou).mean()

    @staticmethod
    def backward(ctx, dl):
        g1, g2 = ctx.saved_tensors
        return g1 * dl, g2 * dl, None


def pairwise_workspace(m: int, device=None) -> torch.Tensor:
    """Device workspace for the indexed pairwise path (dgal_pairwise_workspace_bytes)."""
    nb = int(lib().dgal_pairwise_workspace_bytes(int(m)))
    return torch.empty(nb, dtype=torch.uint8, device=device or "cuda")


def iou_pairwise(rx, ry, cx, cy, K: int | None = None, row_offset: int = 0, thr: float = 0.7,
                 want_iou: bool = True, want_mask: bool = True, nbr_cap: int = 0, out=None,
                 indexed: bool = True, workspace: torch.Tensor | None = None):
    """Pairwise IoU of rows x columns (dgal_iou_pairwise).  Returns
    (iou f32[nr, m] | None, mask u64[nr, ceil(m/64)] | None, nbr_count i32[nr] | None,
     nbr_idx i32[nr, nbr_cap] | None).  mask/nbr semantics: include/dgal.h.
    indexed=True uses the grid-indexed path (a workspace is allocated unless given),
    indexed=False the tiled sweep."""
    _plane(rx, "rx")
    _plane(cx, "cx", device=rx.device)
    K, nr = _K_n(rx, K)
    _, m = _K_n(cx, K)
    dev = rx.device
    _planes(K, nr, dev, rx=rx, ry=ry)
    _planes(K, m, dev, cx=cx, cy=cy)
    words = (m + 63) // 64
    if out is not None:
        iou, mask, cnt, idx = out
        if iou is not None:
            _plane(iou, "iou", numel=nr * m, device=dev)
        if mask is not None:
            _plane(mask, "mask", torch.int64, nr * words, dev)
        if (cnt is None) != (idx is None):
            raise ValueError("nbr_count and nbr_idx go together")
        if cnt is not None:
            _plane(cnt, "nbr_count", torch.int32, nr, dev)
            if idx.dim() != 2 or idx.shape[0] != nr:
                raise ValueError(f"nbr_idx: expected shape [{nr}, cap], got {tuple(idx.shape)}")
            _plane(idx, "nbr_idx", torch.int32, device=dev)
    else:
        iou = torch.empty((nr, m), dtype=torch.float32, device=dev) if want_iou else None
        mask = torch.empty((nr, words), dtype=torch.int64, device=dev) if want_mask else None
        cnt = torch.empty(nr, dtype=torch.int32, device=dev) if nbr_cap > 0 else None
        idx = torch.empty((nr, nbr_cap), dtype=torch.int32, device=dev) if nbr_cap > 0 else None
    if indexed and workspace is None:
        workspace = pairwise_workspace(m, dev)
    if indexed:
        _plane(workspace, "workspace", torch.uint8, device=dev)
        need = int(lib().dgal_pairwise_workspace_bytes(int(m)))
        if workspace.numel() < need:
            raise ValueError(f"workspace: {workspace.numel()} bytes, need {need}")
    ws = workspace if indexed else None
    call("dgal_iou_pairwise", K, nr, _ptr(rx), _ptr(ry), m, _ptr(cx), _ptr(cy), int(row_offset), _ptr(iou),
         float(thr), _ptr(mask), words if mask is not None else 0, _ptr(cnt), _ptr(idx),
         int(idx.shape[1] if idx is not None else 0), _ptr(ws), int(ws.numel()) if ws is not None else 0,
         _stream(dev))
    return iou, mask, cnt, idx


def _nbr_check(nbr_count, nbr_idx, n_rows, dev) -> int:
    """Validate the optional suppressor lists; returns their capacity (0 if absent)."""
    if nbr_count is None and nbr_idx is None:
        return 0
    if (nbr_count is None) != (nbr_idx is None):
        raise ValueError("nbr_count and nbr_idx go together")
    _plane(nbr_count, "nbr_count", torch.int32, n_rows, dev)
    _plane(nbr_idx, "nbr_idx", torch.int32, device=dev)
    if nbr_idx.dim() != 2 or nbr_idx.shape[0] != n_rows:
        raise ValueError(f"nbr_idx: expected shape [{n_rows}, cap], got {tuple(nbr_idx.shape)}")
    return nbr_idx.shape[1]


def nms_round(n_total: int, row_offset: int, mask, nbr_count, nbr_idx, status, undecided, scratch=None):
    """One parallel NMS round over this rank's rows (dgal_nms_round); with `scratch`
    (int32 [>= 2], device) the round runs to the rank-local fixed point."""
    _plane(mask, "mask", torch.int64)
    dev = mask.device
    n_rows = mask.shape[0]
    if mask.dim() != 2 or mask.shape[1] != (n_total + 63) // 64:
        raise ValueError(f"mask: expected shape [n_rows, {(n_total + 63) // 64}], got {tuple(mask.shape)}")
    cap = _nbr_check(nbr_count, nbr_idx, n_rows, dev)
    _plane(status, "status", torch.uint8, device=dev)
    if status.numel() < n_total or row_offset < 0 or row_offset + n_rows > status.numel():
        raise ValueError(f"status: {status.numel()} entries for n_total {n_total}, rows "
                         f"[{row_offset}, {row_offset + n_rows})")
    _plane(undecided, "undecided", torch.int32, 1, dev)
    if scratch is not None:
        _plane(scratch, "scratch", torch.int32, device=dev)
        if scratch.numel() < 2:
            raise ValueError("scratch: needs >= 2 int32")
    call("dgal_nms_round", int(n_total), n_rows, int(row_offset), _ptr(mask), mask.shape[1], _ptr(nbr_count),
         _ptr(nbr_idx), cap, _ptr(status), _ptr(undecided), _ptr(scratch), _stream(mask.device))


def nms_keep(mask, nbr_count=None, nbr_idx=None, status=None, keep=None, grid: bool = True):
    """Greedy NMS keep vector u8[n] from a single-GPU pairwise mask (dgal_nms_keep).
    grid=True runs the rounds grid-wide (cooperative launch); False in one CTA."""
    _plane(mask, "mask", torch.int64)
    n = mask.shape[0]
    dev = mask.device
    if mask.dim() != 2 or mask.shape[1] != (n + 63) // 64:
        raise ValueError(f"mask: expected shape [{n}, {(n + 63) // 64}], got {tuple(mask.shape)}")
    cap = _nbr_check(nbr_count, nbr_idx, n, dev)
    status = torch.empty(n, dtype=torch.uint8, device=dev) if status is None else status
    keep = torch.empty(n, dtype=torch.uint8, device=dev) if keep is None else keep
    _plane(status, "status", torch.uint8, n, dev)
    _plane(keep, "keep", torch.uint8, n, dev)
    scratch = torch.empty(2, dtype=torch.int32, device=dev) if grid else None
    call("dgal_nms_keep", n, _ptr(mask), mask.shape[1], _ptr(nbr_count), _ptr(nbr_idx), cap, _ptr(status),
         _ptr(keep), _ptr(scratch), _stream(dev))
    return keep


def nms(x, y, thr: float = 0.7, K: int | None = None, nbr_cap: int = 64):
    """Rotated NMS of score-sorted polygons: pairwise mask + keep (single GPU)."""
    _, mask, cnt, idx = iou_pairwise(x, y, x, y, K=K, thr=thr, want_iou=False, want_mask=True,
                                     nbr_cap=nbr_cap)
    return nms_keep(mask, cnt, idx)


class PolyIoU(torch.autograd.Function):
    """Differentiable paired IoU: forward = dgal_iou_paired_fwd, backward =
    dgal_iou_paired_bwd through the saved nx / xflags (the paper's listing)."""

    @staticmethod
    def forward(ctx, x1, y1, x2, y2):
        x1, y1, x2, y2 = (t.contiguous() for t in (x1, y1, x2, y2))
        iou, nx, xf = iou_paired_fwd(x1, y1, x2, y2)
        ctx.save_for_backward(x1, y1, x2, y2, nx, xf)
        return iou

    @staticmethod
    def backward(ctx, g):
        x1, y1, x2, y2, nx, xf = ctx.saved_tensors
        return iou_paired_bwd(x1, y1, x2, y2, g.contiguous().float(), nx, xf)


# SURVEY §8(b) shim names (same functions)
iou_paired = iou_paired_fwd
iou_paired_backward = iou_paired_bwd
