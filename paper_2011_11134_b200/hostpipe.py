"""End-to-end paired IoU fwd+bwd on HOST buffers: chunked, multi-stream pipeline
of host->device copy, dgal_iou_paired_fwd, dgal_iou_paired_bwd and device->host
copy, so PCIe traffic in both directions overlaps the kernels.
PyTorch provides pinned buffers, streams and copies; the compute is libdgal."""
from __future__ import annotations

import torch

from . import iou_paired_bwd, iou_paired_fwd


class HostPipeline:
    """Preallocates device staging for `nstreams` chunks of `chunk` pairs."""

    def __init__(self, K: int, chunk: int = 1 << 21, nstreams: int = 3, device=None):
        self.K, self.chunk, self.ns = K, chunk, nstreams
        self.dev = torch.device(device or "cuda")
        self.streams = [torch.cuda.Stream(self.dev) for _ in range(nstreams)]
        f32 = dict(dtype=torch.float32, device=self.dev)
        self.buf = []
        for _ in range(nstreams):
            self.buf.append(dict(
                xin=torch.empty((4, chunk, K), **f32), g=torch.empty(chunk, **f32),
                iou=torch.empty(chunk, **f32), nx=torch.empty(chunk, dtype=torch.uint8, device=self.dev),
                xf=torch.empty((chunk, 2 * K), dtype=torch.uint8, device=self.dev),
                gout=torch.empty((4, chunk, K), **f32)))

    def run(self, x4_host: torch.Tensor, g_host: torch.Tensor, iou_host: torch.Tensor,
            grad4_host: torch.Tensor) -> None:
        """x4_host: pinned [4, n, K] (x1, y1, x2, y2); g_host: pinned [n];
        outputs iou_host [n], grad4_host [4, n, K] (pinned).  Returns when done."""
        n = g_host.numel()
        cur = torch.cuda.current_stream(self.dev)
        for s in self.streams:
            s.wait_stream(cur)
        c = 0
        for off in range(0, n, self.chunk):
            m = min(self.chunk, n - off)
            s = self.streams[c % self.ns]
            b = self.buf[c % self.ns]
            with torch.cuda.stream(s):
                # one contiguous copy per plane (a strided [4, m, K] copy is slow)
                planes = [b["xin"][i, :m] for i in range(4)]
                for i in range(4):
                    planes[i].copy_(x4_host[i, off:off + m], non_blocking=True)
                g = b["g"][:m]
                g.copy_(g_host[off:off + m], non_blocking=True)
                iou, nx, xf = iou_paired_fwd(*planes, out=(b["iou"][:m], b["nx"][:m], b["xf"][:m]))
                go = [b["gout"][i, :m] for i in range(4)]
                iou_paired_bwd(*planes, g, nx, xf, out=tuple(go))
                iou_host[off:off + m].copy_(iou, non_blocking=True)
                for i in range(4):
                    grad4_host[i, off:off + m].copy_(go[i], non_blocking=True)
            c += 1
        for s in self.streams:
            cur.wait_stream(s)
