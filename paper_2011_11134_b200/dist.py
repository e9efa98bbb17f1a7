"""Multi-GPU sharding of the hot path: one process per GPU, torch.distributed
(NCCL over NVLink/NVSwitch) for the plumbing.

* Paired IoU (training loss): pairs are independent and write disjoint slots
  (S:525), so every rank owns the contiguous pair range
  shard_range(n, world, rank) and NO collective touches the data path.
* Pairwise IoU + rotated NMS: rank r owns the row block shard_range(n, world, r)
  against all n columns (its IoU rows, NMS mask rows and suppressor lists stay
  local).  The greedy keep decision runs as parallel rounds (include/dgal.h
  dgal_nms_round): each rank updates the status of its own boxes from the
  global status vector, then the ranks all-gather their status slices — n
  bytes per round (100 KB at n = 1e5) instead of the 1.25 GB mask.  Rounds stop
  when no box is undecided; every rank ends with the identical keep vector,
  bitwise equal to the single-GPU result.
"""
from __future__ import annotations

from typing import Callable, Optional

import torch
import torch.distributed as dist


def shard_range(n: int, world: int, rank: int, block: Optional[int] = None):
    """Contiguous shard [lo, hi) of rank `rank`; blocks of ceil(n/world) (last short)."""
    b = block if block is not None else -(-n // world)
    lo = min(n, rank * b)
    return lo, min(n, lo + b)


def iou_paired_shard(x1, y1, x2, y2, grad, world: int, rank: int):
    """Forward + backward of this rank's contiguous pair shard (no collective).
    Returns (lo, hi, iou, nx, xflags, (gx1, gy1, gx2, gy2)) for rows [lo, hi)."""
    from . import iou_paired_bwd, iou_paired_fwd
    n = x1.shape[0]
    lo, hi = shard_range(n, world, rank)
    s = slice(lo, hi)
    a = [t[s].contiguous() for t in (x1, y1, x2, y2)]
    iou, nx, xf = iou_paired_fwd(*a)
    g = iou_paired_bwd(*a, grad[s].contiguous(), nx, xf)
    return lo, hi, iou, nx, xf, g


iou_paired_sharded = iou_paired_shard   # SURVEY §8(b) name


def _backend(group=None) -> str:
    return dist.get_backend(group) if dist.is_initialized() else "none"


def gather_status(status: torch.Tensor, B: int, group=None) -> None:
    """All-gather every rank's slice status[r*B:(r+1)*B] into every rank's copy, in
    place (NCCL: all_gather_into_tensor on the device, enqueued on the current
    stream, no host sync; gloo: through host memory — the CPU test / shared-GPU
    path)."""
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    mine = status[rank * B:(rank + 1) * B].clone()
    if _backend(group) == "nccl":
        dist.all_gather_into_tensor(status, mine, group=group)
        return
    parts = [torch.empty_like(mine, device="cpu") for _ in range(world)]
    dist.all_gather(parts, mine.cpu(), group=group)
    status.copy_(torch.cat(parts).to(status.device))


def nms_rounds(n: int, lo: int, hi: int, round_fn: Callable[[torch.Tensor], None],
               status: torch.Tensor, group=None, max_rounds: Optional[int] = None,
               check_every: int = 8) -> int:
    """Run NMS rounds to convergence.

    status: this rank's copy of the padded global status vector, uint8
            [world * B] with B = ceil(n / world), zero-initialised;
    round_fn(status): updates status[lo:hi] (this rank's boxes) in place from
            the whole vector (dgal_nms_round on the GPU).
    After every round the ranks all-gather their slices, so all copies agree.
    The host checks for convergence after rounds 1, 2, 4, ... (doubling) and then
    every `check_every` rounds (one device -> host read of "any box undecided" per
    check, not per round: rounds after convergence change nothing, so over-running
    is harmless; with rank-local fixed-point rounds a few rounds suffice).  Every
    rank reads the same gathered vector, so all take the same decision.
    Returns the number of rounds run (a check point, or fewer at the limit).
    """
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    B = status.numel() // world
    assert status.numel() == world * B and lo == min(n, rank * B)
    limit = max_rounds if max_rounds is not None else n + 1
    r, nxt = 0, 1
    while r < limit:
        while r < min(nxt, limit):
            round_fn(status)
            if world > 1:
                gather_status(status, B, group)
            r += 1
        if not bool((status[:n] == 0).any()):
            return r
        nxt = r + min(r, check_every)
    raise RuntimeError("NMS rounds did not converge")  # impossible: >= 1 box decides per round


def pairwise_nms_sharded(x, y, thr: float = 0.7, nbr_cap: int = 64, want_iou: bool = False,
                         group=None):
    """Rotated NMS of n score-sorted polygons (x, y: [n, K] CUDA tensors, same on
    every rank), row-sharded over the ranks of `group`.  Returns
    (keep u8[n] — identical on every rank, local_iou [hi-lo, n] | None, (lo, hi), rounds)."""
    from . import iou_pairwise, nms_round
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    n = x.shape[0]
    B = -(-n // world)
    lo, hi = shard_range(n, world, rank, B)
    rx, ry = x[lo:hi].contiguous(), y[lo:hi].contiguous()
    iou, mask, cnt, idx = iou_pairwise(rx, ry, x, y, row_offset=lo, thr=thr, want_iou=want_iou,
                                       want_mask=True, nbr_cap=nbr_cap, indexed=True)
    status = torch.zeros(world * B, dtype=torch.uint8, device=x.device)
    undecided = torch.zeros(1, dtype=torch.int32, device=x.device)
    scratch = torch.zeros(2, dtype=torch.int32, device=x.device)   # rank-local fixed-point rounds

    def round_fn(st):
        if hi > lo:
            nms_round(n, lo, mask, cnt, idx, st, undecided, scratch)

    rounds = nms_rounds(n, lo, hi, round_fn, status, group=group)
    keep = (status[:n] == 1).to(torch.uint8)
    return keep, iou, (lo, hi), rounds
