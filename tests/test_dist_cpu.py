"""Multi-process (gloo, world_size 2 and 3, CPU) tests of the sharding logic of
paper_2011_11134_b200/dist.py: shard ranges, and the NMS round protocol with its
status all-gather.  The per-round box update here is a test-local CPU stand-in
driven by the oracle's IoU matrix (the product path uses dgal_nms_round on the
GPU); what is tested is the protocol: sharding, the all-gather, termination,
and that every rank ends with the single-process greedy keep vector."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
import synth
from paper_2011_11134_b200.dist import nms_rounds, shard_range


def test_shard_ranges_partition():
    for n in (0, 1, 7, 100, 1 << 24, 100_000):
        for world in (1, 2, 3, 4, 8):
            rs = [shard_range(n, world, r) for r in range(world)]
            covered = []
            for lo, hi in rs:
                assert 0 <= lo <= hi <= n
                covered.extend(range(lo, hi)) if n < 10_000 else None
            assert rs[0][0] == 0 and rs[-1][1] == n or n == 0
            for (a, b), (c, d) in zip(rs, rs[1:]):
                assert b == c or (b == n and c == n)
            if n < 10_000:
                assert covered == list(range(n))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, lower, n, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    B = -(-n // world)
    lo, hi = shard_range(n, world, rank, B)
    status = torch.zeros(world * B, dtype=torch.uint8)

    def round_fn(st):
        snap = st.clone()          # decisions from the gathered vector (like one kernel)
        for i in range(lo, hi):
            if snap[i] != 0:
                continue
            s = snap[lower[i]] if len(lower[i]) else torch.empty(0, dtype=torch.uint8)
            if bool((s == 1).any()):
                st[i] = 2
            elif bool((s == 2).all()):
                st[i] = 1

    rounds = nms_rounds(n, lo, hi, round_fn, status)
    out_q.put((rank, (status[:n] == 1).numpy().astype(np.uint8).tobytes(), rounds))
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_nms_round_protocol_gloo(world):
    sc = synth.gen_cfg2_scene(n_objects=6, per_object=30, seed=21)
    p = sc.polys
    n = p.n
    m = oracle.iou_pairwise(p, p)
    lower = [np.nonzero(m[i, :i] > sc.thr)[0].tolist() for i in range(n)]
    want = oracle.nms_greedy(m, sc.thr)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, lower, n, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    keeps = {r: np.frombuffer(b, np.uint8) for r, b, _ in res}
    for r in range(world):
        assert np.array_equal(keeps[r], want), r
    assert len({rounds for _, _, rounds in res}) == 1
