"""Multi-rank GPU paths on one B200 (S:509, S:525 — results bitwise
identical across GPU counts): 2 and 3 ranks under the gloo backend share cuda:0
(the pool lends one GPU; gloo carries the status all-gather through host memory,
the NCCL path differs only in that call, dist.gather_status).  Every rank runs
the real kernels on its shard: the paired shards concatenated and the row-sharded
NMS keep must equal the single-process results bit for bit."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    import torch.distributed as dist

    import synth
    from paper_2011_11134_b200.dist import iou_paired_shard, pairwise_nms_sharded
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    dev = torch.device("cuda:0")
    torch.cuda.set_device(dev)
    n = 100_003   # ragged shards
    b = synth.gen_config(3, n)
    T = lambda a: torch.from_numpy(a.reshape(n, 4)).to(dev)  # noqa: E731
    X = [T(a) for a in (b.p1.x, b.p1.y, b.p2.x, b.p2.y)]
    g = torch.from_numpy(b.grad).to(dev)
    lo, hi, iou, nx, xf, gr = iou_paired_shard(*X, g, world, rank)
    sc = synth.gen_cfg5_scene(n_objects=120, per_object=50, seed=31)
    m = sc.polys.n
    x = torch.from_numpy(sc.polys.x.reshape(m, 4)).to(dev)
    y = torch.from_numpy(sc.polys.y.reshape(m, 4)).to(dev)
    keep, _, _, rounds = pairwise_nms_sharded(x, y, thr=sc.thr)
    torch.cuda.synchronize()
    q.put((rank, lo, hi, iou.cpu().numpy(), xf.cpu().numpy(), [t.cpu().numpy() for t in gr],
           keep.cpu().numpy(), rounds))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_paths_bitwise_equal_single_gpu(world):
    import paper_2011_11134_b200 as dgal
    import synth
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    res = sorted([q.get(timeout=300) for _ in range(world)], key=lambda t: t[0])
    for pr in procs:
        pr.join(timeout=120)
        assert pr.exitcode == 0
    # single process, same inputs
    dev = torch.device("cuda:0")
    n = 100_003
    b = synth.gen_config(3, n)
    T = lambda a: torch.from_numpy(a.reshape(n, 4)).to(dev)  # noqa: E731
    X = [T(a) for a in (b.p1.x, b.p1.y, b.p2.x, b.p2.y)]
    g = torch.from_numpy(b.grad).to(dev)
    iou, nx, xf = dgal.iou_paired_fwd(*X)
    gr = dgal.iou_paired_bwd(*X, g, nx, xf)
    assert [r[1] for r in res] == sorted(r[1] for r in res) and res[0][1] == 0 and res[-1][2] == n
    assert np.array_equal(np.concatenate([r[3] for r in res]), iou.cpu().numpy())
    assert np.array_equal(np.concatenate([r[4] for r in res]), xf.cpu().numpy())
    for k in range(4):
        assert np.array_equal(np.concatenate([r[5][k] for r in res]), gr[k].cpu().numpy())
    sc = synth.gen_cfg5_scene(n_objects=120, per_object=50, seed=31)
    m = sc.polys.n
    x = torch.from_numpy(sc.polys.x.reshape(m, 4)).to(dev)
    y = torch.from_numpy(sc.polys.y.reshape(m, 4)).to(dev)
    _, mask, cnt, idx = dgal.iou_pairwise(x, y, x, y, thr=sc.thr, want_iou=False, nbr_cap=64)
    keep1 = dgal.nms_keep(mask, cnt, idx).cpu().numpy()
    for r in res:
        assert np.array_equal(r[6], keep1), r[0]
    assert len({r[7] for r in res}) == 1
    assert 0 < keep1.sum() < m
