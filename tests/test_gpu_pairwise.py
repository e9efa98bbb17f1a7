"""GPU parity of the pairwise IoU matrix, the NMS overlap mask / suppressor lists
and the greedy keep decision (dgal_iou_pairwise, dgal_nms_round, dgal_nms_keep)
against the CPU oracle.  R14: mask bits of pairs with |IoU_oracle - thr| <= 1e-5
are "don't care"; keep parity is oracle_scan(gpu_mask) == gpu_keep, and equals
the oracle's own greedy NMS when no pair lies in that band."""
import numpy as np
import pytest
import torch

import oracle
import paper_2011_11134_b200 as dgal
import synth
from gpu_util import IOU_ATOL, dev, to_dev

pytestmark = pytest.mark.gpu
BAND = 1e-5


def _bits(mask_i64, m):
    """uint64 words [n, w] -> bool [n, m]"""
    w = mask_i64.view(np.uint64)
    b = np.unpackbits(w.view(np.uint8).reshape(w.shape[0], -1), axis=1, bitorder="little")
    return b[:, :m].astype(bool)


def _check_mask(gpu_bits, ref_iou, thr, row_offset=0):
    n, m = ref_iou.shape
    want = ref_iou > thr
    rows = np.arange(n)[:, None] + row_offset
    want &= np.arange(m)[None, :] != rows
    care = np.abs(ref_iou - thr) > BAND
    bad = (gpu_bits != want) & care
    assert not bad.any(), f"{int(bad.sum())} mask bits differ (first {np.argwhere(bad)[:5]})"


def _check_lists(gpu_bits, cnt, idx, row_offset=0):
    n = gpu_bits.shape[0]
    cap = idx.shape[1]
    for r in range(n):
        g = row_offset + r
        want = set(np.nonzero(gpu_bits[r, :g])[0].tolist())
        assert cnt[r] == len(want)
        if cnt[r] <= cap:
            assert set(idx[r, :cnt[r]].tolist()) == want


@pytest.mark.parametrize("indexed", [True, False])
@pytest.mark.parametrize("thr", [0.7, 0.3])
def test_cfg2_full(thr, indexed):
    sc = synth.gen_cfg2_scene()
    p = sc.polys
    x, y = to_dev(p)
    iou, mask, cnt, idx = dgal.iou_pairwise(x, y, x, y, thr=thr, nbr_cap=64, indexed=indexed)
    keep = dgal.nms_keep(mask, cnt, idx)
    torch.cuda.synchronize()
    ref = oracle.iou_pairwise(p, p)
    got = iou.cpu().numpy()
    err = np.abs(got - ref)
    assert err.max() <= IOU_ATOL, err.max()
    assert np.all(np.diag(got) == 1.0)
    bits = _bits(mask.cpu().numpy(), p.n)
    _check_mask(bits, ref, thr)
    _check_lists(bits, cnt.cpu().numpy(), idx.cpu().numpy())
    k = keep.cpu().numpy()
    assert np.array_equal(k, oracle.nms_scan_mask(mask.cpu().numpy().view(np.uint64)))
    if not np.any(np.abs(ref - thr) <= BAND):
        assert np.array_equal(k, oracle.nms_greedy(ref, thr))


def test_pairwise_equals_paired_forward():
    """Row r x column c of the matrix is the paired forward of (r, c): the same
    clip; the paired kernel carries line indices in the 3 low mantissa bits of
    the interval parameters, so the two agree to a few ulp."""
    sc = synth.gen_cfg2_scene(n_objects=10, per_object=30, seed=5)
    p = sc.polys
    x, y = to_dev(p)
    iou, _, _, _ = dgal.iou_pairwise(x, y, x, y, want_mask=False)
    n = p.n
    rng = np.random.default_rng(0)
    ri = rng.integers(0, n, 20000)
    ci = rng.integers(0, n, 20000)
    a, b = p.take(ri), p.take(ci)
    x1, y1 = to_dev(a)
    x2, y2 = to_dev(b)
    pi, _, _ = dgal.iou_paired_fwd(x1, y1, x2, y2)
    torch.cuda.synchronize()
    d = np.abs(iou.cpu().numpy()[ri, ci] - pi.cpu().numpy())
    assert d.max() <= 2e-6, d.max()


@pytest.mark.parametrize("indexed", [True, False])
@pytest.mark.parametrize("nr,m", [(1, 1), (37, 1500), (65, 1031), (200, 2049)])
def test_ragged_shapes_and_row_blocks(nr, m, indexed):
    sc = synth.gen_cfg5_scene(n_objects=max(1, (m + 49) // 50), per_object=50, seed=m)
    cols = sc.polys.take(np.arange(m))
    off = min(3, m - 1)
    rows = cols.take(np.arange(off, min(m, off + nr)))
    nr = rows.n
    rx, ry = to_dev(rows)
    cx, cy = to_dev(cols)
    iou, mask, cnt, idx = dgal.iou_pairwise(rx, ry, cx, cy, row_offset=off, thr=0.1, nbr_cap=8,
                                            indexed=indexed)
    torch.cuda.synchronize()
    ref = oracle.iou_pairwise(rows, cols)
    assert np.abs(iou.cpu().numpy() - ref).max() <= IOU_ATOL
    bits = _bits(mask.cpu().numpy(), m)
    _check_mask(bits, ref, 0.1, row_offset=off)
    _check_lists(bits, cnt.cpu().numpy(), idx.cpu().numpy(), row_offset=off)


@pytest.mark.parametrize("indexed", [True, False])
def test_mask_only_and_k8(indexed):
    b = synth.gen_cfg4_pairs(600, seed=3)
    p = b.p1
    x, y = to_dev(p)
    iou, mask, _, _ = dgal.iou_pairwise(x, y, x, y, thr=0.2, indexed=indexed)
    _, mask2, _, _ = dgal.iou_pairwise(x, y, x, y, thr=0.2, want_iou=False, indexed=indexed)
    torch.cuda.synchronize()
    ref = oracle.iou_pairwise(p, p)
    assert np.abs(iou.cpu().numpy() - ref).max() <= IOU_ATOL
    assert torch.equal(mask, mask2)
    _check_mask(_bits(mask.cpu().numpy(), p.n), ref, 0.2)


def test_nms_rounds_equal_keep_and_overflow_fallback():
    sc = synth.gen_cfg5_scene(n_objects=200, per_object=50, seed=9)
    x, y = to_dev(sc.polys)
    n = sc.polys.n
    _, mask, cnt, idx = dgal.iou_pairwise(x, y, x, y, thr=sc.thr, want_iou=False, nbr_cap=64)
    keep = dgal.nms_keep(mask, cnt, idx)
    # overflowing lists (cap 1) exercise the mask-scan path
    _, mask1, cnt1, idx1 = dgal.iou_pairwise(x, y, x, y, thr=sc.thr, want_iou=False, nbr_cap=1)
    keep1 = dgal.nms_keep(mask1, cnt1, idx1)
    keep0 = dgal.nms_keep(mask)           # no lists at all
    # host-driven rounds over two "row blocks" of one problem
    status = torch.zeros(n, dtype=torch.uint8, device=dev())
    und = torch.zeros(1, dtype=torch.int32, device=dev())
    h = n // 2
    for _ in range(10_000):
        und.zero_()
        dgal.nms_round(n, 0, mask[:h], cnt[:h], idx[:h], status, und)
        dgal.nms_round(n, h, mask[h:], cnt[h:], idx[h:], status, und)
        if int(und.item()) == 0:
            break
    torch.cuda.synchronize()
    k = keep.cpu().numpy()
    assert np.array_equal(k, oracle.nms_scan_mask(mask.cpu().numpy().view(np.uint64)))
    assert np.array_equal(keep1.cpu().numpy(), k) and np.array_equal(keep0.cpu().numpy(), k)
    assert np.array_equal((status == 1).to(torch.uint8).cpu().numpy(), k)
    assert 0 < k.sum() < n
    # rank-local fixed-point rounds (scratch): one block = everything in ONE round; two
    # blocks: the same keep in at most as many rounds as single-pass rounds
    scr = torch.zeros(2, dtype=torch.int32, device=dev())
    st1 = torch.zeros(n, dtype=torch.uint8, device=dev())
    und.zero_()
    dgal.nms_round(n, 0, mask, cnt, idx, st1, und, scr)
    assert int(und.item()) == 0
    assert np.array_equal((st1 == 1).to(torch.uint8).cpu().numpy(), k)
    rounds = {}
    for use in (False, True):
        st2 = torch.zeros(n, dtype=torch.uint8, device=dev())
        for r in range(1, 10_000):
            und.zero_()
            dgal.nms_round(n, 0, mask[:h], cnt[:h], idx[:h], st2, und, scr if use else None)
            dgal.nms_round(n, h, mask[h:], cnt[h:], idx[h:], st2, und, scr if use else None)
            if int(und.item()) == 0:
                break
        rounds[use] = r
        assert np.array_equal((st2 == 1).to(torch.uint8).cpu().numpy(), k)
    assert rounds[True] <= rounds[False]


def test_cfg5_full_size_sampled():
    """100k x 100k at the bench's launch configuration: the full IoU matrix and
    mask on the device; 256 sampled rows checked element by element; the keep
    vector checked against the oracle's greedy scan of the GPU mask."""
    sc = synth.gen_cfg5_scene()
    p = sc.polys
    n = p.n
    x, y = to_dev(p)
    iou, mask, cnt, idx = dgal.iou_pairwise(x, y, x, y, thr=sc.thr, nbr_cap=64)
    keep = dgal.nms_keep(mask, cnt, idx)
    torch.cuda.synchronize()
    rng = np.random.default_rng(5)
    rows = np.sort(rng.choice(n, 256, replace=False))
    got = iou[torch.from_numpy(rows).to(dev())].cpu().numpy()
    ref = oracle.iou_pairwise(p.take(rows), p)
    assert np.abs(got - ref).max() <= IOU_ATOL
    bits = _bits(mask[torch.from_numpy(rows).to(dev())].cpu().numpy(), n)
    want = (ref > sc.thr) & (np.arange(n)[None, :] != rows[:, None])
    care = np.abs(ref - sc.thr) > BAND
    assert not ((bits != want) & care).any()
    diag = iou.diagonal().cpu().numpy()
    assert np.all(diag == 1.0)
    del iou
    k = keep.cpu().numpy()
    assert np.array_equal(k, oracle.nms_scan_mask(mask.cpu().numpy().view(np.uint64)))
    assert 0.05 < k.mean() < 0.9


def test_indexed_and_tiled_paths_agree():
    """The grid-indexed path (zero fill + circle-grid candidates) and the tiled sweep
    give bitwise the same matrix, mask and suppressor sets."""
    sc = synth.gen_cfg5_scene(n_objects=300, per_object=50, seed=17)
    x, y = to_dev(sc.polys)
    n = sc.polys.n
    a = dgal.iou_pairwise(x, y, x, y, thr=sc.thr, nbr_cap=64, indexed=True)
    b = dgal.iou_pairwise(x, y, x, y, thr=sc.thr, nbr_cap=64, indexed=False)
    torch.cuda.synchronize()
    assert torch.equal(a[0], b[0]) and torch.equal(a[1], b[1]) and torch.equal(a[2], b[2])
    ia, ib = a[3].cpu().numpy(), b[3].cpu().numpy()
    c = a[2].cpu().numpy()
    for r in range(n):
        k = min(c[r], 64)
        assert set(ia[r, :k].tolist()) == set(ib[r, :k].tolist())
    # degenerate scene: every box identical (one grid cell holds everything)
    xs = x[:1].repeat(700, 1).contiguous()
    ys = y[:1].repeat(700, 1).contiguous()
    u = dgal.iou_pairwise(xs, ys, xs, ys, thr=0.5, indexed=True)
    v = dgal.iou_pairwise(xs, ys, xs, ys, thr=0.5, indexed=False)
    assert torch.equal(u[0], v[0]) and torch.equal(u[1], v[1])
    assert bool((u[0] == 1.0).all())


@pytest.mark.parametrize("K", [4, 8])
def test_indexed_and_tiled_agree_k4_k8(K):
    """Indexed (persistent warps claiming rows) and tiled paths, K = 4 and K = 8:
    matrix, mask, suppressor counts and sets bitwise equal."""
    sc = synth.gen_cfg5_scene(n_objects=300, per_object=50, seed=23)
    p = sc.polys
    n = p.n
    # K = 8: every box vertex repeated (a zero-length edge: the same polygon, include/dgal.h)
    x = torch.from_numpy(np.repeat(p.x.reshape(n, 4), K // 4, axis=1).copy()).to(dev())
    y = torch.from_numpy(np.repeat(p.y.reshape(n, 4), K // 4, axis=1).copy()).to(dev())
    b = dgal.iou_pairwise(x, y, x, y, thr=sc.thr, nbr_cap=64, indexed=False)
    a = dgal.iou_pairwise(x, y, x, y, thr=sc.thr, nbr_cap=64, indexed=True)
    torch.cuda.synchronize()
    assert torch.equal(a[0], b[0]) and torch.equal(a[1], b[1]) and torch.equal(a[2], b[2])
    ia, ib = a[3].cpu().numpy(), b[3].cpu().numpy()
    c = a[2].cpu().numpy()
    for r in range(n):
        k = min(c[r], 64)
        assert sorted(ia[r, :k].tolist()) == sorted(ib[r, :k].tolist())


def test_keep_grid_equals_single_cta_and_oracle():
    """The grid-wide rounds (cooperative launch) and the single-CTA rounds reach the same
    unique fixed point, which is the oracle's greedy scan of the same mask."""
    sc = synth.gen_cfg5_scene(n_objects=400, per_object=50)
    n = sc.polys.n
    x = torch.from_numpy(sc.polys.x.reshape(n, 4)).to(dev())
    y = torch.from_numpy(sc.polys.y.reshape(n, 4)).to(dev())
    _, mask, cnt, idx = dgal.iou_pairwise(x, y, x, y, thr=sc.thr, want_iou=False, nbr_cap=64)
    kg = dgal.nms_keep(mask, cnt, idx, grid=True)
    kc = dgal.nms_keep(mask, cnt, idx, grid=False)
    kl = dgal.nms_keep(mask, grid=True)                       # mask rows only (no lists)
    torch.cuda.synchronize()
    assert torch.equal(kg, kc) and torch.equal(kg, kl)
    ref = oracle.nms_scan_mask(mask.cpu().numpy().view(np.uint64))
    assert np.array_equal(kg.cpu().numpy(), ref)


@pytest.mark.parametrize("indexed", [True, False])
@pytest.mark.parametrize("nr,m", [(0, 5), (5, 0), (0, 0), (1, 1)])
def test_empty_and_single_shapes(nr, m, indexed):
    """Empty row or column sets (include/dgal.h: n_rows == 0 is a no-op; m == 0
    still zeroes nbr_count) and the 1 x 1 matrix (IoU of a polygon with itself
    is 1, no mask bit on the diagonal); then the keep of the empty / single set."""
    p = synth.gen_cfg5_scene(n_objects=1, per_object=max(nr, m, 1), seed=11).polys
    rows, cols = p.take(np.arange(nr)), p.take(np.arange(m))
    rx, ry = to_dev(rows)
    cx, cy = to_dev(cols)
    K = p.K
    # poison the outputs: whatever the library must write is overwritten
    out = (torch.full((nr, m), -7.0, device=dev()), torch.full((nr, (m + 63) // 64), -1, dtype=torch.int64,
                                                             device=dev()),
           torch.full((nr,), 123, dtype=torch.int32, device=dev()), torch.full((nr, 4), -1, dtype=torch.int32,
                                                                             device=dev()))
    iou, mask, cnt, idx = dgal.iou_pairwise(rx, ry, cx, cy, K=K, thr=0.5, nbr_cap=4, out=out, indexed=indexed)
    torch.cuda.synchronize()
    assert torch.all(cnt == 0)
    if nr and m:
        assert iou.cpu().numpy().tolist() == [[1.0]]
        assert int(mask[0, 0]) == 0
    if nr == m:   # the keep of a square (self) mask
        keep = dgal.nms_keep(mask, cnt, idx)
        torch.cuda.synchronize()
        assert keep.shape == (nr,) and torch.all(keep == 1)


def test_pairwise_nms_sharded_single_rank():
    """dist.pairwise_nms_sharded without a process group (world 1): the whole
    problem is rank 0's row block; its keep equals the single-GPU keep and the
    oracle's greedy scan of the mask, its local IoU the full matrix."""
    from paper_2011_11134_b200.dist import pairwise_nms_sharded
    sc = synth.gen_cfg5_scene(n_objects=60, per_object=50, seed=21)
    p = sc.polys
    x, y = to_dev(p)
    keep, iou, (lo, hi), rounds = pairwise_nms_sharded(x, y, thr=sc.thr, want_iou=True)
    iou1, mask, cnt, idx = dgal.iou_pairwise(x, y, x, y, thr=sc.thr, nbr_cap=64)
    keep1 = dgal.nms_keep(mask, cnt, idx)
    torch.cuda.synchronize()
    assert (lo, hi) == (0, p.n) and rounds >= 1
    assert torch.equal(iou, iou1)
    k = keep.cpu().numpy()
    assert np.array_equal(k, keep1.cpu().numpy())
    assert np.array_equal(k, oracle.nms_scan_mask(mask.cpu().numpy().view(np.uint64)))
    assert 0 < k.sum() < p.n


def test_pairwise_far_from_origin():
    """A nuScenes-like scene shifted to (+4.5 km, -3.2 km) (float32 vertices rounded
    there): the indexed and tiled matrices are bitwise equal and match the oracle on
    the same float polygons (IoU <= 1e-5, mask bits outside the R14 band)."""
    sc = synth.gen_cfg5_scene(n_objects=80, per_object=50, seed=41)
    p = sc.polys
    n = p.n
    xs = (p.x.astype(np.float64) + 4500.0).astype(np.float32)
    ys = (p.y.astype(np.float64) - 3200.0).astype(np.float32)
    q = synth.Polys(xs, ys, 4)
    x, y = to_dev(q)
    a = dgal.iou_pairwise(x, y, x, y, thr=sc.thr, nbr_cap=64, indexed=True)
    b = dgal.iou_pairwise(x, y, x, y, thr=sc.thr, nbr_cap=64, indexed=False)
    torch.cuda.synchronize()
    assert torch.equal(a[0], b[0]) and torch.equal(a[1], b[1]) and torch.equal(a[2], b[2])
    rows = np.sort(np.random.default_rng(3).choice(n, 256, replace=False))
    ref = oracle.iou_pairwise(q.take(rows), q)
    got = a[0][torch.from_numpy(rows).to(dev())].cpu().numpy()
    assert np.abs(got - ref).max() <= IOU_ATOL
    bits = _bits(a[1][torch.from_numpy(rows).to(dev())].cpu().numpy(), n)
    want = (ref > sc.thr) & (np.arange(n)[None, :] != rows[:, None])
    assert not ((bits != want) & (np.abs(ref - sc.thr) > BAND)).any()


@pytest.mark.parametrize("s,o", [(1e-6, 0.0), (1e6, 0.0), (1.0, 2e4), (0.05, 1e4)])
@pytest.mark.parametrize("indexed", [True, False])
def test_pairwise_scale_and_offset_extremes(s, o, indexed):
    """A cfg2-like scene scaled by 1e-6 / 1e6, moved 20 km, or shrunk to 5 % 10 km away
    (float vertices rounded after the transform): the full matrix against the oracle at
    1e-5 on both paths (circle prepass, grid cells and evaluator are all relative)."""
    sc = synth.gen_cfg2_scene(n_objects=20, per_object=25)
    n = sc.polys.n
    x = (sc.polys.x.reshape(n, 4).astype(np.float64) * s + o).astype(np.float32)
    y = (sc.polys.y.reshape(n, 4).astype(np.float64) * s - o).astype(np.float32)
    P = synth.Polys(np.ascontiguousarray(x.reshape(-1)), np.ascontiguousarray(y.reshape(-1)), 4)
    ref = oracle.iou_pairwise(P, P)
    X, Y = torch.from_numpy(x).to(dev()), torch.from_numpy(y).to(dev())
    got = dgal.iou_pairwise(X, Y, X, Y, want_mask=False, indexed=indexed)[0].cpu().numpy()
    assert (ref > 0).sum() > 10 * n
    assert np.abs(got - ref).max() <= 1e-5
