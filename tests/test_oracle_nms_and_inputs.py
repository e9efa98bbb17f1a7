"""T0 (CPU): NMS oracle pinned by exhaustive characterisation; pairwise oracle
pinned by the paired oracle; generator and margin-filter properties."""
import itertools

import numpy as np
import pytest

import oracle
import synth
from helpers import margin_filter


def _greedy_fixed_point(iou, thr):
    """Exhaustive: the greedy-NMS keep set is the UNIQUE subset S with
    (a) no i in S is suppressed by an earlier j in S, and
    (b) every i not in S is suppressed by an earlier j in S."""
    n = iou.shape[0]
    sols = []
    for bits in range(1 << n):
        S = [(bits >> i) & 1 for i in range(n)]
        ok = True
        for i in range(n):
            sup = any(S[j] and iou[j, i] > thr for j in range(i))
            if S[i] and sup or (not S[i] and not sup):
                ok = False
                break
        if ok:
            sols.append(S)
    assert len(sols) == 1
    return np.array(sols[0], np.uint8)


@pytest.mark.parametrize("seed", range(6))
def test_nms_greedy_matches_characterisation(seed):
    sc = synth.gen_cfg2_scene(n_objects=2, per_object=5, seed=seed)
    p = sc.polys
    m = oracle.iou_pairwise(p, p)
    for thr in (0.1, 0.3, 0.5, 0.7):
        keep = oracle.nms_greedy(m, thr)
        assert np.array_equal(keep, _greedy_fixed_point(m, thr))
        # the mask scan (R14) on the mask built from the same matrix agrees
        n = m.shape[0]
        words = (n + 63) // 64
        mask = np.zeros((n, words), np.uint64)
        for i in range(n):
            for j in range(i + 1, n):
                if m[i, j] > thr:
                    mask[i, j >> 6] |= np.uint64(1) << np.uint64(j & 63)
        assert np.array_equal(oracle.nms_scan_mask(mask), keep)


def test_pairwise_equals_paired():
    sc = synth.gen_cfg2_scene(n_objects=4, per_object=10, seed=11)
    p = sc.polys
    m = oracle.iou_pairwise(p, p)
    n = p.n
    ii, jj = np.meshgrid(np.arange(n), np.arange(n), indexing="ij")
    f = oracle.iou_paired_fwd(p.take(ii.ravel()), p.take(jj.ravel()))
    assert np.array_equal(m.ravel(), f["iou"])
    assert np.all(np.diag(m) == 1.0)
    ri = np.array([0, 3, 7, 39])
    ci = np.array([5, 3, 0, 1])
    assert np.array_equal(oracle.iou_pairs_indexed(p, p, ri, ci), m[ri, ci])


# ---------------------------------------------------------------------------
# generators
# ---------------------------------------------------------------------------
def _convex_ccw(p):
    x, y = p.xy64()
    ex, ey = np.roll(x, -1, 1) - x, np.roll(y, -1, 1) - y
    cr = ex * np.roll(ey, -1, 1) - ey * np.roll(ex, -1, 1)
    return np.all(cr > 0)


@pytest.mark.parametrize("cfg", [1, 2, 3, 4, 5])
def test_generators_valid_and_deterministic(cfg):
    n = {1: 1024, 2: 2000, 3: 20000, 4: 20000, 5: 20000}[cfg]
    a = synth.gen_config(cfg, n)
    b = synth.gen_config(cfg, n)
    if cfg in (2, 5):
        assert np.array_equal(a.polys.x, b.polys.x) and _convex_ccw(a.polys)
        assert np.all(np.diff(a.scores) <= 0)
        assert a.polys.x.dtype == np.float32
    else:
        assert np.array_equal(a.p1.x, b.p1.x) and np.array_equal(a.p2.y, b.p2.y)
        assert _convex_ccw(a.p1) and _convex_ccw(a.p2)
        assert a.p1.x.dtype == np.float32 and a.n == n


def test_quad_generator_valid():
    """General convex quads (tests' walk-state workload) are convex, CCW, float32."""
    a, b = synth.gen_quad_pairs(20000), synth.gen_quad_pairs(20000)
    assert np.array_equal(a.p1.x, b.p1.x) and _convex_ccw(a.p1) and _convex_ccw(a.p2)
    assert a.p1.K == 4 and a.p1.x.dtype == np.float32


def test_generators_prefix_stable():
    a = synth.gen_cfg3_pairs(70000)
    b = synth.gen_cfg3_pairs(1000)
    assert np.array_equal(a.p1.x[: 4 * 1000], b.p1.x)
    assert np.array_equal(a.grad[:1000], b.grad)


def test_workload_statistics():
    """>= 20% of SPEC-generator pairs overlap; the KITTI paired batch is
    mostly overlapping (~97%); octagon pairs reach nx = 16."""
    f = oracle.iou_paired_fwd(*(lambda b: (b.p1, b.p2))(synth.gen_cfg1_pairs(1000, seed=42)))
    assert (f["iou"] > 0).mean() >= 0.2
    b = synth.gen_cfg3_pairs(4000)
    f = oracle.iou_paired_fwd(b.p1, b.p2)
    assert (f["iou"] > 0).mean() > 0.9
    b = synth.gen_cfg4_pairs(4000)
    f = oracle.iou_paired_fwd(b.p1, b.p2)
    assert f["nx"].max() == 16


@pytest.mark.parametrize("cfg,maxrej", [(1, 0.06), (3, 0.15), (4, 0.2)])
def test_margin_filter_rates(cfg, maxrej):
    b = synth.gen_config(cfg, 4000)
    ok = oracle.margin_ok(b.p1, b.p2)
    assert 1 - ok.mean() < maxrej
    f = margin_filter(b, 1000)
    assert f.n == 1000
