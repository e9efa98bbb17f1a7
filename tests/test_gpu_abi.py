"""The C ABI called raw through ctypes (no Python binding in between): the flag-byte
order the header documents (include/dgal.h, R3), on the S:203 worked example and
the hand-derived cases of tests/golden/canonical_start.json.  Torch only supplies
the device buffers."""
import ctypes
import json
import os

import numpy as np
import pytest
import torch

from paper_2011_11134_b200._lib import lib

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))
GOLD = json.load(open(os.path.join(HERE, "golden", "spec_worked_examples.json")))
CANON = json.load(open(os.path.join(HERE, "golden", "canonical_start.json")))


def _raw_fwd(P_list, Q_list):
    """dgal_iou_paired_fwd(K=4, ...) on raw device pointers; returns (iou, nx, xflags)."""
    dev = torch.device("cuda:0")
    P = np.asarray(P_list, np.float32)
    Q = np.asarray(Q_list, np.float32)
    n = P.shape[0]
    x1, y1, x2, y2 = (torch.from_numpy(np.ascontiguousarray(a)).to(dev)
                      for a in (P[..., 0], P[..., 1], Q[..., 0], Q[..., 1]))
    iou = torch.full((n,), -1.0, device=dev)
    nx = torch.full((n,), 0xEE, dtype=torch.uint8, device=dev)
    xf = torch.full((n, 8), 0xEE, dtype=torch.uint8, device=dev)
    L = lib()
    rc = L.dgal_iou_paired_fwd(ctypes.c_int(4), ctypes.c_int64(n),
                               *(ctypes.c_void_p(t.data_ptr()) for t in (x1, y1, x2, y2, iou, nx, xf)),
                               ctypes.c_void_p(torch.cuda.current_stream(dev).cuda_stream))
    assert rc == 0
    torch.cuda.synchronize()
    return iou.cpu().numpy(), nx.cpu().numpy(), xf.cpu().numpy()


def test_offset_squares_flag_order_through_raw_abi():
    """S:203 offset unit squares: the header's documented sequence C8 42 D3 80
    (Cross(1,0) FromP1(2) Cross(2,3) FromP2(0)), padding 00, IoU 1/7."""
    g = GOLD["offset_squares"]
    iou, nx, xf = _raw_fwd([g["p1"]], [g["p2"]])
    assert nx[0] == 4
    assert list(xf[0]) == [0xC8, 0x42, 0xD3, 0x80, 0, 0, 0, 0]
    assert abs(iou[0] - 1 / 7) < 1e-6


def test_canonical_start_cases_through_raw_abi():
    cases = CANON["cases"]
    iou, nx, xf = _raw_fwd([c["p1"] for c in cases], [c["p2"] for c in cases])
    for k, c in enumerate(cases):
        assert nx[k] == c["nx"], c["name"]
        assert list(xf[k][:c["nx"]]) == c["xflags"], c["name"]
        assert np.all(xf[k][c["nx"]:] == 0), c["name"]
        assert abs(iou[k] - c["iou"][0] / c["iou"][1]) < 2e-6, c["name"]


def test_binding_rejects_mismatched_sizes():
    """The binding checks every buffer against (n, K) before the raw-pointer call
    (the ABI cannot): short planes, wrong-sized out= tensors, wrong dtypes."""
    import paper_2011_11134_b200 as dgal
    dev = torch.device("cuda:0")
    z = lambda *s, dt=torch.float32: torch.zeros(*s, dtype=dt, device=dev)  # noqa: E731
    x = z(16, 4)
    with pytest.raises(ValueError):
        dgal.iou_paired_fwd(x, x, z(15, 4), x)
    with pytest.raises(ValueError):
        dgal.iou_paired_fwd(x, x, x, x, out=(z(16), z(16, dt=torch.uint8), z(16, 4, dt=torch.uint8)))
    with pytest.raises(TypeError):
        dgal.iou_paired_fwd(x, x, x, x, out=(z(16), z(16), z(16, 8, dt=torch.uint8)))
    iou, nx, xf = dgal.iou_paired_fwd(x, x, x, x)
    with pytest.raises(ValueError):
        dgal.iou_paired_bwd(x, x, x, x, z(8), nx, xf)
    with pytest.raises(ValueError):
        dgal.iou_paired_bwd(x, x, x, x, z(16), nx[:8], xf)
    with pytest.raises(ValueError):
        dgal.iou_paired_bwd(x, x, x, x, z(16), nx, xf, out=(x, x, x, z(8, 4)))
    with pytest.raises(ValueError):
        dgal.iou_paired_fused(x, x, x, x, grad=z(4))
    b = z(5, 16)
    with pytest.raises(ValueError):
        dgal.box_iou_paired_bwd(b, b, z(16), nx[:8], z(16, 8, dt=torch.uint8))
    with pytest.raises(ValueError):
        dgal.iou_pairwise(x, x, x, x, out=(z(16, 15), None, None, None))
    with pytest.raises(ValueError):
        dgal.nms_keep(z(16, 2, dt=torch.int64))


@pytest.mark.parametrize("K", [4, 8])
@pytest.mark.parametrize("pinned", [True, False])
@pytest.mark.parametrize("n,chunk", [(7 * 4096 + 17, 4096), (1000, 4096), (1, 4)])
def test_host_buffer_call_equals_device_calls(K, pinned, n, chunk):
    """dgal_iou_paired_host (host buffers in and out, chunked three-stream
    pipeline inside the library): iou and the four gradient planes bitwise equal
    to dgal_iou_paired_fwd + dgal_iou_paired_bwd on device copies of the same
    inputs — ragged last chunk, slots reused across chunks, pinned and pageable."""
    import paper_2011_11134_b200 as dgal
    import synth
    b = synth.gen_config(3 if K == 4 else 4, n)
    dev = torch.device("cuda:0")
    host = [torch.from_numpy(a.reshape(n, K).copy()) for a in (b.p1.x, b.p1.y, b.p2.x, b.p2.y)]
    g = torch.from_numpy(np.random.default_rng(n).uniform(-1, 1, n).astype(np.float32))
    if pinned:
        host = [t.pin_memory() for t in host]
        g = g.pin_memory()
    out = dgal.iou_paired_host(*host, g, chunk=chunk, device=dev)
    torch.cuda.synchronize()
    d = [t.to(dev) for t in host]
    iou, nx, xf = dgal.iou_paired_fwd(*d)
    gr = dgal.iou_paired_bwd(*d, g.to(dev), nx, xf)
    torch.cuda.synchronize()
    assert torch.equal(out[0], iou.cpu())
    for a, c in zip(out[1:], gr):
        assert torch.equal(a, c.cpu())
