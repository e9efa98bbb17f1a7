"""Helpers for the -m gpu parity tests: move synth batches to the device, run the
C-ABI path, fetch results, and compare with the oracle at the north_star
tolerances (IoU <= 1e-5 abs; gradients <= 1e-4 abs OR <= 1e-3 rel; nx/xflags
bit-exact on margin inputs)."""
from __future__ import annotations

import numpy as np
import torch

import oracle
import paper_2011_11134_b200 as dgal

IOU_ATOL = 1e-5
GRAD_ATOL = 1e-4
GRAD_RTOL = 1e-3


def dev():
    return torch.device("cuda:0")


def to_dev(p):
    """synth.Polys -> (x, y) [n, K] float32 CUDA tensors."""
    K = p.K
    return (torch.from_numpy(p.x.reshape(-1, K)).to(dev()),
            torch.from_numpy(p.y.reshape(-1, K)).to(dev()))


def gpu_paired(b, grad=None):
    x1, y1 = to_dev(b.p1)
    x2, y2 = to_dev(b.p2)
    iou, nx, xf = dgal.iou_paired_fwd(x1, y1, x2, y2)
    g = torch.from_numpy(b.grad if grad is None else grad).to(dev())
    gr = dgal.iou_paired_bwd(x1, y1, x2, y2, g, nx, xf)
    torch.cuda.synchronize()
    return (iou.cpu().numpy(), nx.cpu().numpy(), xf.cpu().numpy(),
            tuple(t.cpu().numpy() for t in gr))


def assert_iou_close(got, want, atol=IOU_ATOL):
    err = np.abs(got.astype(np.float64) - want)
    assert err.max() <= atol, f"max IoU error {err.max():.3e} at {int(err.argmax())}"


def assert_grad_close(got, want):
    got = got.astype(np.float64)
    err = np.abs(got - want)
    bad = (err > GRAD_ATOL) & (err > GRAD_RTOL * np.abs(want))
    assert not bad.any(), f"{int(bad.sum())} gradient entries out of tolerance, worst {err.max():.3e}"


def assert_flags_exact(nx, xf, ref):
    bad = np.nonzero(nx != ref["nx"])[0]
    assert bad.size == 0, f"nx differs at {bad[:10]}: gpu {nx[bad[:5]]} oracle {ref['nx'][bad[:5]]}"
    badf = np.nonzero(np.any(xf != ref["xflags"], axis=1))[0]
    assert badf.size == 0, (f"xflags differ at {badf[:10]}: gpu {[list(map(hex, xf[k])) for k in badf[:3]]} "
                            f"oracle {[list(map(hex, ref['xflags'][k])) for k in badf[:3]]}")


def check_paired_against_oracle(b, flags=True, grads=True):
    iou, nx, xf, gr = gpu_paired(b)
    ref = oracle.iou_paired_fwd(b.p1, b.p2)
    assert_iou_close(iou, ref["iou"])
    if flags:
        assert_flags_exact(nx, xf, ref)
    if grads:
        rg = oracle.iou_paired_bwd(b.p1, b.p2, b.grad)
        for got, want in zip(gr, rg):
            assert_grad_close(got.reshape(want.shape), want)
    return iou, nx, xf, gr, ref
