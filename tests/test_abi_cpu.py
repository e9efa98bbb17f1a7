"""CPU-only checks of the C-ABI boundary (no GPU needed): libdgal.so loads, exports
every function include/dgal.h declares, validates arguments on the host before
touching the device, and its kernels are sm_100a SASS with no local memory
(register-resident clip state)."""
import ctypes
import os
import re
import subprocess

import pytest

import paper_2011_11134_b200 as dgal
from paper_2011_11134_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "dgal.h")


def _declared():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(dgal_[a-z_]+)\s*\(", src)))


def test_header_declares_the_boundary():
    names = _declared()
    assert names == sorted(["dgal_iou_paired_fwd", "dgal_iou_paired_bwd", "dgal_iou_paired_fused",
                            "dgal_box_iou_paired_fwd", "dgal_box_iou_paired_bwd", "dgal_box_iou_paired_fused",
                            "dgal_iou_pairwise", "dgal_fused_workspace_bytes", "dgal_iou_paired_host",
                            "dgal_paired_host_workspace_bytes",
                            "dgal_pairwise_workspace_bytes", "dgal_nms_round", "dgal_nms_keep",
                            "dgal_status_string", "dgal_build_info"])


def test_library_exports_every_declared_symbol():
    L = dgal.lib()
    for name in _declared():
        assert hasattr(L, name), name
        assert name in _lib.SIGNATURES
    out = subprocess.run(["nm", "-D", "--defined-only", _lib.SO_PATH], capture_output=True,
                         text=True, check=True).stdout
    exported = set(re.findall(r"\bT (dgal_\w+)", out))
    assert set(_declared()) <= exported


def test_status_strings_and_build_info():
    L = dgal.lib()
    assert L.dgal_status_string(0) == b"DGAL_OK"
    assert L.dgal_status_string(3) == b"DGAL_ERR_MISALIGNED"
    assert L.dgal_status_string(99) == b"DGAL_ERR_UNKNOWN"
    assert b"sm_100a" in L.dgal_build_info()


def test_host_side_validation_without_gpu():
    """Errors are returned before anything is enqueued (no CUDA call happens)."""
    L = dgal.lib()
    buf = ctypes.create_string_buffer(4096 + 16)
    a = (ctypes.addressof(buf) + 15) & ~15           # 16-byte aligned host address
    P = ctypes.c_void_p
    # unsupported K
    assert L.dgal_iou_paired_fwd(5, 8, P(a), P(a), P(a), P(a), P(a), P(a), P(a), None) == 2
    # negative n, NULL pointers
    assert L.dgal_iou_paired_fwd(4, -1, P(a), P(a), P(a), P(a), P(a), P(a), P(a), None) == 1
    assert L.dgal_iou_paired_fwd(4, 8, None, P(a), P(a), P(a), P(a), P(a), P(a), None) == 1
    # misaligned plane
    assert L.dgal_iou_paired_fwd(4, 8, P(a + 4), P(a), P(a), P(a), P(a), P(a), P(a), None) == 3
    # misaligned xflags for K=8 (needs 16 B)
    assert L.dgal_iou_paired_fwd(8, 8, P(a), P(a), P(a), P(a), P(a), P(a), P(a + 8), None) == 3
    # fused: misaligned dL/dIoU or IoU output (4 B), misaligned gradient plane (16 B),
    # refine workspace missing / too small / misaligned
    ws = L.dgal_fused_workspace_bytes(8)
    assert ws == 48 and L.dgal_fused_workspace_bytes(1 << 24) == 16 + 4 * (1 << 24)
    assert L.dgal_fused_workspace_bytes(5) == 48        # 16 + 20 -> 48 (16-byte multiple)
    F1 = ctypes.c_float(1.0)
    assert L.dgal_iou_paired_fused(4, 8, P(a), P(a), P(a), P(a), P(a + 2), F1, None,
                                   P(a), P(a), P(a), P(a), P(a), ws, None) == 3
    assert L.dgal_iou_paired_fused(4, 8, P(a), P(a), P(a), P(a), None, F1, P(a + 1),
                                   P(a), P(a), P(a), P(a), P(a), ws, None) == 3
    assert L.dgal_iou_paired_fused(8, 8, P(a), P(a), P(a), P(a), None, F1, None,
                                   P(a), P(a + 8), P(a), P(a), P(a), ws, None) == 3
    assert L.dgal_iou_paired_fused(4, 8, P(a), P(a), P(a), P(a), None, F1, None,
                                   P(a), P(a), P(a), P(a), None, ws, None) == 1
    assert L.dgal_iou_paired_fused(4, 8, P(a), P(a), P(a), P(a), None, F1, None,
                                   P(a), P(a), P(a), P(a), P(a), ws - 1, None) == 1
    assert L.dgal_iou_paired_fused(4, 8, P(a), P(a), P(a), P(a), None, F1, None,
                                   P(a), P(a), P(a), P(a), P(a + 4), ws, None) == 3
    # host-buffer call: workspace size (3 slots), bad K / chunk, NULL, short or misaligned workspace
    hw = L.dgal_paired_host_workspace_bytes(4, 1024)
    assert hw == 3 * (8 * 16384 + 2 * 4096 + 1024 + 8192)
    assert L.dgal_paired_host_workspace_bytes(8, 1024) == 3 * (8 * 32768 + 2 * 4096 + 1024 + 16384)
    assert L.dgal_paired_host_workspace_bytes(5, 1024) == 0 and L.dgal_paired_host_workspace_bytes(4, 0) == 0
    W = 1 << 20   # any 256-aligned address: validation rejects these before any CUDA call
    h = [P(a)] * 10
    assert L.dgal_iou_paired_host(6, 8, *h, 1024, P(W), hw, None) == 2
    assert L.dgal_iou_paired_host(4, 8, *h, 1022, P(W), hw, None) == 1         # chunk % 4
    assert L.dgal_iou_paired_host(4, 8, *h, 0, P(W), hw, None) == 1
    assert L.dgal_iou_paired_host(4, -1, *h, 1024, P(W), hw, None) == 1
    assert L.dgal_iou_paired_host(4, 8, *([P(a)] * 9), None, 1024, P(W), hw, None) == 1
    assert L.dgal_iou_paired_host(4, 8, *h, 1024, None, hw, None) == 1
    assert L.dgal_iou_paired_host(4, 8, *h, 1024, P(W), hw - 1, None) == 1
    assert L.dgal_iou_paired_host(4, 8, *h, 1024, P(W + 128), hw, None) == 3
    assert L.dgal_iou_paired_host(4, 0, *([None] * 10), 1024, None, 0, None) == 0
    # n == 0 is a no-op
    assert L.dgal_iou_paired_fwd(4, 0, None, None, None, None, None, None, None, None) == 0
    assert L.dgal_iou_paired_bwd(4, 0, *([None] * 11), None) == 0
    # boxes: bad dims / layout, NULL, misaligned, n == 0
    assert L.dgal_box_iou_paired_fwd(4, 0, 8, P(a), P(a), P(a), P(a), P(a), None) == 1
    assert L.dgal_box_iou_paired_fwd(2, 2, 8, P(a), P(a), P(a), P(a), P(a), None) == 1
    assert L.dgal_box_iou_paired_fwd(2, 0, 8, None, P(a), P(a), P(a), P(a), None) == 1
    assert L.dgal_box_iou_paired_fwd(3, 1, 8, P(a + 2), P(a), P(a), P(a), P(a), None) == 3
    assert L.dgal_box_iou_paired_fwd(2, 0, 8, P(a), P(a), P(a), P(a), P(a + 4), None) == 3
    assert L.dgal_box_iou_paired_fwd(2, 0, 0, None, None, None, None, None, None) == 0
    assert L.dgal_box_iou_paired_bwd(3, 0, 8, P(a), P(a), None, P(a), P(a), P(a), P(a), None) == 1
    assert L.dgal_box_iou_paired_fused(2, 0, 8, P(a), P(a), None, 1.0, None, None, P(a), P(a), 48, None) == 1
    assert L.dgal_box_iou_paired_fused(2, 0, 8, P(a), P(a), None, 1.0, None, P(a), P(a), None, 48, None) == 1
    assert L.dgal_box_iou_paired_fused(2, 0, 8, P(a), P(a), None, 1.0, None, P(a), P(a), P(a), 47, None) == 1
    assert L.dgal_box_iou_paired_fused(2, 0, 8, P(a), P(a), None, 1.0, None, P(a), P(a), P(a + 4), 48, None) == 3
    # pairwise: nothing requested, negative threshold with a mask, short mask rows
    args = [4, 8, P(a), P(a), 8, P(a), P(a), 0]
    assert L.dgal_iou_pairwise(*args, None, 0.5, None, 0, None, None, 0, None, 0, None) == 1
    assert L.dgal_iou_pairwise(*args, None, -0.1, P(a), 1, None, None, 0, None, 0, None) == 1
    assert L.dgal_iou_pairwise(*[4, 8, P(a), P(a), 200, P(a), P(a), 0], None, 0.5, P(a), 1, None, None,
                               0, None, 0, None) == 1
    # lists without a mask; a workspace that is too small
    assert L.dgal_iou_pairwise(*args, P(a), 0.5, None, 0, P(a), P(a), 4, None, 0, None) == 1
    assert L.dgal_iou_pairwise(*args, P(a), 0.5, None, 0, None, None, 0, P(a), 16, None) == 1
    assert L.dgal_pairwise_workspace_bytes(100_000) > 100_000 * 24
    # no columns: a no-op without lists, half-given lists rejected (with lists it zeroes nbr_count: GPU test)
    assert L.dgal_iou_pairwise(*[4, 8, None, None, 0, None, None, 0], None, 0.5, None, 0, None, None, 0, None, 0,
                               None) == 0
    assert L.dgal_iou_pairwise(*[4, 8, None, None, 0, None, None, 0], None, 0.5, None, 0, P(a), None, 0, None, 0,
                               None) == 1
    # NMS: row block outside the problem
    assert L.dgal_nms_round(10, 8, 4, P(a), 1, None, None, 0, P(a), P(a), None, None) == 1
    assert L.dgal_nms_round(10, 8, 0, P(a), 1, None, None, 0, P(a), P(a), P(a + 2), None) == 3
    assert L.dgal_nms_keep(0, None, 0, None, None, 0, None, None, None, None) == 0
    assert L.dgal_nms_keep(100, P(a), 1, None, None, 0, P(a), P(a), None, None) == 1
    assert L.dgal_nms_keep(10, P(a), 1, None, None, 0, P(a), P(a), P(a + 2), None) == 3


def test_python_binding_rejects_cpu_tensors():
    import torch
    x = torch.zeros((4, 4))
    with pytest.raises(TypeError):
        dgal.iou_paired_fwd(x, x, x, x)


def _sass_stats():
    import sys
    sys.path.insert(0, os.path.join(ROOT, "tools"))
    import sass_stats
    return sass_stats.sass_by_kernel(_lib.SO_PATH)


def test_sass_is_sm100a_register_resident():
    """Every kernel is compiled to sm_100a SASS; no LDL/STL (local memory) anywhere:
    the fixed-capacity polygons, clip intervals and flag bytes live in registers."""
    out = subprocess.run(["cuobjdump", "-lelf", _lib.SO_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    stats = _sass_stats()
    names = " ".join(stats)
    for k in ("paired_fwd_direct_kernelILi4", "paired_fwd_direct_kernelILi8", "paired_bwd_kernelILi4",
              "paired_fused_kernelILi4", "paired_fused_kernelILi8",
              "paired_bwd_kernelILi8", "pairwise_kernelILi4", "nms_keep_kernel", "nms_round_kernel", "nms_keep_grid_kernel", "nms_round_grid_kernel",
              "box_fwd_kernelILi2", "box_fwd_kernelILi3", "box_bwd_kernelILi2", "box_bwd_kernelILi3",
              "box_fused_kernelILi2", "box_fused_kernelILi3"):
        assert k in names, k
    for name, c in stats.items():
        assert c.get("LDL", 0) == 0 and c.get("STL", 0) == 0, (name, c.get("LDL"), c.get("STL"))
