"""ctypes loader of libdgal.so (include/dgal.h).  No fallback of any kind: if the
library is missing or a call fails, this raises."""
from __future__ import annotations

import ctypes
import os

HERE = os.path.dirname(os.path.abspath(__file__))
# DGAL_CHECKED=1 selects the bounds-checked build (device asserts), see build.py
SO_PATH = os.path.join(HERE, "libdgal_checked.so" if os.environ.get("DGAL_CHECKED") == "1" else "libdgal.so")
# DGAL_SO=<path>: load another build of the same library (A/B timing of build
# variants, tools/probes/); it must be a libdgal build, there is no other path.
SO_PATH = os.environ.get("DGAL_SO", SO_PATH)

_P = ctypes.c_void_p
_I64 = ctypes.c_int64
_I32 = ctypes.c_int32
_INT = ctypes.c_int
_F = ctypes.c_float

#: every exported symbol of include/dgal.h with its ctypes signature
SIGNATURES = {
    "dgal_iou_paired_fwd": (_INT, [_INT, _I64, _P, _P, _P, _P, _P, _P, _P, _P]),
    "dgal_iou_paired_bwd": (_INT, [_INT, _I64, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P]),
    "dgal_iou_paired_fused": (_INT, [_INT, _I64, _P, _P, _P, _P, _P, _F, _P, _P, _P, _P, _P, _P,
                                     ctypes.c_size_t, _P]),
    "dgal_fused_workspace_bytes": (ctypes.c_size_t, [_I64]),
    "dgal_iou_paired_host": (_INT, [_INT, _I64, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _I64, _P,
                                    ctypes.c_size_t, _P]),
    "dgal_paired_host_workspace_bytes": (ctypes.c_size_t, [_INT, _I64]),
    "dgal_box_iou_paired_fwd": (_INT, [_INT, _INT, _I64, _P, _P, _P, _P, _P, _P]),
    "dgal_box_iou_paired_bwd": (_INT, [_INT, _INT, _I64, _P, _P, _P, _P, _P, _P, _P, _P]),
    "dgal_box_iou_paired_fused": (_INT, [_INT, _INT, _I64, _P, _P, _P, _F, _P, _P, _P, _P, ctypes.c_size_t, _P]),
    "dgal_iou_pairwise": (_INT, [_INT, _I64, _P, _P, _I64, _P, _P, _I64, _P, _F, _P, _I64, _P, _P,
                                 _I32, _P, ctypes.c_size_t, _P]),
    "dgal_pairwise_workspace_bytes": (ctypes.c_size_t, [_I64]),
    "dgal_nms_round": (_INT, [_I64, _I64, _I64, _P, _I64, _P, _P, _I32, _P, _P, _P, _P]),
    "dgal_nms_keep": (_INT, [_I64, _P, _I64, _P, _P, _I32, _P, _P, _P, _P]),
    "dgal_status_string": (ctypes.c_char_p, [_INT]),
    "dgal_build_info": (ctypes.c_char_p, []),
}

STATUS = {0: "DGAL_OK", 1: "DGAL_ERR_INVALID_ARG", 2: "DGAL_ERR_UNSUPPORTED_K",
          3: "DGAL_ERR_MISALIGNED", 4: "DGAL_ERR_CUDA"}


class DgalError(RuntimeError):
    def __init__(self, fn: str, code: int):
        super().__init__(f"{fn} failed: {STATUS.get(code, code)}")
        self.code = code


_lib = None


def lib() -> ctypes.CDLL:
    """Load libdgal.so (built in-tree by __graft_entry__.build()).  Raises if absent."""
    global _lib
    if _lib is None:
        if not os.path.exists(SO_PATH):
            raise ImportError(f"{SO_PATH} is not built: run `python -c 'import __graft_entry__ as g; "
                              f"g.build()'` (nvcc, sm_100a). There is no fallback path.")
        L = ctypes.CDLL(SO_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def call(name: str, *args) -> None:
    rc = getattr(lib(), name)(*args)
    if rc != 0:
        raise DgalError(name, rc)
