"""In-tree build of libdgal.so (nvcc, sm_100a).  Used by __graft_entry__.build()
and the Makefile; the built .so travels to the GPU box with the repo snapshot."""
from __future__ import annotations

import glob
import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
SO = os.path.join(HERE, "libdgal.so")
CSRC = os.path.join(HERE, "csrc")
HEADER = os.path.join(ROOT, "include", "dgal.h")

NVCC_FLAGS = [
    "-O3", "-std=c++17",
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-lineinfo",
    "-Xcompiler", "-fPIC", "-shared",
    "-Xptxas", "-v",
]


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")))


def _stale(so: str = SO) -> bool:
    if not os.path.exists(so):
        return True
    t = os.path.getmtime(so)
    deps = sources() + glob.glob(os.path.join(CSRC, "*.cuh")) + glob.glob(os.path.join(CSRC, "*.h")) + [HEADER]
    return any(os.path.getmtime(d) > t for d in deps)


SO_CHECKED = os.path.join(HERE, "libdgal_checked.so")


def build(force: bool = False, verbose: bool = False, checked: bool = False) -> str:
    """Release library (or, checked=True, libdgal_checked.so with device-side
    bounds asserts: -DDGAL_CHECKED, selected at load time by DGAL_CHECKED=1)."""
    out = SO_CHECKED if checked else SO
    if not (force or _stale(out)):
        return out
    nvcc = os.environ.get("NVCC", "nvcc")
    extra = ["-DDGAL_CHECKED"] if checked else []
    cmd = [nvcc, *NVCC_FLAGS, *extra, "-o", out + ".tmp", *sources()]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError("nvcc failed:\n" + r.stdout + r.stderr)
    if verbose:
        print(r.stderr)
    os.replace(out + ".tmp", out)
    if not checked:
        with open(os.path.join(HERE, "ptxas_report.txt"), "w") as f:
            f.write(r.stderr)
    return out


if __name__ == "__main__":
    import sys
    build(force=True, verbose=True, checked="--checked" in sys.argv)
