#!/usr/bin/env python
"""Static SASS instructions in the main (tile) loop of one kernel: the span between the
target of the kernel's longest backward branch and that branch.  For the issue-bound
paired kernels this is ~ the dynamic warp-instructions per 32 pairs (ncu), so an A/B
of a source change can be read here, on the CPU, before it goes to the GPU.

    python tools/loop_count.py [--so build/ab/libdgal_X.so] [--cubin dgal_paired] \
        --kernel 'paired_fwd_direct_kernelILi4' [--mix]
"""
from __future__ import annotations

import argparse
import collections
import os
import re
import subprocess
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SO = os.path.join(ROOT, "paper_2011_11134_b200", "libdgal.so")
INS = re.compile(r"^\s+/\*([0-9a-f]{4,5})\*/\s+(@!?U?P[0-9T]\s+)?([A-Z][A-Z0-9_.]*)([^;]*);")


def kernel_sass(so: str, cubin: str, kernel: str) -> list[tuple[int, str, str]]:
    if so.endswith(".cubin"):   # nvcc -cubin of one source (fast A/B)
        txt = subprocess.run(["cuobjdump", "-sass", so], capture_output=True, text=True, check=True).stdout
    else:
        with tempfile.TemporaryDirectory() as d:
            subprocess.run(["cuobjdump", "-xelf", "all", so], cwd=d, capture_output=True, check=True)
            cub = [f for f in os.listdir(d) if f.startswith(cubin + ".")][0]
            txt = subprocess.run(["cuobjdump", "-sass", os.path.join(d, cub)], capture_output=True, text=True,
                                 check=True).stdout
    out, on = [], False
    for line in txt.splitlines():
        if "Function :" in line:
            on = kernel in line
            continue
        if on:
            m = INS.match(line)
            if m:
                out.append((int(m.group(1), 16), m.group(3), m.group(4)))
    return out


def main(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--so", default=SO)
    ap.add_argument("--cubin", default="dgal_paired")
    ap.add_argument("--kernel", required=True)
    ap.add_argument("--mix", action="store_true")
    ap.add_argument("--contains", default="LDGSTS",
                    help="only loops whose body holds this opcode (the tile loop's prefetch); '' for any")
    a = ap.parse_args(argv)
    ins = kernel_sass(a.so, a.cubin, a.kernel)
    best = None
    for off, op, rest in ins:
        if op == "BRA" or op.startswith("BRA."):
            m = re.search(r"0x([0-9a-f]+)", rest)
            if m:
                tgt = int(m.group(1), 16)
                has = not a.contains or any(o2 == a.contains or o2.startswith(a.contains + ".")
                                            for o3, o2, _ in ins if tgt <= o3 <= off)
                if tgt < off and has and (best is None or off - tgt > best[1] - best[0]):
                    best = (tgt, off)
    if best is None:
        print(f"{a.kernel}: total {len(ins)}, no backward branch")
        return
    lo, hi = best
    body = [op for off, op, _ in ins if lo <= off <= hi]
    print(f"{a.kernel}: total {len(ins)}, loop [{lo:#x}, {hi:#x}] {len(body)} instructions")
    if a.mix:
        for op, c in collections.Counter(body).most_common(40):
            print(f"  {c:4d} {op}")


if __name__ == "__main__":
    main()
