#!/usr/bin/env python
"""Per-kernel SASS statistics of libdgal.so (cuobjdump -sass): instruction count,
opcode histogram, local-memory instructions (LDL/STL must be 0), registers.

    python tools/sass_stats.py [libdgal.so] [--top 20] [--kernel regex]
"""
from __future__ import annotations

import argparse
import collections
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
INSTR = re.compile(r"^\s+/\*[0-9a-f]{4,5}\*/\s+(?:@!?U?P[0-9T]\s+)?([A-Z][A-Z0-9_]*)")


def demangle_short(name: str) -> str:
    m = re.match(r"_ZN4dgal\d+(\w+?)(?:ILi(\d)EE)?E", name)
    if not m:
        return name
    return m.group(1) + (f"<{m.group(2)}>" if m.group(2) else "")


def sass_by_kernel(so: str) -> dict:
    out = subprocess.run(["cuobjdump", "-sass", so], capture_output=True, text=True, check=True).stdout
    kernels, cur = {}, None
    for line in out.splitlines():
        m = re.search(r"Function : (\S+)", line)
        if m:
            cur = m.group(1)
            kernels[cur] = collections.Counter()
            continue
        if cur:
            mi = INSTR.match(line)
            if mi:
                kernels[cur][mi.group(1)] += 1
    return kernels


def main(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("so", nargs="?", default=os.path.join(ROOT, "paper_2011_11134_b200", "libdgal.so"))
    ap.add_argument("--top", type=int, default=16)
    ap.add_argument("--kernel", default=".")
    a = ap.parse_args(argv)
    for name, c in sass_by_kernel(a.so).items():
        if not re.search(a.kernel, name):
            continue
        local = c.get("LDL", 0) + c.get("STL", 0)
        print(f"{demangle_short(name):24s} {sum(c.values()):6d} instr  LDL/STL={local}  " +
              " ".join(f"{k}:{v}" for k, v in c.most_common(a.top)))
    return 0


if __name__ == "__main__":
    sys.exit(main())
