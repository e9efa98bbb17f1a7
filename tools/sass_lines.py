#!/usr/bin/env python
"""Static SASS instructions of one kernel attributed to source lines (-lineinfo),
split by pipe (alu = IADD3/LOP3/SHF/FMNMX/FSETP/ISETP/SEL/..., fma = FADD/FMUL/FFMA/
IMAD/HFMA2, other).  The K=4 forward is bound by the ALU pipe (half rate), so
this is the map of where its ALU work comes from.

    python tools/sass_lines.py --cubin dgal_paired --kernel 'paired_fwd_direct_kernelILi4' [--top 40]
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
FMA = {"FADD", "FMUL", "FFMA", "IMAD", "HFMA2", "FMUL2", "FADD2", "FFMA2", "IMUL", "HADD2", "HMUL2"}
ALU = {"IADD3", "LOP3", "SHF", "FMNMX", "FMNMX3", "FSETP", "ISETP", "SEL", "FSEL", "PLOP3", "LEA", "LEA.HI",
       "PRMT", "IABS", "IMNMX", "VIADD", "VIMNMX", "FLO", "BREV", "POPC", "P2R", "R2P", "FCHK", "ISCADD", "MOV",
       "IADD", "FSWZADD", "VIADDMNMX"}
INSTR = re.compile(r"^\s+/\*[0-9a-f]{4,5}\*/\s+(?:@!?U?P[0-9T]\s+)?([A-Z][A-Z0-9_]*)")
LINE = re.compile(r'//## File "([^"]+)", line (\d+)')


def main(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--so", default=SO)
    ap.add_argument("--cubin", default="dgal_paired")
    ap.add_argument("--kernel", required=True)
    ap.add_argument("--top", type=int, default=40)
    a = ap.parse_args(argv)
    with tempfile.TemporaryDirectory() as d:
        subprocess.run(["cuobjdump", "-xelf", "all", a.so], cwd=d, capture_output=True, check=True)
        cub = [f for f in os.listdir(d) if f.startswith(a.cubin + ".")][0]
        txt = subprocess.run(["nvdisasm", "-g", "-c", os.path.join(d, cub)], capture_output=True, text=True,
                             check=True).stdout
    cur_k, loc = None, None
    per = collections.defaultdict(lambda: collections.Counter())
    tot = collections.Counter()
    for ln in txt.splitlines():
        if ln.startswith("//-----") and ".text." in ln:
            cur_k = ln.split(".text.")[1].split()[0]
            continue
        if not cur_k or not re.search(a.kernel, cur_k):
            continue
        m = LINE.search(ln)
        if m:
            loc = f"{os.path.basename(m.group(1))}:{m.group(2)}"
            continue
        mi = INSTR.match(ln)
        if mi:
            op = mi.group(1)
            pipe = "alu" if op in ALU else "fma" if op in FMA else "other"
            per[loc][pipe] += 1
            per[loc]["op:" + op] += 1
            tot[pipe] += 1
    print(f"total: {dict(tot)}")
    rows = sorted(per.items(), key=lambda kv: -(2 * kv[1]["alu"] + kv[1]["fma"]))
    for loc, c in rows[: a.top]:
        ops = " ".join(f"{k[3:]}:{v}" for k, v in c.most_common() if k.startswith("op:"))
        print(f"{loc:28s} alu {c['alu']:4d} fma {c['fma']:4d} other {c['other']:3d}  {ops}")


if __name__ == "__main__":
    main()
