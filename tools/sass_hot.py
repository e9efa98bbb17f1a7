#!/usr/bin/env python
"""Dynamic (ncu source page) instruction counts of one kernel, attributed to CUDA
source lines via the -lineinfo of nvdisasm (the two SASS listings are zipped by
instruction index), split by pipe.  Input: `ncu -i X.ncu-rep --page source --csv
--print-source sass > X.csv`.

    python tools/sass_hot.py gpurun_out/fwd4_src.csv --cubin dgal_paired --kernel 'paired_fwd_direct_kernelILi4'
"""
from __future__ import annotations

import argparse
import collections
import csv
import os
import re
import subprocess
import sys
import tempfile

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from sass_lines import ALU, FMA, INSTR, LINE, SO  # noqa: E402


def main(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("csv")
    ap.add_argument("--so", default=SO)
    ap.add_argument("--cubin", default="dgal_paired")
    ap.add_argument("--kernel", required=True)
    ap.add_argument("--top", type=int, default=45)
    ap.add_argument("--units", type=float, default=0,
                    help="normalise per unit (e.g. warps of 32 pairs) instead of per launched warp")
    ap.add_argument("--block", default=".", help="regex on the ncu 'Kernel Name' row (several kernels in one csv)")
    a = ap.parse_args(argv)
    with tempfile.TemporaryDirectory() as d:
        subprocess.run(["cuobjdump", "-xelf", "all", a.so], cwd=d, capture_output=True, check=True)
        cub = [f for f in os.listdir(d) if f.startswith(a.cubin + ".")][0]
        txt = subprocess.run(["nvdisasm", "-g", "-c", os.path.join(d, cub)], capture_output=True, text=True,
                             check=True).stdout
    seq, cur_k, loc = [], None, None
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
            seq.append((loc, mi.group(1)))
    rows = list(csv.reader(open(a.csv)))
    starts = [i for i, r in enumerate(rows) if r and r[0] == "Kernel Name"] + [len(rows)]
    blk = next(i for i in range(len(starts) - 1) if re.search(a.block, rows[starts[i]][1]))
    rows = rows[starts[blk]:starts[blk + 1]]
    hdr = rows[1]
    ie, ss = hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)")
    data = [r for r in rows[2:] if len(r) > ie]
    if len(data) != len(seq):
        print(f"warning: {len(data)} ncu rows vs {len(seq)} nvdisasm instructions", file=sys.stderr)
    per = collections.defaultdict(collections.Counter)
    tot = collections.Counter()
    for (loc, op), r in zip(seq, data):
        n = int(r[ie]); s = int(r[ss])
        pipe = "alu" if op in ALU else "fma" if op in FMA else "other"
        per[loc][pipe] += n; per[loc]["samples"] += s; per[loc]["op:" + op] += n
        tot[pipe] += n; tot["samples"] += s
    warps = a.units or int(data[0][ie])   # the entry instruction runs once per launched warp
    print(f"warps {warps}; per warp: alu {tot['alu']/warps:.0f} fma {tot['fma']/warps:.0f} other {tot['other']/warps:.0f}"
          f"  (issue {(tot['alu']+tot['fma']+tot['other'])/warps:.0f}, alu-cycles {2*tot['alu']/warps:.0f})")
    for loc, c in sorted(per.items(), key=lambda kv: -kv[1]["samples"])[: a.top]:
        ops = " ".join(f"{k[3:]}:{v/warps:.1f}" for k, v in c.most_common(8) if k.startswith("op:"))
        print(f"{loc:26s} smp {100*c['samples']/tot['samples']:5.1f}% alu {c['alu']/warps:6.1f} fma {c['fma']/warps:6.1f}"
              f" oth {c['other']/warps:5.1f}  {ops}")


if __name__ == "__main__":
    main()
