"""Build libdgal variants for A/B timing: python tools/probes/ab_build.py NAME -DMACRO=V ...
-> build/ab/libdgal_NAME.so (same sources and flags as build.py plus the macros)."""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from paper_2011_11134_b200 import build as b  # noqa: E402

name, macros = sys.argv[1], sys.argv[2:]
out = os.path.join(ROOT, "build", "ab", f"libdgal_{name}.so")
os.makedirs(os.path.dirname(out), exist_ok=True)
r = subprocess.run(["nvcc", *b.NVCC_FLAGS, *macros, "-o", out, *b.sources()], capture_output=True, text=True)
if r.returncode:
    sys.exit(r.stderr)
regs = [l for l in r.stderr.splitlines() if "registers" in l]
print(out)
