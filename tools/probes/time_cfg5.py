"""cfg5 (100k x 100k pairwise + NMS) through bench.bench_cfg5 with the loaded libdgal
(DGAL_SO selects a build): python tools/probes/time_cfg5.py [label]."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path[:0] = [ROOT]
import bench  # noqa: E402

label = sys.argv[1] if len(sys.argv) > 1 else os.environ.get("DGAL_SO", "libdgal.so")
ctx = bench.Ctx(1, 0, 0)
r = bench.bench_cfg5(ctx, steps=10, warmup=2, peak=6552.3)
print(label, {k: r[k] for k in ("ms_matrix", "ms_matrix_plus_nms", "kept")}, flush=True)
