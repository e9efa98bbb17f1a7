"""cfg2 (2000 x 2000 pairwise + mask + lists + keep) through bench.bench_cfg2 with the loaded
libdgal (DGAL_SO selects a build): eager and CUDA-graph ms per step."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path[:0] = [ROOT]
import bench  # noqa: E402

label = sys.argv[1] if len(sys.argv) > 1 else os.environ.get("DGAL_SO", "libdgal.so")
ctx = bench.Ctx(1, 0, 0)
r = bench.bench_cfg2(ctx, steps=200, warmup=10)
print(label, {k: r[k] for k in ("ms_per_step", "cuda_graph_ms_per_step", "kept")}, flush=True)
