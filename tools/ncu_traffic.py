#!/usr/bin/env python
"""profiles/ncu_traffic.json (read by bench.py as roofline.traffic) from the
per-launch summary of an `ncu --set full` capture of tools/prof_run.py --once
(tools/ncu_summary.py --json): dram__bytes_read.sum + dram__bytes_write.sum of
each hot kernel's launch.

    python tools/ncu_traffic.py gpurun_out/full_summary.json > profiles/ncu_traffic.json
"""
import json
import re
import sys

KEYS = [  # (key, kernel regex); first match in launch order (the second pw_zero is the mask fill)
    ("paired_fwd_k4", r"paired_fwd_direct_kernel<4>"), ("paired_bwd_k4", r"paired_bwd(_pt)?_kernel<4>"),
    ("paired_fused_k4", r"paired_fused_kernel<4>"), ("paired_fwd_k8", r"paired_fwd_direct_kernel<8>"),
    ("paired_bwd_k8", r"paired_bwd_kernel<8>"), ("paired_fused_k8", r"paired_fused_kernel<8>"),
    ("box_fwd_d2", r"box_fwd_kernel<2>"), ("box_bwd_d2", r"box_bwd_kernel<2>"), ("box_fused_d2", r"box_fused_kernel<2>"),
    ("box_fwd_d3", r"box_fwd_kernel<3>"), ("box_bwd_d3", r"box_bwd_kernel<3>"), ("box_fused_d3", r"box_fused_kernel<3>"),
    ("pw_zero_iou", r"pw_zero"), ("pw_candidates_k4", r"pw_candidates<4>"), ("nms_keep", r"nms_keep"),
    ("paired_fused_refine_k4", r"paired_fused_refine_kernel<4>"), ("box_fused_refine_d2", r"box_fused_refine_kernel<2>"),
]


def main(path):
    launches = json.load(open(path))
    out = {}
    for key, rx in KEYS:
        d = next((d for d in launches if re.search(rx, d["kernel"])), None)
        if d is not None:
            out[f"{key}_bytes_per_launch"] = int(round((d["dram_read_GB"] + d["dram_write_GB"]) * 1e9, -3))
    out["source"] = (f"{sys.argv[2] if len(sys.argv) > 2 else path} (ncu --set full --clock-control none, "
                     "tools/prof_run.py --once, B200)")
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main(sys.argv[1])
