#!/usr/bin/env python
"""Markdown rows of the profiles/README.md kernel table from an ncu summary JSON
(tools/ncu_summary.py --json): time, DRAM bytes, warp-instructions per 32 pairs, issue,
pipes, occupancy, top stalls.   python tools/profiles_table.py profiles/r02_ncu_full_summary.json"""
import json
import sys

L = json.load(open(sys.argv[1]))
byk = {}
for d in L:
    byk.setdefault(d["kernel"].split("(")[0].replace("void ", "").replace("unnamed>::", ""), []).append(d)
U4, U8 = (1 << 24) / 32, (1 << 22) / 32


def stalls(d):
    return ", ".join([x for x in d.get("top_stalls_per_issue", {}) if x != "selected"][:2])


def row(name, size, alg, units, idx=0):
    d = byk[name][idx]
    rw = d["dram_read_GB"] + d["dram_write_GB"]
    return (f"| {name} ({size}) | {d['time_ms']:.3f} ms | {rw:.2f} GB ({alg}) | {d['warp_inst'] / units:.0f} | "
            f"{d['issue_active_pct']:.0f} % | {d.get('alu_pipe_pct', 0):.0f} / {d.get('fma_pipe_pct', 0):.0f} % | "
            f"{d['occupancy_pct']:.0f} % ({d['regs']:.0f}) | {stalls(d)} |")


rows = [row("paired_fwd_direct_kernel<4>", "2^24", "1.29", U4), row("paired_bwd_pt_kernel<4>", "2^24", "2.35", U4),
        row("paired_fused_kernel<4>", "2^24", "2.21", U4)]
r = byk["paired_fused_refine_kernel<4>"][0]
rows.append(f"| paired_fused_refine_kernel<4> | {r['time_ms']:.3f} ms | 3 MB | — | {r['issue_active_pct']:.0f} % | — | "
            f"({r['regs']:.0f}) | long_scoreboard |")
rows += [row("paired_fwd_direct_kernel<8>", "2^22", "0.62", U8), row("paired_bwd_kernel<8>", "2^22", "1.16", U8),
         row("paired_fused_kernel<8>", "2^22", "1.09", U8),
         row("box_fwd_kernel<2>", "2^24", "0.89", U4), row("box_bwd_kernel<2>", "2^24", "1.56", U4),
         row("box_fused_kernel<2>", "2^24", "1.41", U4), row("box_fwd_kernel<3>", "2^24", "1.16", U4),
         row("box_bwd_kernel<3>", "2^24", "2.10", U4), row("box_fused_kernel<3>", "2^24", "1.95", U4)]
z, c, nk = byk["pw_zero"][0], byk["pw_candidates<4>"][0], byk["nms_keep_grid_kernel"][0]
rows.append(f"| pw_zero (40 GB IoU matrix) | {z['time_ms']:.3f} ms | {z['dram_write_GB']:.1f} GB (40.0) | — | "
            f"{z['issue_active_pct']:.0f} % | — | — | drain, mio_throttle (7.6 TB/s) |")
rows.append(f"| pw_candidates<4> (1e5 × 1e5) | {c['time_ms']:.3f} ms | {c['dram_read_GB'] + c['dram_write_GB']:.2f} GB | — | "
            f"{c['issue_active_pct']:.0f} % | {c['alu_pipe_pct']:.0f} / {c['fma_pipe_pct']:.0f} % | "
            f"{c['occupancy_pct']:.0f} % ({c['regs']:.0f}) | wait, long_scoreboard |")
rows.append(f"| nms_keep_grid (1e5 boxes) | {nk['time_ms']:.3f} ms | 3 MB | — | {nk['issue_active_pct']:.0f} % | — | "
            f"cooperative grid | barrier (grid.sync) |")
print("| kernel (size) | time | DRAM R+W (algorithmic) | warp-instr / 32 pairs | issue active | ALU / FMA pipe | "
      "occupancy (regs) | top stalls |")
print("|---|---|---|---|---|---|---|---|")
print("\n".join(rows))
