#!/usr/bin/env python
"""Summarise an ncu --set full report (raw page CSV): per kernel launch, the
metrics the DESIGN.md roofline discussion uses.  Usage:
    ncu -i rep.ncu-rep --page raw --csv > raw.csv; python tools/ncu_summary.py raw.csv [--json out.json]"""
import csv
import json
import sys

METRICS = [
    ("time_ms", "gpu__time_duration.sum"),
    ("dram_read_GB", "dram__bytes_read.sum"),
    ("dram_write_GB", "dram__bytes_write.sum"),
    ("dram_pct_peak", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"),
    ("regs", "launch__registers_per_thread"),
    ("occupancy_pct", "sm__warps_active.avg.pct_of_peak_sustained_active"),
    ("issue_active_pct", "smsp__issue_active.avg.pct_of_peak_sustained_active"),
    ("warp_inst", "smsp__inst_executed.sum"),
    ("threads_per_inst", "smsp__thread_inst_executed_per_inst_executed.ratio"),
    ("fma_pipe_pct", "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active"),
    ("alu_pipe_pct", "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active"),
    ("xu_pipe_pct", "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active"),
    ("lsu_pipe_pct", "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active"),
    ("local_ld_bytes", "l1tex__t_bytes_pipe_lsu_mem_local_op_ld.sum"),
    ("local_st_bytes", "l1tex__t_bytes_pipe_lsu_mem_local_op_st.sum"),
    # --set full on ncu 2025.2 carries sectors (32 B) rather than bytes for local memory
    ("local_ld_sectors", "l1tex__t_sectors_pipe_lsu_mem_local_op_ld.sum"),
    ("local_st_sectors", "l1tex__t_sectors_pipe_lsu_mem_local_op_st.sum"),
]


def main(argv):
    rows = list(csv.reader(open(argv[1])))
    hdr, units = rows[0], rows[1]
    idx = {k: hdr.index(m) for k, m in METRICS if m in hdr}
    stall = [(h, i) for i, h in enumerate(hdr) if h.startswith("smsp__average_warps_issue_stalled_")
             and h.endswith("_per_issue_active.ratio")]
    out = []
    for r in rows[2:]:
        d = {"kernel": r[hdr.index("Kernel Name")]}
        for k, i in idx.items():
            try:
                v = float(r[i].replace(",", ""))
            except ValueError:
                v = r[i]
            if k.endswith("_GB") and units[i] == "Gbyte":
                pass
            elif k.endswith("_GB") and units[i] == "Mbyte":
                v = v / 1e3
            d[k] = v
        st = sorted(((float(r[i] or 0), h.replace("smsp__average_warps_issue_stalled_", "")
                      .replace("_per_issue_active.ratio", "")) for h, i in stall), reverse=True)[:6]
        d["top_stalls_per_issue"] = {n: round(v, 3) for v, n in st}
        out.append(d)
    for d in out:
        print(json.dumps(d))
    if "--json" in argv:
        json.dump(out, open(argv[argv.index("--json") + 1], "w"), indent=1)


if __name__ == "__main__":
    main(sys.argv)
