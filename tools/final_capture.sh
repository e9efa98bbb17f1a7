#!/bin/bash
# End-of-round GPU capture (one gpurun call): GPU suite (release + checked build), the
# default bench line, the bench's ncu launch list, and an `ncu --set full` summary of
# every hot kernel (tools/prof_run.py --once).  Outputs under gpurun_out/$TAG_*.
TAG=${1:-r02}
mkdir -p gpurun_out
python -m pytest tests -m gpu -q 2>&1 | tail -3 > gpurun_out/${TAG}_gpu_suite.log
DGAL_CHECKED=1 python -m pytest tests -m gpu -q 2>&1 | tail -5 > gpurun_out/${TAG}_checked_build_gpu_suite.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1
python bench.py > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches_bench.csv \
    python bench.py --steps 2 --warmup 3 --no-e2e --no-secondary --no-cpu-baseline > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k "regex:paired_|box_|pw_candidates|pw_zero|nms_keep" \
    -o /tmp/${TAG}_full python tools/prof_run.py --once > gpurun_out/${TAG}_prof_run.log 2>&1
ncu -i /tmp/${TAG}_full.ncu-rep --page raw --csv > gpurun_out/${TAG}_full_raw.csv 2>/dev/null
python tools/ncu_summary.py gpurun_out/${TAG}_full_raw.csv --json gpurun_out/${TAG}_ncu_full_summary.json > gpurun_out/${TAG}_ncu_full_summary.txt
ls -la gpurun_out/${TAG}_*
