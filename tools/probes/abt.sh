#!/bin/bash
# A/B timing of build/ab/libdgal_<v>.so variants (time_paired.py, 3 rounds) + bitwise forward
# comparison of each against the first: bash tools/probes/abt.sh TAG v1 v2 ...
tag=$1; shift
mkdir -p gpurun_out
for v in "$@"; do DGAL_SO=build/ab/libdgal_$v.so python tools/probes/cmp_fwd_builds.py /tmp/fwd_$v.npz; done
for v in "${@:2}"; do echo "== $1 vs $v"; python tools/probes/cmp_fwd_npz.py /tmp/fwd_$1.npz /tmp/fwd_$v.npz; done > gpurun_out/${tag}_cmp.log 2>&1
for r in 1 2 3; do for v in "$@"; do DGAL_SO=build/ab/libdgal_$v.so python tools/probes/time_paired.py $v; done; done > gpurun_out/${tag}_time.log 2>&1
