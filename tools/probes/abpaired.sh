for r in 1 2; do for v in "$@"; do DGAL_SO=build/ab/libdgal_$v.so python tools/probes/time_paired.py $v; done; done
