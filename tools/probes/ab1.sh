mkdir -p gpurun_out
python -m pytest tests -m gpu -q -x 2>&1 | tail -3 > gpurun_out/ab1_suite.log
for v in base new; do DGAL_SO=build/ab/libdgal_$v.so python tools/probes/cmp_fwd_builds.py /tmp/fwd_$v.npz; done
python tools/probes/cmp_fwd_npz.py /tmp/fwd_base.npz /tmp/fwd_new.npz > gpurun_out/ab1_cmp.log 2>&1
python - >> gpurun_out/ab1_cmp.log 2>&1 <<'PY'
import numpy as np
a,b=np.load('/tmp/fwd_base.npz'),np.load('/tmp/fwd_new.npz')
d=np.abs(a['iou'].astype(np.float64)-b['iou'])
print('iou max diff', d.max(), 'n>1e-6', (d>1e-6).sum(), 'n>0', (d>0).sum())
PY
for r in 1 2 3; do for v in base new; do DGAL_SO=build/ab/libdgal_$v.so python tools/probes/time_paired.py $v; done; done > gpurun_out/ab1_time.log 2>&1
