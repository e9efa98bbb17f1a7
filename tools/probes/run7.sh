python -m pytest tests -m gpu -q -x 2>&1 | tail -4 > gpurun_out/ab7_suite.log
bash tools/probes/abt.sh ab7 prev dup
python tools/probes/time_box.py > gpurun_out/ab7_box.log 2>&1
DGAL_SO=build/ab/libdgal_prev.so python tools/probes/time_box.py >> gpurun_out/ab7_box.log 2>&1
