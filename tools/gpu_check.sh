#!/bin/bash
# quick GPU iteration: parity tests, frame stage times (poly1 + exp), ncu launch list
cd "$(dirname "$0")/.."
python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
python tools/profile_frame.py --frames 5 ${PF_ARGS} > gpurun_out/prof_frame.log 2>&1; tail -1 gpurun_out/prof_frame.log
python tools/profile_frame.py --frames 5 --kernel exp --mode StopThePop > gpurun_out/prof_frame_exp.log 2>&1; tail -1 gpurun_out/prof_frame_exp.log
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python tools/profile_frame.py --frames 8 ${PF_ARGS} > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/launches.csv
