#!/bin/bash
# Collects the round's profiling evidence into gpurun_out/prof_*:
#   launch lists of one C2 frame (ncu gpu__time_duration, cold, serialised) for
#   poly1 and exp, a full ncu capture of the blend / preprocess / duplicate
#   kernels (raw + details pages), the blend's per-source-line counters and
#   their region summary, the SASS evidence, and the measured peaks.
cd "$(dirname "$0")/.."
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/prof_launches_c2.csv \
    python tools/profile_frame.py --frames 3 > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/prof_launches_c2_exp.csv \
    python tools/profile_frame.py --frames 3 --kernel exp --mode StopThePop > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:"blend16|k_geometry|k_shade|k_preprocess|k_dup" -s 3 -c 3 \
    -o gpurun_out/prof_full_c2 python tools/profile_frame.py --frames 3 > /dev/null 2>&1
ncu -i gpurun_out/prof_full_c2.ncu-rep --page details --csv > gpurun_out/prof_full_c2_details.csv 2>/dev/null
ncu -i gpurun_out/prof_full_c2.ncu-rep --page raw --csv > gpurun_out/prof_full_c2_raw.csv 2>/dev/null
bash tools/ncu_kernel.sh blend16 prof_blend_src > /dev/null 2>&1
python tools/src_regions.py gpurun_out/prof_blend_src_src.csv > gpurun_out/prof_blend_regions.txt 2>&1
python tools/src_report.py gpurun_out/prof_blend_src_src.csv 40 >> gpurun_out/prof_blend_regions.txt 2>&1
python tools/sass_report.py > gpurun_out/prof_sass_blend16.txt 2>&1
python tools/peaks.py > gpurun_out/prof_peaks.txt 2>&1
