#!/bin/bash
# Full ncu capture of one kernel of a C2 frame + its source/SASS page:
#   tools/ncu_kernel.sh <kernel-regex> <name> [profile_frame args...]
cd "$(dirname "$0")/.."
re=$1; name=$2; shift 2
ncu --set full --clock-control none --import-source on -k regex:"$re" -s 1 -c 1 \
    -o gpurun_out/$name python tools/profile_frame.py --frames 2 "$@" > gpurun_out/$name.log 2>&1
ncu -i gpurun_out/$name.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/${name}_src.csv 2>/dev/null
ncu -i gpurun_out/$name.ncu-rep --page raw --csv > gpurun_out/${name}_raw.csv 2>/dev/null
