#!/bin/bash
# A/B timing of alternative library builds in _ab/*.so (same box, interleaved):
#   tools/ab.sh [profile_frame args]
cd "$(dirname "$0")/.."
for round in 1 2; do
  for lib in _ab/*.so; do
    echo "== $lib (round $round)"
    PS_B200_LIB=$lib python tools/profile_frame.py --frames 12 "$@" | tail -1
  done
done
for round in 1 2; do
  for lib in _ab/*.so; do
    echo "== $lib back-to-back frames, no stage events (round $round)"
    PS_B200_LIB=$lib python tools/host_overhead.py | tail -1
  done
done
for lib in _ab/*.so; do
  echo "== $lib kernels"
  PS_B200_LIB=$lib ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ab_l.csv \
      python tools/profile_frame.py --frames 8 "$@" > /dev/null 2>&1
  python tools/launch_summary.py gpurun_out/ab_l.csv
done
