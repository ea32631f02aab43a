#!/bin/bash
# Quick A/B of _ab/*.so variants: median stage times (profile_frame, stage events),
# two interleaved rounds:  tools/ab_quick.sh [profile_frame args]
cd "$(dirname "$0")/.."
for round in 1 2; do
  for lib in _ab/*.so; do
    echo "== $lib (round $round) $*"
    PS_B200_LIB=$lib python tools/profile_frame.py --frames 12 "$@" | tail -1
  done
done
