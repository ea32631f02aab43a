# K1 ablations at C2 (poly1): stage medians, three interleaved rounds
for round in 1 2 3; do for lib in _ab/*.so; do echo "== $lib (round $round)"; PS_B200_LIB=$lib python tools/profile_frame.py --frames 12 | tail -1; done; done
