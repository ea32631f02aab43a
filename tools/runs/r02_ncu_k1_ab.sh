# ncu launch durations of K1 for two library builds on the same box
for lib in _ab/a0_head.so _ab/a1_cur.so; do
  PS_B200_LIB=$lib ncu --metrics gpu__time_duration.sum,sm__cycles_elapsed.avg.per_second --clock-control none -k regex:k_preprocess --csv --log-file gpurun_out/k1ab.csv python tools/profile_frame.py --frames 3 > /dev/null 2>&1
  echo "== $lib"; grep -o '"gpu__time_duration.sum","[a-z]*","[0-9.,]*"\|"sm__cycles_elapsed.avg.per_second","[a-z]*","[0-9.,]*"' gpurun_out/k1ab.csv | tail -6
done
for lib in _ab/a0_head.so _ab/a1_cur.so; do echo "== $lib"; PS_B200_LIB=$lib python tools/profile_frame.py --frames 12 | tail -1; done
