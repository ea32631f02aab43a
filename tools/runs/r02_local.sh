timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gputest3.log 2>&1; echo rc=$?; tail -3 gpurun_out/gputest3.log
tools/ab_quick.sh 2>&1 | grep -v "^{"; tools/ab_quick.sh --kernel exp --mode StopThePop 2>&1 | grep -v "^{"
for k in "poly1 OpacityAware" "exp StopThePop" "poly3 OpacityAware" "poly2p OpacityAware"; do set -- $k; python tools/profile_frame.py --frames 2 --kernel $1 --mode $2 | head -1 | cut -c1-90; done
