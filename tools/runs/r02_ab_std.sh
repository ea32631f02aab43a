# GPU tests with the product build, then A/B of _ab/*.so at C2 poly1, C3, C2 exp / StopThePop, C5
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/gputest.log 2>&1; echo rc=$?; tail -3 gpurun_out/gputest.log
tools/ab_quick.sh 2>&1 | grep -v "^{"
tools/ab_quick.sh --workload c3 2>&1 | grep -v "^{"
tools/ab_quick.sh --kernel exp --mode StopThePop 2>&1 | grep -v "^{"
tools/ab_quick.sh --workload c5 2>&1 | grep -v "^{"
