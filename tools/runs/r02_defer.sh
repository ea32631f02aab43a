# deferred fp64 tight tiers (K1u): GPU tests, then A/B vs the committed build at C2, exp, C3
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gputest.log 2>&1; echo rc=$?; tail -5 gpurun_out/gputest.log
tools/ab_quick.sh 2>&1 | grep -v "^{"
tools/ab_quick.sh --workload c3 2>&1 | grep -v "^{"
tools/ab_quick.sh --kernel exp --mode StopThePop 2>&1 | grep -v "^{"
