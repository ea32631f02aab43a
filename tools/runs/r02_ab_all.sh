# GPU tests, then A/B of the _ab/*.so variants at C2 (poly1, exp), C3, C4 (one view), C5
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gputest.log 2>&1; echo rc=$?; tail -3 gpurun_out/gputest.log
tools/ab_quick.sh 2>&1 | grep -v "^{"; tools/ab_quick.sh --kernel exp --mode StopThePop 2>&1 | grep -v "^{"
for w in c3 c4 c5; do tools/ab_quick.sh --workload $w 2>&1 | grep -v "^{"; done
