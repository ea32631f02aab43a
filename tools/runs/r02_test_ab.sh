# GPU tests, then A/B of the _ab/*.so variants at C2 (poly1 / exp), stage medians
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gputest.log 2>&1; echo rc=$?; tail -3 gpurun_out/gputest.log
bash tools/runs/r02_ab.sh
