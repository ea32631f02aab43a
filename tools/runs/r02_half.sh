# half-tile blend: smoke with a timeout first (deadlock guard), then GPU tests and A/B
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" || { echo SMOKE-FAILED; exit 1; }
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gputest.log 2>&1; echo rc=$?; tail -3 gpurun_out/gputest.log
timeout 600 bash tools/runs/r02_ab.sh
for w in c3 c4 c5; do timeout 300 tools/ab_quick.sh --workload $w 2>&1 | grep -v "^{"; done
