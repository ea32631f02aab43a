#!/bin/bash
# Round-end GPU evidence: parity suite, smoke, the bench lines (C2 default, C3-C5,
# the reference arm) and the profile collection, all into gpurun_out/.
cd "$(dirname "$0")/.."
python -m pytest tests -m gpu -q > gpurun_out/final_tests.log 2>&1
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke.log 2>&1
python bench.py > gpurun_out/bench.log 2>&1
python bench.py --workload c3 > gpurun_out/bench_c3.log 2>&1
python bench.py --workload c4 > gpurun_out/bench_c4.log 2>&1
python bench.py --workload c5 > gpurun_out/bench_c5.log 2>&1
python bench.py --impl reference > gpurun_out/bench_ref.log 2>&1
bash tools/collect_profiles.sh
