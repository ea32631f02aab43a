#!/bin/bash
# compute-sanitizer over tools/sanitize_run.py: memcheck, racecheck
# (shared-memory hazards), synccheck (barrier misuse), initcheck (uninitialised
# device reads). Summaries into gpurun_out/sanitize_*.txt.
cd "$(dirname "$0")/.."
for tool in memcheck racecheck synccheck initcheck; do
  timeout 1200 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize_run.py \
      > gpurun_out/sanitize_$tool.txt 2>&1
  echo "$tool: $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY' gpurun_out/sanitize_$tool.txt | tail -1)"
done
# the per-CTA counter variant of the fused K1 (CTA_RED, > 1.5M splats in the
# product) on the same small workload: a build with the threshold at 0
if [ -f _ab/ctared.so ]; then
  for tool in racecheck synccheck; do
    PS_B200_LIB=_ab/ctared.so timeout 1200 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize_run.py \
        > gpurun_out/sanitize_ctared_$tool.txt 2>&1
    echo "$tool (CTA_RED K1): $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY' gpurun_out/sanitize_ctared_$tool.txt | tail -1)"
  done
fi
