#!/bin/bash
# compute-sanitizer passes over every hand-rolled device protocol (scripts/sanitize_cases.py)
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
: > gpurun_out/summary.txt
for tool in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 20 --error-exitcode 9 python scripts/sanitize_cases.py > gpurun_out/sanitizer_$tool.log 2>&1; echo "sanitizer $tool exit $?" >> gpurun_out/summary.txt
  tail -3 gpurun_out/sanitizer_$tool.log >> gpurun_out/summary.txt
done
cat gpurun_out/summary.txt
