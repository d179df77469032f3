#!/bin/bash
# Round-2 session c: baseline of HEAD on a fresh box -- GPU suite, default bench line, trunk stage timeline
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
: > gpurun_out/summary.txt
timeout 1200 python -m pytest tests -q -m gpu -p no:cacheprovider --timeout 600 -x > gpurun_out/tests_c.log 2>&1; echo "tests exit $?" >> gpurun_out/summary.txt
tail -3 gpurun_out/tests_c.log >> gpurun_out/summary.txt
timeout 600 python bench.py --steps 50 --warmup 5 > gpurun_out/bench_c2_c.log 2>&1; echo "bench exit $?" >> gpurun_out/summary.txt
tail -1 gpurun_out/bench_c2_c.log | cut -c1-400 >> gpurun_out/summary.txt
timeout 300 python scripts/small_stages.py > gpurun_out/small_stages_c.jsonl 2>&1; echo "stages $?" >> gpurun_out/summary.txt
head -1 gpurun_out/small_stages_c.jsonl >> gpurun_out/summary.txt
cat gpurun_out/summary.txt
