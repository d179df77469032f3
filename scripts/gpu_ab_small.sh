#!/bin/bash
# trunk-kernel variant check: fwd_small GPU tests, then A/B of env variants on C2, stage timeline
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_fwd_small.py -q -m gpu -p no:cacheprovider --timeout 300 -x > gpurun_out/tests_small.log 2>&1; echo "tests $?"
tail -3 gpurun_out/tests_small.log
ROUNDS=${ROUNDS:-3} WL=c2 bash scripts/ab_bench.sh "$@" 2>&1 | tee gpurun_out/ab_small.txt
timeout 300 python scripts/small_stages.py > gpurun_out/small_stages.jsonl 2>&1; echo "stages $?"
head -1 gpurun_out/small_stages.jsonl
