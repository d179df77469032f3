#!/bin/bash
# trunk-kernel iteration: fwd_small parity tests, stage timeline, C2 bench line
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
: > gpurun_out/summary.txt
timeout 600 python -m pytest tests/test_gpu_fwd_small.py tests/test_gpu_forward.py -q -m gpu -p no:cacheprovider --timeout 300 -x > gpurun_out/tests_small.log 2>&1; echo "tests exit $?" >> gpurun_out/summary.txt
tail -15 gpurun_out/tests_small.log >> gpurun_out/summary.txt
timeout 300 python scripts/small_stages.py > gpurun_out/small_stages.jsonl 2>&1; echo "stages $?" >> gpurun_out/summary.txt
head -1 gpurun_out/small_stages.jsonl >> gpurun_out/summary.txt
grep gemm_task gpurun_out/small_stages.jsonl | head -8 >> gpurun_out/summary.txt
timeout 300 python bench.py --steps 50 --warmup 5 --no-cpu-baseline --no-cpu-latency --no-c4-ref > gpurun_out/bench_c2.log 2>&1; echo "bench exit $?" >> gpurun_out/summary.txt
tail -1 gpurun_out/bench_c2.log | cut -c1-330 >> gpurun_out/summary.txt
cat gpurun_out/summary.txt
