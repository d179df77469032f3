#!/bin/bash
# quick check: GPU kernel + forward tests, C2 and C4 bench (no CPU baseline)
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
: > gpurun_out/summary.txt
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_forward.py ${EXTRA_TESTS} -q -m gpu -p no:cacheprovider --timeout 300 -rf -x > gpurun_out/tests_quick.log 2>&1; echo "tests exit $?" >> gpurun_out/summary.txt
timeout 600 python bench.py --steps 100 --warmup 10 --no-cpu-baseline > gpurun_out/bench_c2.log 2>&1; echo "bench c2 exit $?" >> gpurun_out/summary.txt
timeout 600 python bench.py --workload c4 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_c4.log 2>&1; echo "bench c4 exit $?" >> gpurun_out/summary.txt
for s in ${SCRIPTS}; do timeout 600 python $s > gpurun_out/$(basename $s .py).jsonl 2>&1; echo "$s exit $?" >> gpurun_out/summary.txt; done
cat gpurun_out/summary.txt
