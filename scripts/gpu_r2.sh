#!/bin/bash
# Round-2 GPU session: new parity bars + concurrency tests (report -> gpurun_out/parity_report.jsonl),
# the whole GPU suite, smoke, the default bench line and the reference arm.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
: > gpurun_out/summary.txt
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > gpurun_out/gpu.txt 2>&1
nproc >> gpurun_out/gpu.txt
export PRLAB_PARITY_REPORT=$PWD/gpurun_out/parity_report.jsonl
: > $PRLAB_PARITY_REPORT
timeout 1200 python -m pytest tests/test_gpu_parity_bars.py tests/test_gpu_concurrency.py -q -m gpu -p no:cacheprovider --timeout 900 -rf > gpurun_out/tests_new.log 2>&1; echo "new tests exit $?" >> gpurun_out/summary.txt
if [ -z "$SKIP_SUITE" ]; then
timeout 1500 python -m pytest tests -q -m gpu -p no:cacheprovider --timeout 900 -rf --deselect tests/test_gpu_parity_bars.py --deselect tests/test_gpu_concurrency.py > gpurun_out/tests_gpu.log 2>&1; echo "suite exit $?" >> gpurun_out/summary.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke exit $?" >> gpurun_out/summary.txt
fi
timeout 900 python bench.py ${BENCH_ARGS} > gpurun_out/bench_c2.log 2>&1; echo "bench exit $?" >> gpurun_out/summary.txt
if [ -z "$SKIP_REF" ]; then
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.log 2>&1; echo "bench ref exit $?" >> gpurun_out/summary.txt
fi
cat gpurun_out/summary.txt
