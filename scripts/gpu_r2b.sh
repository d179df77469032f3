#!/bin/bash
# Round-2 GPU session b: full_fp16 fast path tests + ablation, memory report, parity bars,
# the tests that exercise full_fp16 / GEMMs, C4 bench, compute-sanitizer passes.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
: > gpurun_out/summary.txt
export PRLAB_PARITY_REPORT=$PWD/gpurun_out/parity_report_b.jsonl
: > $PRLAB_PARITY_REPORT
timeout 1500 python -m pytest tests/test_gpu_fp16_fast.py tests/test_gpu_parity_bars.py tests/test_gpu_sweep.py tests/test_gpu_forward.py tests/test_gpu_kernels.py tests/test_gpu_concurrency.py -q -m gpu -p no:cacheprovider --timeout 900 -rf > gpurun_out/tests_b.log 2>&1; echo "tests exit $?" >> gpurun_out/summary.txt
timeout 900 python scripts/ablation.py > gpurun_out/ablation_c5.jsonl 2> gpurun_out/ablation_c5.err; echo "ablation exit $?" >> gpurun_out/summary.txt
timeout 600 python scripts/memory_report.py > gpurun_out/memory_report.jsonl 2> gpurun_out/memory_report.err; echo "memory exit $?" >> gpurun_out/summary.txt
timeout 600 python bench.py --workload c4 --steps 10 --warmup 3 --no-cpu-baseline --no-c4-ref > gpurun_out/bench_c4.log 2>&1; echo "bench c4 exit $?" >> gpurun_out/summary.txt
# sanitizer passes on small shapes of every hand-rolled protocol (GEMM mbarrier rings, CTA pairs,
# cluster split-K, streaming attention, the persistent trunk's grid barrier)
for tool in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 20 --error-exitcode 9 python scripts/sanitize_cases.py > gpurun_out/sanitizer_$tool.log 2>&1; echo "sanitizer $tool exit $?" >> gpurun_out/summary.txt
done
cat gpurun_out/summary.txt
