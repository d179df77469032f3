#!/bin/bash
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_kernels.py -q -m gpu -p no:cacheprovider --timeout 300 -rf -x > gpurun_out/test_gpu_kernels.log 2>&1; echo "kernels exit $?" >> gpurun_out/summary.txt
timeout 900 python -m pytest tests/test_gpu_forward.py -q -m gpu -p no:cacheprovider --timeout 300 -rf > gpurun_out/test_gpu_forward.log 2>&1; echo "forward exit $?" >> gpurun_out/summary.txt
timeout 300 python scripts/attn_phases.py > gpurun_out/attn_phases.jsonl 2>&1; echo "phases exit $?" >> gpurun_out/summary.txt
timeout 600 python scripts/sweep_gemm.py ${SWEEP:-c4} > gpurun_out/sweep.jsonl 2> gpurun_out/sweep.err; echo "sweep exit $?" >> gpurun_out/summary.txt
timeout 600 python bench.py --steps 200 --warmup 10 --no-cpu-baseline > gpurun_out/bench_c2.log 2>&1; echo "bench c2 exit $?" >> gpurun_out/summary.txt
timeout 600 python bench.py --workload c4 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_c4.log 2>&1; echo "bench c4 exit $?" >> gpurun_out/summary.txt
cat gpurun_out/summary.txt
