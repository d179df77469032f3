#!/bin/bash
# attention exp-offload sweep: phase stamps for each PRLAB_ATTN_POLY variant
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
for v in 0 34 85; do
  PRLAB_ATTN_POLY=$v timeout 300 python scripts/attn_phases.py > gpurun_out/attn_poly_$v.jsonl 2>&1
done
timeout 600 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_forward.py -q -m gpu -p no:cacheprovider --timeout 300 -x > gpurun_out/tests_quick.log 2>&1; echo "tests $?"
timeout 600 python bench.py --workload c4 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_c4.log 2>&1; echo "c4 $?"
