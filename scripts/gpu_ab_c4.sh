#!/bin/bash
# attention / large-batch variant check: kernel + forward GPU tests, then C4 A/B of env variants
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_forward.py tests/test_gpu_sweep.py -q -m gpu -p no:cacheprovider --timeout 600 -x 2>&1 | tail -4
for r in $(seq ${ROUNDS:-2}); do
  for e in "NONE=1" "$@"; do
    v=$(env $e timeout 300 python bench.py --workload c4 --steps 20 --warmup 5 --no-cpu-baseline --no-e2e 2>/dev/null | grep '^{' | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['roofline']['breakdown_us_per_forward'].get('attention'))")
    echo "$r $e $v"
  done
done 2>&1 | tee gpurun_out/ab_c4.txt
