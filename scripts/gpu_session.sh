#!/bin/bash
# One GPU session: tests, smoke, bench, launch list.  Logs -> gpurun_out/
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > gpurun_out/gpu.txt 2>&1
nproc >> gpurun_out/gpu.txt
for t in ${TESTS:-tests/test_gpu_kernels.py tests/test_gpu_forward.py}; do
  n=$(basename $t .py)
  timeout ${TEST_TIMEOUT:-900} python -m pytest $t -q -m gpu -p no:cacheprovider --timeout 300 -rf > gpurun_out/$n.log 2>&1
  echo "$t exit $?" >> gpurun_out/summary.txt
done
if [ -z "$NO_SMOKE" ]; then
  timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke exit $?" >> gpurun_out/summary.txt
fi
if [ -z "$NO_BENCH" ]; then
  timeout 600 python bench.py ${BENCH_ARGS:---steps 30 --warmup 5} > gpurun_out/bench.log 2>&1; echo "bench exit $?" >> gpurun_out/summary.txt
fi
if [ -n "$NCU" ]; then
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
     python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-profile > gpurun_out/ncu_bench.log 2>&1
  echo "ncu exit $?" >> gpurun_out/summary.txt
fi
cat gpurun_out/summary.txt
