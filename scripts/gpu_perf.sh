#!/bin/bash
# perf session: kernel tests (fast), bench C2 + C4, optional ncu launch list
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_kernels.py -q -m gpu -p no:cacheprovider --timeout 300 -rf -x > gpurun_out/test_gpu_kernels.log 2>&1; echo "kernels exit $?" >> gpurun_out/summary.txt
if [ -n "$FWD" ]; then timeout 900 python -m pytest tests/test_gpu_forward.py -q -m gpu -p no:cacheprovider --timeout 300 -rf > gpurun_out/test_gpu_forward.log 2>&1; echo "forward exit $?" >> gpurun_out/summary.txt; fi
timeout 600 python bench.py --steps 200 --warmup 10 --no-cpu-baseline > gpurun_out/bench_c2.log 2>&1; echo "bench c2 exit $?" >> gpurun_out/summary.txt
timeout 600 python bench.py --workload c4 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_c4.log 2>&1; echo "bench c4 exit $?" >> gpurun_out/summary.txt
if [ -n "$NCU" ]; then
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c2.csv \
     python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-profile > /dev/null 2>&1
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c4.csv \
     python bench.py --workload c4 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-profile > /dev/null 2>&1
  echo "ncu exit $?" >> gpurun_out/summary.txt
fi
cat gpurun_out/summary.txt
