#!/bin/bash
# overlapped drop-in forward: concurrency tests, then the C2 bench line (e2e with 2 concurrent
# callers; single-caller latency alongside), and an A/B of the serial path
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
: > gpurun_out/summary.txt
timeout 600 python -m pytest tests/test_gpu_concurrency.py tests/test_gpu_dropin.py -q -m gpu -p no:cacheprovider --timeout 300 > gpurun_out/tests_conc.log 2>&1; echo "tests exit $?" >> gpurun_out/summary.txt
tail -3 gpurun_out/tests_conc.log >> gpurun_out/summary.txt
for c in 2 3 1; do
  timeout 300 python bench.py --steps 50 --warmup 5 --no-cpu-baseline --no-cpu-latency --no-c4-ref --no-profile --e2e-callers $c > gpurun_out/bench_e2e_c$c.log 2>&1; echo "bench callers=$c exit $?" >> gpurun_out/summary.txt
  tail -1 gpurun_out/bench_e2e_c$c.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], json.dumps(d['e2e']))" >> gpurun_out/summary.txt
done
cat gpurun_out/summary.txt
