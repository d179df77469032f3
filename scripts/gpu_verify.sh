#!/bin/bash
# full GPU suite + C2 bench line + C4 bench line on one box
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
: > gpurun_out/summary.txt
timeout 1500 python -m pytest tests -q -m gpu -p no:cacheprovider --timeout 600 > gpurun_out/tests_verify.log 2>&1; echo "tests exit $?" >> gpurun_out/summary.txt
tail -3 gpurun_out/tests_verify.log >> gpurun_out/summary.txt
grep -E "FAILED|Error" gpurun_out/tests_verify.log | head -10 >> gpurun_out/summary.txt
timeout 600 python bench.py --steps 50 --warmup 5 > gpurun_out/bench_c2_verify.log 2>&1; echo "bench c2 exit $?" >> gpurun_out/summary.txt
tail -1 gpurun_out/bench_c2_verify.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c2', d['ms_per_step'], d['value'], 'e2e', d['e2e']['value'], d['clocks'])" >> gpurun_out/summary.txt
timeout 600 python bench.py --workload c4 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-c4-ref > gpurun_out/bench_c4_verify.log 2>&1; echo "bench c4 exit $?" >> gpurun_out/summary.txt
tail -1 gpurun_out/bench_c4_verify.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c4', d['ms_per_step'], d['value'], d['roofline']['breakdown_us_per_forward'], d['clocks'])" >> gpurun_out/summary.txt
cat gpurun_out/summary.txt
