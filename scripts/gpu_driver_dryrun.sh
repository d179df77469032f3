#!/bin/bash
# what the driver runs at round end: smoke(), the default bench line, the reference arm
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke $?"; tail -1 gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench_default.log 2>&1; echo "bench $?"
timeout 900 python bench.py --impl reference > gpurun_out/bench_reference.log 2>&1; echo "reference $?"
tail -1 gpurun_out/bench_default.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print({k: d[k] for k in ('value','ms_per_step','gpu_launches','clocks')}); print('e2e', d['e2e']['value'], 'cpu', d['cpu_baseline']['value'], d['cpu_baseline']['cores']); print('roof', d['roofline']['frac'], d['roofline'].get('traffic_source')); print('c4', d.get('c4_single_gpu',{}).get('ms_per_step'))"
tail -1 gpurun_out/bench_reference.log | cut -c1-300
