#!/bin/bash
# LayerNorm variant check: kernel/forward tests, ncu time of the C4 LayerNorm, C4 bench
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_forward.py tests/test_gpu_sweep.py -q -m gpu -p no:cacheprovider --timeout 600 -x 2>&1 | tail -2
timeout 600 ncu --set full --clock-control none -k regex:"ln_f16|embed_f32" -c 3 -o gpurun_out/c4_ln python bench.py --workload c4 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-profile > /dev/null 2>&1
python scripts/ncu_summary.py gpurun_out/c4_ln.ncu-rep 2>/dev/null | grep -E "kernel|time|dram|occ"
for r in 1 2; do timeout 300 python bench.py --workload c4 --steps 20 --warmup 5 --no-cpu-baseline --no-e2e 2>/dev/null | grep '^{' | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['clocks']['sm_mhz'])"; done
