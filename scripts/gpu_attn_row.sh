#!/bin/bash
# row-owner streaming attention: parity tests, C4-shape timing A/B against the half-row kernel,
# phase stamps, C4 forward A/B
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_fp16_fast.py -q -m gpu -p no:cacheprovider --timeout 600 -x -k "attn or attention or fp16" 2>&1 | tail -3
for e in PRLAB_ATTN_ROW=0 PRLAB_ATTN_ROW=1 PRLAB_ATTN_ROW=0 PRLAB_ATTN_ROW=1; do echo "$e $(env $e timeout 120 python scripts/attn_time.py)"; done
for e in PRLAB_ATTN_ROW=0 PRLAB_ATTN_ROW=1; do echo "$e noncausal $(env $e CAUSAL=0 timeout 120 python scripts/attn_time.py)"; done
timeout 120 python scripts/fa_phases.py
for e in PRLAB_ATTN_ROW=0 PRLAB_ATTN_ROW=1; do echo "$e c4 $(env $e timeout 300 python bench.py --workload c4 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-c4-ref 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['roofline']['breakdown_us_per_forward'])")"; done
