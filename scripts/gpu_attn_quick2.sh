#!/bin/bash
# attention variant check: parity tests of the default kernel, C4-shape timing of each variant, phases
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
timeout 600 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_fp16_fast.py -q -m gpu -p no:cacheprovider --timeout 300 -x -k "attn or attention or fp16" 2>&1 | tail -1
for e in PRLAB_ATTN_ROW=0 PRLAB_ATTN_ROW=1 PRLAB_ATTN_ROW=2; do echo "$e $(env $e timeout 120 python scripts/attn_time.py) $(env $e CAUSAL=0 timeout 120 python scripts/attn_time.py | cut -c40-)"; done
timeout 120 python scripts/fa_phases.py
