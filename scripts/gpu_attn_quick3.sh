#!/bin/bash
# row-owner attention variants: parity under each threads-per-row setting, C4-shape timing
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
for v in 1 2 4; do PRLAB_ATTN_ROW=$v timeout 600 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_fp16_fast.py -q -m gpu -p no:cacheprovider --timeout 300 -x -k "attn or attention or fp16" 2>&1 | tail -1; done
for r in 1 2; do for e in PRLAB_ATTN_ROW=1 PRLAB_ATTN_ROW=2 PRLAB_ATTN_ROW=4; do echo "$e $(env $e timeout 120 python scripts/attn_time.py) $(env $e CAUSAL=0 timeout 120 python scripts/attn_time.py | cut -c40-)"; done; done
