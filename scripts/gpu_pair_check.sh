#!/bin/bash
# CTA-pair trunk (128 < B*S <= 256): parity tests, C3 timings against the multi-kernel path
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_fwd_small.py -q -m gpu -p no:cacheprovider --timeout 300 -x 2>&1 | tail -4
for e in PRLAB_NO_SMALL_PAIR=1 NONE=1; do
  for bs in "2 128" "4 64" "8 32" "1 128"; do echo "$e $(env $e timeout 300 python scripts/launches_m256.py bert_base $bs)"; done
done
