#!/bin/bash
# fp32-policy path: parity tests, forward timing (BERT s512 / s128, GPT-2 s128), C5 ablation lines
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_forward.py tests/test_gpu_parity_bars.py tests/test_gpu_kernels.py tests/test_gpu_dropin.py -q -m gpu -p no:cacheprovider --timeout 600 2>&1 | tail -3
for e in PRLAB_NO_ATTN_F32_TILED=1 NONE=1; do
  echo "$e $(env $e POLICY=fp32 timeout 300 python scripts/launches_m256.py bert_base 1 512) $(env $e POLICY=fp32 timeout 300 python scripts/launches_m256.py bert_base 1 128) $(env $e POLICY=fp32 timeout 300 python scripts/launches_m256.py gpt2_small 1 128)"
done
