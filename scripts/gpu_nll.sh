#!/bin/bash
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_logits_reduce.py -q -m gpu -p no:cacheprovider --timeout 600 -x 2>&1 | tail -15
timeout 300 python scripts/nll_bench.py | tee gpurun_out/nll_bench.jsonl
PRLAB_NO_FUSED_NLL=1 timeout 300 python scripts/nll_bench.py | tee -a gpurun_out/nll_bench.jsonl
