#!/bin/bash
# env-switch A/B of the trunk on one box: parity tests under each variant, alternating rounds of
# the C2 bench, and the stage timeline of the baseline and of each variant.
# usage: gpu_ab_env.sh VAR=VAL [VAR=VAL ...]
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
for e in "$@"; do env "$e" timeout 600 python -m pytest tests/test_gpu_fwd_small.py -q -m gpu -p no:cacheprovider --timeout 300 -x 2>&1 | tail -1; done
ROUNDS=${ROUNDS:-3} WL=c2 bash scripts/ab_bench.sh "$@" 2>/dev/null | grep -v "\*.so" | tee gpurun_out/ab_env.txt
for e in NONE=1 "$@"; do
  echo "== $e"
  env "$e" timeout 300 python scripts/small_stages.py > gpurun_out/small_stages_env.jsonl 2>&1; head -1 gpurun_out/small_stages_env.jsonl | cut -c1-600
done
