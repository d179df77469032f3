#!/bin/bash
# copy-out tuning of the drop-in forward (C2): widening threads x row chunks, plus the fp32 copy
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
for t in 4 8 12; do for c in 6 8 12 16; do
  PRLAB_HOST_COPY=widen PRLAB_WIDEN_THREADS=$t PRLAB_WIDEN_CHUNKS=$c timeout 120 python scripts/e2e_sweep.py
done; done 2>&1 | grep '^{' | tee gpurun_out/e2e_sweep.jsonl
PRLAB_HOST_COPY=fp32 timeout 120 python scripts/e2e_sweep.py | tee -a gpurun_out/e2e_sweep.jsonl
