#!/bin/bash
# attention variants: default build vs _lib/ab/*.so at C4 shape (and causal=0), 3 rounds
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
timeout 600 python -m pytest tests/test_gpu_kernels.py -q -m gpu -p no:cacheprovider --timeout 300 -x -k "attn or attention" 2>&1 | tail -1
for r in 1 2 3; do
  for lib in paper_2603_28708_b200/_lib/libprlab_gpu.so paper_2603_28708_b200/_lib/ab/*.so; do
    echo "$r $(basename $lib) $(PRLAB_GPU_LIB=$lib timeout 120 python scripts/attn_time.py) $(PRLAB_GPU_LIB=$lib CAUSAL=0 timeout 120 python scripts/attn_time.py)"
  done
done
