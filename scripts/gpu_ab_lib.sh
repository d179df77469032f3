#!/bin/bash
# Same-box A/B of two builds of the library: abtmp/base.so (PRLAB_GPU_LIB) vs the in-tree build,
# on the batch-1 / mid-size trunk (scripts/trunk_vs_head.py), 3 alternating rounds
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
for rep in 1 2 3; do
  for v in base new; do
    if [ $v = base ]; then export PRLAB_GPU_LIB=$PWD/abtmp/base.so; else unset PRLAB_GPU_LIB; fi
    echo "$v $(timeout 300 python scripts/trunk_vs_head.py) $(B=2 CFG=bert_base timeout 300 python scripts/trunk_vs_head.py)"
  done
done
