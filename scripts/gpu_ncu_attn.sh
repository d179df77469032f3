#!/bin/bash
# ncu --set full of the C4 attention kernel (layer 0), with source-level metrics
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
TAG=${TAG:-attn_fa}
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"attn_" -c 1 \
   -o gpurun_out/${TAG} python bench.py --workload c4 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-profile > gpurun_out/ncu_${TAG}.log 2>&1
echo "ncu exit $?"
