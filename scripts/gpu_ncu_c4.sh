#!/bin/bash
# ncu --set full of one instance of every C4 tensor-core kernel (layer 0) and the LM head
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
TAG=${TAG:-c4}
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"gemm_tc|attn_tc" -c 5 \
   -o gpurun_out/${TAG}_layer python bench.py --workload c4 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-profile > gpurun_out/ncu_${TAG}_layer.log 2>&1
echo "ncu layer exit $?"
if [ -z "$NO_HEAD" ]; then
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"gemm_tc" --launch-skip 48 -c 1 \
   -o gpurun_out/${TAG}_head python bench.py --workload c4 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-profile > gpurun_out/ncu_${TAG}_head.log 2>&1
echo "ncu head exit $?"
fi
