#!/bin/bash
# ncu --set full of one instance of every tensor-core kernel of layer 0 and the LM head,
# at C2 (batch 1, seq 128) and C4 (batch 32, seq 512)
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
for wl in c2 c4; do
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:"gemm_|attn_|ln_f16|embed_f32" -c 8 \
     -o gpurun_out/${wl}_layer python bench.py --workload $wl --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-profile > gpurun_out/ncu_${wl}_layer.log 2>&1
  echo "ncu $wl layer exit $?"
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:"gemm_tc" --launch-skip 48 -c 1 \
     -o gpurun_out/${wl}_head python bench.py --workload $wl --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-profile > gpurun_out/ncu_${wl}_head.log 2>&1
  echo "ncu $wl head exit $?"
done
