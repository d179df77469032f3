#!/bin/bash
# Session refresh: C4 layer-0 kernels + head (attention now split into tile units), the
# fused-NLL head (EPI_ROWSTAT), and the C2 trunk + head; launch lists of both workloads.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"gemm_|attn_tc|ln_f16|embed_f32" -c 8 \
   -o gpurun_out/c4_layer python bench.py --workload c4 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-profile > gpurun_out/ncu_c4_layer.log 2>&1
echo "ncu c4 layer exit $?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"gemm_tc" --launch-skip 48 -c 1 \
   -o gpurun_out/c4_head python bench.py --workload c4 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-profile > gpurun_out/ncu_c4_head.log 2>&1
echo "ncu c4 head exit $?"
# the fused-statistics head: 49th tensor-core GEMM of the nll forward (4 per layer x 12 + head)
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"gemm_tc2" --launch-skip 48 -c 1 \
   -o gpurun_out/c4_head_rowstat python scripts/nll_bench.py > gpurun_out/ncu_c4_rowstat.log 2>&1
echo "ncu rowstat exit $?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"fwd_small|gemm_tc" -c 2 \
   -o gpurun_out/c2_small python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-profile > gpurun_out/ncu_c2_small.log 2>&1
echo "ncu c2 exit $?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c4.csv \
   python bench.py --workload c4 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-profile > /dev/null 2>&1
echo "launches c4 exit $?"
