#!/bin/bash
# C2 (batch 1, seq 128) = the persistent trunk kernel + the LM head: one `ncu --set full`
# capture of each, the step's launch list, and the traffic entry bench.py reads
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
B="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-profile"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:fwd_small -c 1 -o gpurun_out/c2_fwd_small $B > gpurun_out/ncu_c2_fwd_small.log 2>&1
echo "ncu trunk exit $?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"gemm_" -c 1 -o gpurun_out/c2_head $B > gpurun_out/ncu_c2_head.log 2>&1
echo "ncu head exit $?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c2_small.csv $B > /dev/null 2>&1
echo "ncu launches exit $?"
