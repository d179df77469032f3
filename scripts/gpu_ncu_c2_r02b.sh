#!/bin/bash
# C2 (batch 1, seq 128): ncu --set full of the barrier-free persistent trunk + the LM head,
# the launch list, and the traffic entries bench.py reads; reports stay on the box (/tmp)
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out /tmp/ncu_reps
B="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-profile"
timeout 900 ncu -f --set full --import-source on --clock-control none -k regex:fwd_small -c 1 -o /tmp/ncu_reps/c2_fwd_small $B > gpurun_out/ncu_c2_fwd_small.log 2>&1
echo "ncu trunk exit $?"
timeout 900 ncu -f --set full --import-source on --clock-control none -k regex:"gemm_" -c 1 -o /tmp/ncu_reps/c2_head $B > gpurun_out/ncu_c2_head.log 2>&1
echo "ncu head exit $?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c2_small.csv $B > /dev/null 2>&1
echo "ncu launches exit $?"
cp profiles/r02/traffic.json gpurun_out/traffic.json
python scripts/ncu_traffic.py gpurun_out/traffic.json c2=small:/tmp/ncu_reps/c2_fwd_small.ncu-rep,/tmp/ncu_reps/c2_head.ncu-rep > /dev/null 2>&1; echo "traffic $?"
python scripts/ncu_summary.py /tmp/ncu_reps/c2_fwd_small.ncu-rep > gpurun_out/ncu_c2_fwd_small.txt 2>&1
python scripts/ncu_summary.py /tmp/ncu_reps/c2_head.ncu-rep > gpurun_out/ncu_c2_head.txt 2>&1
ncu -i /tmp/ncu_reps/c2_fwd_small.ncu-rep --page details --csv > gpurun_out/ncu_c2_fwd_small_details.csv 2>&1
head -20 gpurun_out/ncu_c2_fwd_small.txt
