#!/bin/bash
# C4 (GPT-2 32x512, forward + fused NLL): ncu --set full of layer 0's kernels and of the
# fused-statistics LM head, their summaries and the traffic entries bench.py reads
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out /tmp/ncu_reps
wl=c4
B="python bench.py --workload $wl --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-profile"
timeout 900 ncu -f --set full --import-source on --clock-control none -k regex:"gemm_|attn_|ln_f16|embed_f32" -c 8 -o /tmp/ncu_reps/${wl}_layer $B > gpurun_out/ncu_${wl}_layer.log 2>&1
echo "layer $?"
timeout 900 ncu -f --set full --import-source on --clock-control none -k regex:"gemm_tc" --launch-skip 48 -c 1 -o /tmp/ncu_reps/${wl}_head $B > gpurun_out/ncu_${wl}_head.log 2>&1
echo "head $?"
cp profiles/r02/traffic.json gpurun_out/traffic.json
python scripts/ncu_traffic.py gpurun_out/traffic.json c4=/tmp/ncu_reps/${wl}_layer.ncu-rep,/tmp/ncu_reps/${wl}_head.ncu-rep > /dev/null 2>&1; echo "traffic $?"
python scripts/ncu_summary.py /tmp/ncu_reps/${wl}_layer.ncu-rep > gpurun_out/ncu_${wl}_layer.txt 2>&1
python scripts/ncu_summary.py /tmp/ncu_reps/${wl}_head.ncu-rep > gpurun_out/ncu_${wl}_head.txt 2>&1
grep -A3 "attn_fa_row\|gemm_tc2_kernel<256, 1\|gemm_tc2_kernel<256, 4" gpurun_out/ncu_${wl}_layer.txt gpurun_out/ncu_${wl}_head.txt | head -20
