#!/bin/bash
# Round-2 profile set: C2 trunk/head ncu --set full + launch list, C4 layer/head ncu --set full,
# traffic.json inputs, the C3 sweep on the current paths
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
bash scripts/gpu_ncu_small.sh
bash scripts/gpu_ncu_full.sh 2>&1 | grep c4
python scripts/ncu_traffic.py gpurun_out/traffic.json c2=small:gpurun_out/c2_fwd_small.ncu-rep,gpurun_out/c2_head.ncu-rep c4=gpurun_out/c4_layer.ncu-rep,gpurun_out/c4_head.ncu-rep > /dev/null 2>&1; echo "traffic $?"
for f in c2_fwd_small c2_head c4_layer c4_head; do python scripts/ncu_summary.py gpurun_out/$f.ncu-rep > gpurun_out/ncu_$f.txt 2>&1; done
timeout 1500 python scripts/sweep_c3.py > gpurun_out/sweep_c3.jsonl 2> gpurun_out/sweep_c3.err; echo "sweep $?"
ls gpurun_out
# the --set full reports are large (the copy-back limit is 64 MiB): keep summaries, traffic, sass/source of the trunk
ncu -i gpurun_out/c2_fwd_small.ncu-rep --page details --csv > gpurun_out/ncu_c2_fwd_small_details.csv 2>/dev/null
mkdir -p /tmp/ncu_reps && mv gpurun_out/*.ncu-rep /tmp/ncu_reps/ 2>/dev/null
du -sh gpurun_out
