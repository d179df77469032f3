#!/bin/bash
# ncu --set full (source-level) of one launch of the row-owner attention kernel at C4 shape
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
TAG=${TAG:-attn_row}
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"attn_fa" -s 3 -c 1 \
   -o gpurun_out/${TAG} python scripts/attn_time.py > gpurun_out/ncu_${TAG}.log 2>&1
echo "ncu exit $?"
ncu -i gpurun_out/${TAG}.ncu-rep --page source --csv --print-source sass > gpurun_out/${TAG}_sass.csv 2>/dev/null
ncu -i gpurun_out/${TAG}.ncu-rep --page details --csv > gpurun_out/${TAG}_details.csv 2>/dev/null
ls -la gpurun_out/ | grep $TAG
