#!/bin/bash
# CTA-pair trunk (B=2, S=128, BERT-base): one `ncu --set full` capture, raw metrics + source
# page exported as CSV (the .ncu-rep stays on the box: gpurun_out is size-capped)
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
export B=${B:-2} S=${S:-128}
timeout 900 ncu --replay-mode ${REPLAY:-application} -f ${NCU_SETS:---set full} --import-source on --clock-control none -k regex:fwd_small -c 1 -o /tmp/pair_trunk \
  python scripts/small_stages.py ${CFG:-bert_base} > gpurun_out/ncu_pair.log 2>&1
echo "ncu exit $?"
ncu -i /tmp/pair_trunk.ncu-rep --page raw --csv > gpurun_out/ncu_pair_raw.csv 2>&1
ncu -i /tmp/pair_trunk.ncu-rep --page source --csv --print-source sass > gpurun_out/ncu_pair_sass.csv 2>&1
ncu -i /tmp/pair_trunk.ncu-rep --page details --csv > gpurun_out/ncu_pair_details.csv 2>&1
ls -la gpurun_out/ncu_pair*
