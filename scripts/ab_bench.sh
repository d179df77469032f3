#!/bin/bash
# A/B timing of library variants on one box: alternates the in-tree build with
# paper_2603_28708_b200/_lib/ab/*.so (PRLAB_GPU_LIB) over several rounds.
# usage: ROUNDS=3 WL=c2 scripts/ab_bench.sh [extra env assignments as VAR=VAL variant names...]
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
WL=${WL:-c2}
for r in $(seq ${ROUNDS:-3}); do
  for lib in paper_2603_28708_b200/_lib/libprlab_gpu.so paper_2603_28708_b200/_lib/ab/*.so; do
    v=$(PRLAB_GPU_LIB=$lib timeout 300 python bench.py --workload $WL --steps ${STEPS:-200} --warmup 10 --no-cpu-baseline --no-e2e --no-profile 2>/dev/null | grep '^{' | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'])")
    echo "$r $(basename $lib) $v"
  done
  for e in "$@"; do
    v=$(env $e timeout 300 python bench.py --workload $WL --steps ${STEPS:-200} --warmup 10 --no-cpu-baseline --no-e2e --no-profile 2>/dev/null | grep '^{' | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'])")
    echo "$r $e $v"
  done
done
