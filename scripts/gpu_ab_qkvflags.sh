#!/bin/bash
# A/B: QKV -> attention through per-task flags (default) vs a grid barrier (PRLAB_SMALL_BARRIERS=1)
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
for rep in 1 2; do
  for mode in flags barrier; do
    if [ $mode = barrier ]; then export PRLAB_SMALL_BARRIERS=1; else unset PRLAB_SMALL_BARRIERS; fi
    echo "$mode c2 $(timeout 300 python bench.py --steps 200 --warmup 10 --no-cpu-baseline --no-e2e --no-profile 2>/dev/null | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["ms_per_step"], 4))')"
    echo "$mode c3 $(OUT=f16 B=2 S=128 timeout 300 python scripts/c3_point.py | python -c 'import json,sys; print(json.loads(sys.stdin.read())["ms_p50"])')"
  done
done
