#!/bin/bash
# Round-end validation of HEAD: every GPU test, smoke, default bench (C2, cpu_baseline + e2e),
# C4 bench, the reference arm, C3 sweep + C5 ablation, launch lists, C4 ncu for traffic.json.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
: > gpurun_out/summary.txt
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > gpurun_out/gpu.txt 2>&1
timeout 1500 python -m pytest tests -q -m gpu -p no:cacheprovider --timeout 600 -rf > gpurun_out/tests_gpu.log 2>&1; echo "tests exit $?" >> gpurun_out/summary.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke exit $?" >> gpurun_out/summary.txt
timeout 900 python bench.py > gpurun_out/bench_c2.log 2>&1; echo "bench c2 exit $?" >> gpurun_out/summary.txt
timeout 600 python bench.py --workload c4 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c4.log 2>&1; echo "bench c4 exit $?" >> gpurun_out/summary.txt
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.log 2>&1; echo "bench ref exit $?" >> gpurun_out/summary.txt
timeout 900 python scripts/sweep_c3.py > gpurun_out/sweep_c3.jsonl 2> gpurun_out/sweep_c3.err; echo "sweep c3 exit $?" >> gpurun_out/summary.txt
timeout 900 python scripts/ablation.py > gpurun_out/ablation_c5.jsonl 2> gpurun_out/ablation_c5.err; echo "ablation exit $?" >> gpurun_out/summary.txt
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c2.csv \
   python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-profile > /dev/null 2>&1
echo "ncu c2 launches exit $?" >> gpurun_out/summary.txt
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c4.csv \
   python bench.py --workload c4 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-profile > /dev/null 2>&1
echo "ncu c4 launches exit $?" >> gpurun_out/summary.txt
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"gemm_|attn_|ln_f16|embed_f32" -c 8 \
   -o gpurun_out/c4_layer python bench.py --workload c4 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-profile > gpurun_out/ncu_c4_layer.log 2>&1
echo "ncu c4 layer exit $?" >> gpurun_out/summary.txt
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"gemm_tc" --launch-skip 48 -c 1 \
   -o gpurun_out/c4_head python bench.py --workload c4 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-profile > gpurun_out/ncu_c4_head.log 2>&1
echo "ncu c4 head exit $?" >> gpurun_out/summary.txt
cat gpurun_out/summary.txt
