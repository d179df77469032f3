#!/bin/bash
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_kernels.py -q -m gpu -p no:cacheprovider --timeout 300 -rf -x > gpurun_out/test_gpu_kernels.log 2>&1; echo "kernels exit $?" >> gpurun_out/summary.txt
timeout 300 python scripts/attn_phases.py > gpurun_out/attn_phases.jsonl 2>&1; echo "phases exit $?" >> gpurun_out/summary.txt
timeout 600 python scripts/sweep_gemm.py c2 > gpurun_out/sweep.jsonl 2> gpurun_out/sweep.err; echo "sweep exit $?" >> gpurun_out/summary.txt
timeout 600 python bench.py --steps 200 --warmup 10 --no-cpu-baseline > gpurun_out/bench_c2.log 2>&1; echo "bench c2 exit $?" >> gpurun_out/summary.txt
timeout 900 ncu --set full --clock-control none --import-source on -k regex:attn_tc_kernel -s 30 -c 1 -o gpurun_out/prof_attn_c4 \
     python bench.py --workload c4 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-profile > gpurun_out/ncu2.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm_tc_kernel -s 26 -c 3 -o gpurun_out/prof_gemm_c4 \
     python bench.py --workload c4 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-profile > gpurun_out/ncu1.log 2>&1
echo "ncu exit $?" >> gpurun_out/summary.txt
cat gpurun_out/summary.txt
