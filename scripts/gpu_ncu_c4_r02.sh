cd "${GRAFT_REPO_ROOT}"
mkdir -p gpurun_out
wl=c4
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"gemm_|attn_|ln_f16|embed_f32" -c 8 -o gpurun_out/${wl}_layer python bench.py --workload $wl --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-profile > gpurun_out/ncu_${wl}_layer.log 2>&1
echo "layer $?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"gemm_tc" --launch-skip 48 -c 1 -o gpurun_out/${wl}_head python bench.py --workload $wl --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-profile > gpurun_out/ncu_${wl}_head.log 2>&1
echo "head $?"
cp profiles/r02/traffic.json gpurun_out/traffic.json
python scripts/ncu_traffic.py gpurun_out/traffic.json c4=gpurun_out/c4_layer.ncu-rep,gpurun_out/c4_head.ncu-rep > /dev/null 2>&1; echo "traffic $?"
python scripts/ncu_summary.py gpurun_out/c4_layer.ncu-rep > gpurun_out/ncu_c4_layer.txt 2>&1
python scripts/ncu_summary.py gpurun_out/c4_head.ncu-rep > gpurun_out/ncu_c4_head.txt 2>&1
mkdir -p /tmp/ncu_reps && mv gpurun_out/*.ncu-rep /tmp/ncu_reps/
