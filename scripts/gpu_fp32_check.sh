#!/bin/bash
# fp32-policy path: tensor-core linear tests, fp32 parity tests, forward timing A/B (SIMT vs 3xTF32), C5 ablation
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_kernels.py -q -m gpu -p no:cacheprovider --timeout 300 -k "f32_tensor_core" 2>&1 | tail -1
timeout 1500 python -m pytest tests -q -m gpu -p no:cacheprovider --timeout 600 > gpurun_out/tests_fp32tc.log 2>&1; echo "suite $?"; tail -2 gpurun_out/tests_fp32tc.log
for e in PRLAB_NO_TF32X3=1 NONE=1; do
  echo "$e $(env $e POLICY=fp32 timeout 300 python scripts/launches_m256.py bert_base 1 512) $(env $e POLICY=fp32 timeout 300 python scripts/launches_m256.py bert_base 1 128)"
done
timeout 900 python scripts/ablation.py > gpurun_out/ablation_c5.jsonl 2> gpurun_out/ablation_c5.err; echo "ablation $?"; cat gpurun_out/ablation_c5.jsonl | cut -c1-200
