#!/bin/bash
# attention variant check: attention parity tests, then the kernel's ncu time at C4
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_kernels.py -q -m gpu -p no:cacheprovider -k "attention" --timeout 300 -x 2>&1 | tail -2
bash scripts/gpu_ncu_attn.sh
python scripts/ncu_summary.py gpurun_out/attn_fa.ncu-rep 2>/dev/null | head -3
