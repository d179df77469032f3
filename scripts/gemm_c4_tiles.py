#!/usr/bin/env python3
"""C4 fused GEMMs (FFN1 GELU, Wo / FFN2 residual): tile width x CTA-pair / single-CTA kernel,
CUDA-graph timed (sweep_gemm.time_cfg); which configuration hides the fused epilogue best."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from sweep_gemm import time_cfg  # noqa: E402

M, H, F = 16384, 768, 3072
for name, (n, k, epi) in {"ffn1": (F, H, 1), "wo": (H, H, 2), "ffn2": (H, F, 2)}.items():
    for bn, lean, what in [(0, 0, "auto"), (256, 2, "pair bn256"), (128, 2, "pair bn128"), (256, -2, "1cta bn256"),
                           (128, -2, "1cta bn128")]:
        try:
            us, tf, _ = time_cfg(M, n, k, epi, bn, 1, lean)
            print(json.dumps({"gemm": name, "cfg": what, "us": round(us, 2), "tflops": round(tf, 1)}), flush=True)
        except Exception as e:  # noqa: BLE001
            print(json.dumps({"gemm": name, "cfg": what, "error": str(e)[:120]}), flush=True)
