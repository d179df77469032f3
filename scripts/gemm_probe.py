#!/usr/bin/env python3
"""Pacing probe of the CTA-pair GEMM at the C4 shapes: normal vs no-load (operand
TMA skipped after the first fill: MMA + epilogue only) -> is the main loop
operand-feed bound or MMA/epilogue bound?"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from sweep_gemm import shapes, time_cfg  # noqa: E402

M = 16384
for name, (m, n, k, epi) in shapes(M).items():
    res = {"gemm": name, "M": m, "N": n, "K": k}
    for mode, v in (("normal", None), ("no_operands", "3"), ("no_A", "1"), ("no_B", "2")):
        if v:
            os.environ["PRLAB_DBG_GEMM_NOLOAD"] = v
        else:
            os.environ.pop("PRLAB_DBG_GEMM_NOLOAD", None)
        us, tf, _ = time_cfg(m, n, k, epi, 0, 0, 0, reps=10)
        res[mode] = {"us": round(us, 2), "tflops": round(tf, 1)}
    os.environ.pop("PRLAB_DBG_GEMM_NOLOAD", None)
    print(json.dumps(res), flush=True)
