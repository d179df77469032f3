#!/usr/bin/env python3
"""C4 GEMM shapes with each epilogue variant, next to cuBLAS (torch.matmul fp16) on the same box:
how much of each GEMM is its epilogue (GELU / fp32 residual reduce-add) vs the main loop."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from sweep_gemm import time_cfg  # noqa: E402

M, H, F = 16384, 768, 3072


def cublas(m, n, k, reps=20):
    a = torch.randn(m, k, device="cuda").half()
    b = torch.randn(n, k, device="cuda").half()
    for _ in range(3):
        torch.matmul(a, b.t())
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = 1e9
    for _ in range(3):
        e0.record()
        for _ in range(reps):
            torch.matmul(a, b.t())
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1) * 1000 / reps)
    return best


for name, (n, k, epis) in {"qkv": (3 * H, H, (0, 3)), "wo": (H, H, (2, 0, 3)), "ffn1": (F, H, (1, 0, 3)),
                           "ffn2": (H, F, (2, 0, 3))}.items():
    row = {"gemm": name, "M": M, "N": n, "K": k, "cublas_us": round(cublas(M, n, k), 2)}
    for e in epis:
        us, tf, _ = time_cfg(M, n, k, e, 0, 0, 0)
        row[f"epi{e}_us"] = round(us, 2)
    print(json.dumps(row), flush=True)
