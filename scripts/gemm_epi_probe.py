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


def cublas_fused_equivalent(m, n, k, op, reps=20):
    """cuBLAS GEMM + the same epilogue as separate torch ops (what an unfused stack runs):
    qkv: + bias -> fp16; ffn1: + bias, GELU -> fp16; wo / ffn2: x += (acc + bias) in fp32."""
    a = torch.randn(m, k, device="cuda").half()
    b = torch.randn(n, k, device="cuda").half()
    bias = torch.randn(n, device="cuda").half()
    x = torch.randn(m, n, device="cuda")

    def step():
        y = torch.matmul(a, b.t())
        if op == "gelu":
            torch.nn.functional.gelu(y + bias)
        elif op == "resid":
            x.add_(y + bias)
        else:
            y + bias
    for _ in range(3):
        step()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = 1e9
    for _ in range(3):
        e0.record()
        for _ in range(reps):
            step()
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1) * 1000 / reps)
    return best


for name, (n, k, epis, op) in {"qkv": (3 * H, H, (0, 3), "bias"), "wo": (H, H, (2, 0, 3), "resid"),
                               "ffn1": (F, H, (1, 0, 3), "gelu"), "ffn2": (H, F, (2, 0, 3), "resid")}.items():
    row = {"gemm": name, "M": M, "N": n, "K": k, "cublas_us": round(cublas(M, n, k), 2),
           "cublas_plus_torch_epilogue_us": round(cublas_fused_equivalent(M, n, k, op), 2)}
    for e in epis:
        us, tf, _ = time_cfg(M, n, k, e, 0, 0, 0)
        row[f"epi{e}_us"] = round(us, 2)
    print(json.dumps(row), flush=True)
