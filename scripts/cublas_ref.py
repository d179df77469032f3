#!/usr/bin/env python3
"""cuBLAS (torch.matmul, fp16 in / fp16 out, fp32 accumulate) on the C4 linear shapes, for
context next to the tcgen05 kernels' bench breakdown: M = 16384 rows (GPT-2, B=32, S=512).
CUDA events, best of 5 x 20 launches per shape; TFLOP/s = 2MNK / time."""
import json

import torch

M = 16384
shapes = {"qkv": (2304, 768), "wo": (768, 768), "ffn1": (3072, 768), "ffn2": (768, 3072), "head": (50257, 768)}
for name, (N, K) in shapes.items():
    a = torch.randn(M, K, device="cuda", dtype=torch.float16)
    w = torch.randn(N, K, device="cuda", dtype=torch.float16)
    for _ in range(3):
        c = a @ w.t()
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(20):
            c = a @ w.t()
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1) / 20)
    print(json.dumps({"gemm": name, "M": M, "N": N, "K": K, "us": round(best * 1e3, 2),
                      "tflops": round(2 * M * N * K / best / 1e9, 1)}))
