#!/usr/bin/env python3
"""Launch one GEMM configuration a few times (for ncu): one_gemm.py M N K epi bn splits lean"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2603_28708_b200 as pg  # noqa: E402

M, N, K, epi, bn, sp, ln = (int(x) for x in sys.argv[1:8])
A = (torch.randn(M, K, device="cuda") * 0.5).half()
W = (torch.randn(N, K, device="cuda") * 0.02).half()
bias = torch.zeros(N, device="cuda")
out = torch.zeros(M, N, device="cuda", dtype=torch.float32 if epi == 2 else torch.float16)
for _ in range(4):
    pg.linear_f16_device_ex(A, W, bias, out, M, N, K, N, epi, bn, sp, ln)
torch.cuda.synchronize()
