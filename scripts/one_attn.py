#!/usr/bin/env python3
"""Launch the fused attention a few times (for ncu): one_attn.py B S causal"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2603_28708_b200 as pg  # noqa: E402

B, S, causal = (int(x) for x in sys.argv[1:4])
H, hd = 12, 64
qkv = (torch.randn(B * S, 3 * H * hd, device="cuda") * 1.5).half()
ctx = torch.empty(B * S, H * hd, device="cuda", dtype=torch.float16)
for _ in range(3):
    pg.attention_f16_device(qkv, ctx, B, S, H, hd, causal)
torch.cuda.synchronize()
