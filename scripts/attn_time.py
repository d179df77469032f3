#!/usr/bin/env python3
"""Attention kernel time at a given shape (CUDA events, 50 launches after warm-up)."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2603_28708_b200 as pg  # noqa: E402

B, S, causal = int(os.environ.get("B", 32)), int(os.environ.get("S", 512)), int(os.environ.get("CAUSAL", 1))
H, hd = 12, 64
qkv = (torch.randn(B * S, 3 * H * hd, device="cuda") * 1.5).half()
ctx = torch.empty(B * S, H * hd, device="cuda", dtype=torch.float16)
for _ in range(5):
    pg.attention_f16_device(qkv, ctx, B, S, H, hd, causal)
torch.cuda.synchronize()
best = 1e9
for _ in range(5):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(50):
        pg.attention_f16_device(qkv, ctx, B, S, H, hd, causal)
    e1.record()
    torch.cuda.synchronize()
    best = min(best, e0.elapsed_time(e1) * 1000 / 50)
print(json.dumps({"lib": os.path.basename(os.environ.get("PRLAB_GPU_LIB", "default")), "B": B, "S": S,
                  "causal": causal, "us": round(best, 2)}))
