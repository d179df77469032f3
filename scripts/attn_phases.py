#!/usr/bin/env python3
"""Per-phase clock64 breakdown of the fused attention CTA (debug stamps)."""
import ctypes as C
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2603_28708_b200 as pg  # noqa: E402

NAMES = ["setup", "q_wait", "qk+s_wait", "pass1", "pass2", "pass3", "pv+o_wait"]


def run(B, S, causal, H=12, hd=64):
    qkv = (torch.randn(B * S, 3 * H * hd, device="cuda") * 1.5).half()
    ctx = torch.empty(B * S, H * hd, device="cuda", dtype=torch.float16)
    nqt = (S + 127) // 128
    grid = B * H * nqt
    dbg = torch.zeros(grid, 8, dtype=torch.int64, device="cuda")
    for _ in range(3):
        pg.attention_f16_device(qkv, ctx, B, S, H, hd, causal)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        pg.attention_f16_device(qkv, ctx, B, S, H, hd, causal)
    e1.record()
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) * 100
    pg._check(pg.lib().prlab_gpu_attention_f16_device_dbg(C.c_void_p(qkv.data_ptr()), C.c_void_p(ctx.data_ptr()),
                                                          B, S, H, hd, causal, None, C.c_void_p(dbg.data_ptr())))
    torch.cuda.synchronize()
    d = dbg.cpu().double()
    out = {"B": B, "S": S, "causal": causal, "kernel_us": round(us, 2), "ctas": grid}
    for qt in range(nqt):
        rows = d[qt::nqt]
        ph = {}
        for i in range(7):
            j0, j1 = (0, 1) if i == 0 else ((1, 2) if i == 1 else (i, i + 1))
            if i == 2:
                j0, j1 = 2, 3
            ph[NAMES[i]] = round(float((rows[:, j1] - rows[:, j0]).mean()), 0)
        ph["total"] = round(float((rows[:, 7] - rows[:, 0]).mean()), 0)
        out[f"qt{qt}_cycles"] = ph
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    for B, S, c in [(32, 512, 1), (32, 512, 0), (1, 128, 1), (32, 128, 0)]:
        run(B, S, c)
