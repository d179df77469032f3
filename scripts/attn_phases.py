#!/usr/bin/env python3
"""Fused attention timing: kernel time (CUDA events), per-CTA busy cycles and the
per-tile phase stamps of CTA 0 (clock64, debug build of the stamps)."""
import ctypes as C
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2603_28708_b200 as pg  # noqa: E402

PH = ["s_wait+pass1+prev_epilogue", "max_bar+pass2", "sum_bar", "pass3"]


def run(B, S, causal, H=12, hd=64):
    qkv = (torch.randn(B * S, 3 * H * hd, device="cuda") * 1.5).half()
    ctx = torch.empty(B * S, H * hd, device="cuda", dtype=torch.float16)
    dbg = torch.zeros(max(B * H, 148), 256, dtype=torch.int64, device="cuda")
    for _ in range(3):
        pg.attention_f16_device(qkv, ctx, B, S, H, hd, causal)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20):
        pg.attention_f16_device(qkv, ctx, B, S, H, hd, causal)
    e1.record()
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) * 1000 / 20
    pg._check(pg.lib().prlab_gpu_attention_f16_device_dbg(C.c_void_p(qkv.data_ptr()), C.c_void_p(ctx.data_ptr()),
                                                          B, S, H, hd, causal, None, C.c_void_p(dbg.data_ptr())))
    torch.cuda.synchronize()
    d = dbg.cpu().double()
    used = d[:, 0] > 0
    busy = (d[used, 1] - d[used, 0])
    flops = 4 * B * H * S * S * hd // (2 if causal else 1)
    out = {"B": B, "S": S, "causal": causal, "kernel_us": round(us, 2), "ctas": int(used.sum()),
           "cta_cycles_mean": round(float(busy.mean()), 0), "cta_cycles_max": round(float(busy.max()), 0),
           "cta_cycles_min": round(float(busy.min()), 0), "tflops_executed": round(flops / us / 1e6, 1)}
    c0 = d[0]
    tiles = []
    for t in range(14):
        st = c0[8 + t * 8: 16 + t * 8]
        if st[0] == 0:
            break
        ph = {PH[i]: int(st[i + 1] - st[i]) for i in range(4)}
        if t > 0:
            ph["since_prev_tile"] = int(st[0] - c0[8 + (t - 1) * 8])
        tiles.append(ph)
    out["cta0_tiles"] = tiles

    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    for B, S, c in [(32, 512, 1), (32, 512, 0), (1, 128, 1), (32, 128, 0), (8, 256, 0), (1, 512, 1)]:
        run(B, S, c)
