#!/usr/bin/env python3
"""Tile-configuration sweep of the tcgen05 GEMM on the forward's shapes.

Each config is launched 20x inside one CUDA graph (no host overhead) and timed
with CUDA events; prints one JSON line per (shape, config) to stdout."""
import itertools
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2603_28708_b200 as pg  # noqa: E402

H, F, V = 768, 3072, 50257


def shapes(M):
    return {"qkv": (M, 3 * H, H, 0), "wo": (M, H, H, 2), "ffn1": (M, F, H, 1), "ffn2": (M, H, F, 2),
            "head": (M, V, H, 3)}


def time_cfg(M, N, K, epi, bn, splits, lean, reps=20):
    dev = "cuda"
    A = (torch.randn(M, K, device=dev) * 0.5).half()
    W = (torch.randn(N, K, device=dev) * 0.02).half()
    bias = torch.zeros(N, device=dev)
    ldo = N if epi == 2 else (N + 7) // 8 * 8
    out = torch.zeros(M, ldo, device=dev, dtype=torch.float32 if epi == 2 else torch.float16)
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        pg.linear_f16_device_ex(A, W, bias if epi != 3 else None, out, M, N, K, ldo, epi, bn, splits,
                                lean, s.cuda_stream)
        s.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            for _ in range(reps):
                pg.linear_f16_device_ex(A, W, bias if epi != 3 else None, out, M, N, K, ldo, epi, bn,
                                        splits, lean, torch.cuda.current_stream().cuda_stream)
        g.replay()
        s.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        for _ in range(3):
            g.replay()
        e1.record(s)
        s.synchronize()
    us = e0.elapsed_time(e1) * 1000 / (3 * reps)
    flops = 2 * M * N * K
    nbytes = 2 * (M * K + N * K) + (8 if epi == 2 else 2) * M * N
    return us, flops / us / 1e6, nbytes / us / 1e3


def main():
    which = sys.argv[1] if len(sys.argv) > 1 else "both"
    # per-launch floor: the smallest possible GEMM (one 128x64 tile, one k-block)
    for epi in (0, 2):
        us, _, _ = time_cfg(128, 64, 64, epi, 64, 1, -1)
        print(json.dumps({"M": 128, "gemm": f"floor_epi{epi}", "bn": 64, "splits": 1, "lean": -1,
                          "us": round(us, 2)}), flush=True)
    Ms = {"c2": [128], "c4": [16384], "both": [128, 16384]}[which]
    for M in Ms:
        for name, (m, n, k, epi) in shapes(M).items():
            if M <= 512:
                cfgs = [(0, 0, 0)] + [(bn, sp, ln) for bn, sp, ln in
                                      itertools.product([64, 128], [1, 2, 3, 4, 6, 8, -3], [1, -1])]
            else:
                cfgs = [(0, 0, 0)] + [(bn, 1, ln) for bn in (128, 256) for ln in (-2, 2)]
            for bn, sp, ln in cfgs:
                if name == "head" and sp not in (0, 1):
                    continue
                try:
                    us, tf, gbs = time_cfg(m, n, k, epi, bn, sp, ln)
                    print(json.dumps({"M": m, "gemm": name, "bn": bn, "splits": sp, "lean": ln,
                                      "us": round(us, 2), "tflops": round(tf, 1),
                                      "gbs": round(gbs, 1)}), flush=True)
                except Exception as e:  # noqa: BLE001
                    print(json.dumps({"M": m, "gemm": name, "bn": bn, "splits": sp, "lean": ln,
                                      "error": str(e)[:200]}), flush=True)


if __name__ == "__main__":
    main()
