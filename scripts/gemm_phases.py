#!/usr/bin/env python3
"""%globaltimer phase stamps of the cluster split-K GEMM at batch-1 shapes."""
import ctypes as C
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2603_28708_b200 as pg  # noqa: E402

H, F = 768, 3072
SHAPES = {"qkv": (128, 3 * H, H, 0), "wo": (128, H, H, 2), "ffn1": (128, F, H, 1), "ffn2": (128, H, F, 2)}


def main():
    dbg = torch.zeros(4096, 8, dtype=torch.int64, device="cuda")
    for name, (M, N, K, epi) in SHAPES.items():
        A = (torch.randn(M, K, device="cuda") * 0.5).half()
        W = (torch.randn(N, K, device="cuda") * 0.02).half()
        bias = torch.zeros(N, device="cuda")
        out = torch.zeros(M, N, device="cuda", dtype=torch.float32 if epi == 2 else torch.float16)
        for _ in range(3):
            pg.linear_f16_device(A, W, bias, out, M, N, K, N, epi)
        torch.cuda.synchronize()
        dbg.zero_()
        pg._check(pg.lib().prlab_gpu_debug_gemm_stamps(C.c_void_p(dbg.data_ptr())))
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        pg.linear_f16_device(A, W, bias, out, M, N, K, N, epi)
        e1.record()
        torch.cuda.synchronize()
        pg._check(pg.lib().prlab_gpu_debug_gemm_stamps(None))
        d = dbg.cpu().double()
        used = d[:, 0] > 0
        d = d[used]
        t0 = d[:, 0].min()
        rel = (d - t0) / 1000.0  # us from the first CTA start
        names = ["start", "setup", "after_pdl_wait", "acc_ready", "partial_written", "cluster_sync1", "reduced", "end"]
        out_d = {"gemm": name, "ctas": int(used.sum()), "event_us": round(e0.elapsed_time(e1) * 1000, 2)}
        for i, n in enumerate(names):
            out_d[n] = [round(float(rel[:, i].min()), 2), round(float(rel[:, i].mean()), 2), round(float(rel[:, i].max()), 2)]
        print(json.dumps(out_d), flush=True)


if __name__ == "__main__":
    main()
