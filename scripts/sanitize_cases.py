#!/usr/bin/env python3
"""Small invocations of every hand-rolled device protocol, for compute-sanitizer
(memcheck / racecheck / synccheck; scripts/gpu_r2b.sh):
  * tcgen05 GEMMs: one-CTA (TMA ring + TMEM double buffer), CTA pair (cta_group::2,
    multicast commits), cluster split-K (DSMEM reduction), every epilogue;
  * attention: exact two-pass (attn_tc) and streaming (attn_fa) kernels, causal and not;
  * the batch-1 persistent kernel (grid barrier, per-stage TMA/MMA protocol), its CTA-pair
    variant (128 < B*S <= 256: cta_group::2 tasks, remote arrivals, multicast commits) and the
    multi-kernel forward (PDL chain) through the drop-in forward, hybrid and full_fp16;
  * the fp32 policy: 3xTF32 GEMMs (converter warps, split-K reduce) and the tiled attention."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2603_28708_b200 as pg  # noqa: E402

dev = "cuda"
g = torch.Generator(device=dev).manual_seed(0)
st = torch.cuda.current_stream().cuda_stream
for (M, N, K) in [(128, 256, 768), (512, 768, 768), (128, 768, 3072), (300, 200, 192)]:
    A = (torch.randn(M, K, device=dev, generator=g) * 0.5).half()
    W = (torch.randn(N, K, device=dev, generator=g) * 0.05).half()
    b = torch.randn(N, device=dev, generator=g) * 0.1
    o16 = torch.empty(M, (N + 7) // 8 * 8, device=dev, dtype=torch.float16)
    o32 = torch.zeros(M, N, device=dev)
    for epi in (0, 1, 3):
        pg.linear_f16_device(A, W, b if epi != 3 else None, o16, M, N, K, o16.shape[1], epi, st)
    pg.linear_f16_device(A, W, b, o32, M, N, K, N, 2, st)
    torch.cuda.synchronize()
    print("gemm", M, N, K, "ok", flush=True)
for (B, S, causal) in [(1, 128, 1), (2, 96, 0), (1, 256, 1), (1, 384, 0)]:
    H, hd = 12, 64
    qkv = torch.randn(B * S, 3 * H * hd, device=dev, generator=g).half()
    ctx = torch.empty(B * S, H * hd, device=dev, dtype=torch.float16)
    pg.attention_f16_device(qkv, ctx, B, S, H, hd, causal, st)
    torch.cuda.synchronize()
    print("attention", B, S, causal, "ok", flush=True)
cfg = pg.ModelConfig.preset("gpt2_small").replace(num_layers=2, vocab=4096)
m = pg.DeviceModel(cfg, pg.build_model(cfg))
for (B, S) in [(1, 64), (2, 96), (2, 160)]:
    ids = pg.random_tokens(cfg.vocab, B, S, 3)
    for pol in ("hybrid", "full_fp16", "fp32"):
        out = m.forward(ids, B, S, pol)
        assert np.isfinite(out).all()
    print("forward", B, S, "ok", flush=True)
m.close()
print("sanitize cases done")
