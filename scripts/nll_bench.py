#!/usr/bin/env python3
"""Forward + per-row NLL/argmax at C4 (GPT-2, B=32, S=512, hybrid): the head's log-softmax
fused into its GEMM epilogue (default) vs logits + row_nll (PRLAB_NO_FUSED_NLL=1), and the
plain logits forward for reference.  CUDA events, one JSON line."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2603_28708_b200 as pg  # noqa: E402

B, S = int(os.environ.get("B", 32)), int(os.environ.get("S", 512))
cfg = pg.ModelConfig.preset("gpt2_small")
m = pg.DeviceModel(cfg, pg.build_model(cfg))
M, V = B * S, cfg.vocab
ids = torch.from_numpy(pg.random_tokens(V, B, S, 3)).cuda()
tg = torch.roll(ids.view(-1), -1).to(torch.int32).contiguous()
nll = torch.empty(M, dtype=torch.float64, device="cuda")
am = torch.empty(M, dtype=torch.int32, device="cuda")
ld = (V + 7) // 8 * 8
logits = torch.empty(M, ld, dtype=torch.float16, device="cuda")
st = torch.cuda.current_stream().cuda_stream


def timed(fn, n=10):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n


fused = []
t_nll = timed(lambda: fused.append(m.forward_nll_device(ids.data_ptr(), tg.data_ptr(), B, S, "hybrid",
                                                        nll.data_ptr(), am.data_ptr(), st)))
t_fwd = timed(lambda: m.forward_device(ids.data_ptr(), B, S, "hybrid", logits.data_ptr(), pg.OUT_F16, ld, st, False))
m.sync_status()
print(json.dumps({"B": B, "S": S, "fused": bool(fused[-1]), "env_no_fused": os.environ.get("PRLAB_NO_FUSED_NLL"),
                  "forward_nll_ms": round(t_nll, 4), "forward_logits_ms": round(t_fwd, 4),
                  "nll_mean": float(nll.mean().item())}))
