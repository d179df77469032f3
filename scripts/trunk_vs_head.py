#!/usr/bin/env python3
"""Batch-1 step split: the persistent trunk alone (forward_trunk_device) against the whole
forward (trunk + LM head), CUDA events over 200 launches each.  Env: CFG, B, S."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2603_28708_b200 as pg  # noqa: E402

cfg = pg.ModelConfig.preset(os.environ.get("CFG", "gpt2_small"))
B, S = int(os.environ.get("B", 1)), int(os.environ.get("S", 128))
m = pg.DeviceModel(cfg, pg.build_model(cfg))
ids = torch.from_numpy(pg.random_tokens(cfg.vocab, B, S, 3)).cuda()
ld = (cfg.vocab + 7) // 8 * 8
out = torch.empty(B * S, ld, device="cuda", dtype=torch.float16)
st = torch.cuda.current_stream().cuda_stream


def timed(fn, n=200):
    for _ in range(10):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n * 1000


full = timed(lambda: m.forward_device(ids.data_ptr(), B, S, "hybrid", out.data_ptr(), pg.OUT_F16, ld, st, True))
trunk = timed(lambda: m.forward_trunk_device(ids.data_ptr(), B, S, "hybrid", st))
print(json.dumps({"B": B, "S": S, "forward_us": round(full, 1), "trunk_us": round(trunk, 1),
                  "head_and_gaps_us": round(full - trunk, 1)}))
