#!/usr/bin/env python3
"""Quick check of the cluster batch-1 trunk (fwd_cluster.cu) on the GPU: parity vs the CPU
oracle (hybrid) and vs the one-CTA-per-SM trunk (fwd_small, the default; the cluster kernel is opt-in, PRLAB_FWD_CLUSTER=1) on
several (model, B, S), then device time of the C2 forward with each trunk."""
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2603_28708_b200 as pg  # noqa: E402
from oracle.oracle import PRESETS, Oracle, compare_logits  # noqa: E402

o = Oracle()
cases = [("gpt2_small", 1, 128), ("bert_base", 1, 128), ("gpt2_small", 4, 32), ("gpt2_small", 2, 48),
         ("bert_base", 3, 40), ("gpt2_small", 1, 100), ("gpt2_small", 1, 7)]
models = {}
for name, B, S in cases:
    cfg = PRESETS[name]
    if name not in models:
        models[name] = (pg.DeviceModel(pg.ModelConfig(**cfg.__dict__), o.build_model(cfg)), o.build_model(cfg))
    m, p = models[name]
    ids = o.random_tokens(cfg.vocab, B, S, 1234)
    os.environ["PRLAB_FWD_CLUSTER"] = "1"
    try:
        got = m.forward(ids, B, S, "hybrid")
    except Exception as e:
        print(json.dumps({"case": [name, B, S], "error": str(e)}), flush=True)
        continue
    cpuh = o.forward(cfg, p, ids, B, S, "hybrid")
    r = compare_logits(cpuh, got)
    print(json.dumps({"case": [name, B, S], "vs_cpu_hybrid": r}), flush=True)
# timing: C2 forward (trunk + head) with each trunk
cfg = PRESETS["gpt2_small"]
m, p = models["gpt2_small"]
for trunk in ("cluster", "small"):
    if trunk == "small":
        os.environ["PRLAB_FWD_CLUSTER"] = "0"
    m2 = pg.DeviceModel(pg.ModelConfig(**cfg.__dict__), p)
    ids = torch.from_numpy(o.random_tokens(cfg.vocab, 1, 128, 1234)).cuda()
    ld = (cfg.vocab + 7) // 8 * 8
    out = torch.empty(128, ld, dtype=torch.float16, device="cuda")
    st = torch.cuda.current_stream().cuda_stream
    for _ in range(10):
        m2.forward_device(ids.data_ptr(), 1, 128, "hybrid", out.data_ptr(), pg.OUT_F16, ld, st, True)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(50):
        m2.forward_device(ids.data_ptr(), 1, 128, "hybrid", out.data_ptr(), pg.OUT_F16, ld, st, True)
    e1.record()
    torch.cuda.synchronize()
    # trunk alone
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0.record()
    for _ in range(50):
        m2.forward_trunk_device(ids.data_ptr(), 1, 128, "hybrid", st)
    t1.record()
    torch.cuda.synchronize()
    m2.sync_status(st)
    print(json.dumps({"trunk": trunk, "forward_ms": e0.elapsed_time(e1) / 50, "trunk_ms": t0.elapsed_time(t1) / 50}),
          flush=True)
    m2.close()
