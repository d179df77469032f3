#!/usr/bin/env python3
"""One C3 point: BERT-base (or CFG) hybrid forward at B x S, device time per forward
(CUDA events around 50 back-to-back forward_device calls, p50 of 5 repeats), fp32 logits
as in scripts/sweep_c3.py.  Env: B, S, CFG, POLICY, OUT (f32 | f16)."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2603_28708_b200 as pg  # noqa: E402

cfg = pg.ModelConfig.preset(os.environ.get("CFG", "bert_base"))
B, S = int(os.environ.get("B", 2)), int(os.environ.get("S", 128))
pol = os.environ.get("POLICY", "hybrid")
m = pg.DeviceModel(cfg, pg.build_model(cfg))
ids = torch.from_numpy(pg.random_tokens(cfg.vocab, B, S, 11)).cuda()
f16 = os.environ.get("OUT", "f32") == "f16"
ld = (cfg.vocab + 7) // 8 * 8 if f16 else int(os.environ.get("LD32", (cfg.vocab + 3) // 4 * 4))
out = torch.empty(B * S, ld, device="cuda", dtype=torch.float16 if f16 else torch.float32)
st = torch.cuda.current_stream()
run = lambda: m.forward_device(ids.data_ptr(), B, S, pol, out.data_ptr(), pg.OUT_F16 if f16 else pg.OUT_F32, ld, st.cuda_stream, True)
for _ in range(5):
    run()
torch.cuda.synchronize()
ts = []
for _ in range(5):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for _ in range(50):
        run()
    e1.record(st)
    torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1) / 50)
print(json.dumps({"cfg": cfg.name if hasattr(cfg, "name") else os.environ.get("CFG", "bert_base"), "B": B, "S": S,
                  "policy": pol, "out": "f16" if f16 else "f32", "ms_p50": round(sorted(ts)[2], 4), "ms_min": round(min(ts), 4)}))
