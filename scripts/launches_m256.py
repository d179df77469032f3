#!/usr/bin/env python3
"""One forward at a given (model, B, S), launched a few times: for an ncu launch list."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2603_28708_b200 as pg  # noqa: E402

name, B, S = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
cfg = pg.ModelConfig.preset(name)
m = pg.DeviceModel(cfg, pg.build_model(cfg))
ids = torch.from_numpy(pg.random_tokens(cfg.vocab, B, S, 5)).cuda()
ld = (cfg.vocab + 7) // 8 * 8
POL = os.environ.get("POLICY", "hybrid")
OUTT = pg.OUT_F16 if POL == "hybrid" else pg.OUT_F32
out = torch.empty(B * S, ld, device="cuda", dtype=torch.float16 if POL == "hybrid" else torch.float32)
st = torch.cuda.current_stream().cuda_stream
for _ in range(int(os.environ.get("REPS", 3))):
    m.forward_device(ids.data_ptr(), B, S, POL, out.data_ptr(), OUTT, ld, st, os.environ.get("GRAPH", "1") == "1")
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(20):
    m.forward_device(ids.data_ptr(), B, S, POL, out.data_ptr(), OUTT, ld, st, True)
e1.record()
torch.cuda.synchronize()
print({"model": name, "B": B, "S": S, "policy": POL, "ms": e0.elapsed_time(e1) / 20})
