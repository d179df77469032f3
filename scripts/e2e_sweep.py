"""Time the drop-in host forward (prlab_gpu_forward: host ids -> host fp32 logits) for
GPT-2 small at batch 1 x seq 128, as bench.py's e2e leg does; prints ms per call.
Run under different PRLAB_WIDEN_* / PRLAB_NO_HOST_WIDEN settings to tune the copy-out."""
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2603_28708_b200 as pg  # noqa: E402

cfg = pg.ModelConfig.preset("gpt2_small")
m = pg.DeviceModel(cfg, pg.build_model(cfg))
B, S = 1, 128
ids = torch.from_numpy(pg.random_tokens(cfg.vocab, B, S, 3)).pin_memory().numpy()
out = torch.empty((B, S, cfg.vocab), dtype=torch.float32).pin_memory().numpy()
f = pg.lib().prlab_gpu_forward
pol = pg._policy("hybrid")
import ctypes as C
for _ in range(5):
    pg._check(f(m._h, ids.ctypes.data_as(C.POINTER(C.c_int32)), B, S, C.byref(pol), out.ctypes.data_as(C.POINTER(C.c_float)), None))
ts = []
for _ in range(40):
    t0 = time.perf_counter()
    pg._check(f(m._h, ids.ctypes.data_as(C.POINTER(C.c_int32)), B, S, C.byref(pol), out.ctypes.data_as(C.POINTER(C.c_float)), None))
    ts.append(time.perf_counter() - t0)
ts = np.array(ts) * 1e3
print(json.dumps({"env": {k: v for k, v in os.environ.items() if k.startswith("PRLAB_")}, "ms_median": round(float(np.median(ts)), 3),
                  "ms_min": round(float(ts.min()), 3)}))
