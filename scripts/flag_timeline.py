#!/usr/bin/env python3
"""Critical-path timeline of the barrier-free persistent trunk (fwd_small.cu, flag mode):
every CTA stamps the end of each stage; per stage the LAST CTA's end minus the previous
stage's last end (the chain the next stage waits on), and the median CTA's.  Env: CFG, B, S."""
import ctypes as C
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2603_28708_b200 as pg  # noqa: E402

NAMES = ["qkv", "attn+wo", "rln2", "ffn1", "ffn2", "rln1"]
cfg = pg.ModelConfig.preset(os.environ.get("CFG", "gpt2_small"))
B, S = int(os.environ.get("B", 1)), int(os.environ.get("S", 128))
m = pg.DeviceModel(cfg, pg.build_model(cfg))
ids = torch.from_numpy(pg.random_tokens(cfg.vocab, B, S, 3)).cuda()
ld = (cfg.vocab + 7) // 8 * 8
out = torch.empty(B * S, ld, device="cuda", dtype=torch.float16)
st = torch.cuda.current_stream().cuda_stream
for _ in range(3):
    m.forward_device(ids.data_ptr(), B, S, "hybrid", out.data_ptr(), pg.OUT_F16, ld, st, False)
torch.cuda.synchronize()
dbg = torch.zeros(300000, dtype=torch.int64, device="cuda")
pg._check(pg.lib().prlab_gpu_debug_small_stamps(C.c_void_p(dbg.data_ptr())))
m.forward_device(ids.data_ptr(), B, S, "hybrid", out.data_ptr(), pg.OUT_F16, ld, st, False)
torch.cuda.synchronize()
pg._check(pg.lib().prlab_gpu_debug_small_stamps(None))
L, G = cfg.num_layers, 148
d = dbg.cpu().numpy()[250000:250000 + L * 6 * G].astype(np.float64).reshape(L, 6, G)
live = d > 0
t0 = d[live].min()
last = np.where(live, d, -np.inf).max(2)
med = np.array([[np.median(d[l, k][live[l, k]]) for k in range(6)] for l in range(L)])
rows = []
prev = t0
for l in range(L):
    for k in range(6):
        rows.append({"layer": l, "stage": NAMES[k], "last_us": round((last[l, k] - prev) / 1e3, 2),
                     "median_end_after_prev_last_us": round((med[l, k] - prev) / 1e3, 2)})
        prev = last[l, k]
agg = {}
for r in rows:
    agg.setdefault(r["stage"], []).append(r["last_us"])
qw = dbg.cpu().numpy()[262000:262000 + L * G].astype(np.float64).reshape(L, G)
if qw[1].max() > 0:  # QKV CTAs released from the rows wait, after the previous layer's last RLN1 row
    rel = [(qw[l][qw[l] > 0] - last[l - 1, 5]) / 1e3 for l in range(1, L)]
    print(json.dumps({"qkv_wait_release_after_last_rln1_us": {"median": round(float(np.median(np.concatenate(rel))), 2),
                                                               "max": round(float(np.max(np.concatenate(rel))), 2)}}))
fw = dbg.cpu().numpy()[264000:264000 + L * G].astype(np.float64).reshape(L, G)
if fw[1].max() > 0:  # FFN1 CTAs released from the RLN2-rows wait, and their task end (stage 3 stamp)
    rel = np.concatenate([(fw[l][fw[l] > 0] - last[l, 2]) / 1e3 for l in range(1, L)])
    dur = np.concatenate([(d[l, 3][fw[l] > 0] - fw[l][fw[l] > 0]) / 1e3 for l in range(1, L)])
    print(json.dumps({"ffn1_wait_release_after_last_rln2_us": {"median": round(float(np.median(rel)), 2),
                                                                "max": round(float(rel.max()), 2)},
                      "ffn1_task_us": {"median": round(float(np.median(dur)), 2), "p90": round(float(np.percentile(dur, 90)), 2),
                                       "max": round(float(dur.max()), 2)}}))
print(json.dumps({"total_us": round((last[-1, 5] - t0) / 1e3, 1),
                  "per_stage_last_us_avg": {k: round(float(np.mean(v)), 2) for k, v in agg.items()}}))
for r in rows[6:12]:
    print(json.dumps(r))
gt = dbg.cpu().numpy()[220000:220000 + 64 * 8].astype(np.float64).reshape(64, 8)
for t in range(3, 9):  # CTA 0's GEMM tasks of layer 1 (qkv, ffn1, ffn2): phases after the task start
    g = gt[t]
    if g[0] == 0:
        break
    print(json.dumps({"gemm_task_cta0": ["qkv", "ffn1", "ffn2"][t % 3], "b_ready_us": round((g[1] - g[0]) / 1e3, 2),
                      "first_a_us": round((g[2] - g[0]) / 1e3, 2), "mma_issued_us": round((g[3] - g[0]) / 1e3, 2),
                      "acc_ready_us": round((g[4] - g[0]) / 1e3, 2), "epilogue_done_us": round((g[5] - g[0]) / 1e3, 2)}))
