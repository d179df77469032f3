#!/usr/bin/env python3
"""Phase timeline of the cluster batch-1 trunk (fwd_cluster.cu) at C2: %globaltimer stamps
of CTA 0 and CTA 15 of every cluster per layer (prlab_gpu_debug_cluster_stamps)."""
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2603_28708_b200 as pg  # noqa: E402
import ctypes as C  # noqa: E402

os.environ["PRLAB_FWD_CLUSTER"] = "1"  # the cluster kernel is opt-in

name = os.environ.get("CL_MODEL", "gpt2_small")
B, S = int(os.environ.get("CL_B", "1")), int(os.environ.get("CL_S", "128"))
cfg = pg.ModelConfig.preset(name)
m = pg.DeviceModel(cfg, pg.build_model(cfg))
L = cfg.num_layers
ids = torch.from_numpy(pg.random_tokens(cfg.vocab, B, S, 1234)).cuda()
st = torch.cuda.current_stream().cuda_stream
dbg = torch.zeros(4 * 2 * L * 16, dtype=torch.int64, device="cuda")
for _ in range(5):
    m.forward_trunk_device(ids.data_ptr(), B, S, "hybrid", st)
pg.lib().prlab_gpu_debug_cluster_stamps(C.c_void_p(dbg.data_ptr()))
m.forward_trunk_device(ids.data_ptr(), B, S, "hybrid", st)
torch.cuda.synchronize()
pg.lib().prlab_gpu_debug_cluster_stamps(None)
d = dbg.cpu().numpy().reshape(4, 2, L, 16).astype(np.float64)
names = ["start", "ln1", "qkv_acc", "kv_pub", "flags", "attn_done", "ctx_sync", "wo_acc", "x_sync",
         "ln2", "ffn1_acc", "ffn2_acc", "part_st", "part_sync", "reduce", "wait_cyc"]
nclus = (B * S + 31) // 32
t0 = d[:nclus, :, 0, 0].min()
for r in range(nclus):
    for k in range(2):
        for l in range(L):
            row = d[r, k, l]
            rel = {names[i]: round((row[i] - t0) / 1000.0, 2) for i in range(15) if row[i] > 0}
            print(json.dumps({"cluster": r, "cta": [0, 15][k], "layer": l, "us": rel,
                              "mma_wait_kcyc": round(row[15] / 1000.0, 1)}))
# per-phase durations averaged over layers (cluster 0, CTA 0)
row = d[0, 0]
dur = {}
for i in range(1, 15):
    v = row[:, i] - row[:, i - 1]
    ok = (row[:, i] > 0) & (row[:, i - 1] > 0)
    if ok.any():
        dur[f"{names[i-1]}->{names[i]}"] = round(float(v[ok].mean()) / 1000.0, 2)
print(json.dumps({"avg_phase_us_cluster0_cta0": dur,
                  "layer_us": round(float(np.diff(row[:, 0]).mean()) / 1000.0, 2)}))
