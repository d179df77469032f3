#!/usr/bin/env python3
"""Per-stage timeline of the batch-1 persistent forward (fwd_small.cu): for every stage,
the stage's work time (last CTA arriving at the barrier minus the previous release) and
the barrier latency (release minus last arrival), from %globaltimer stamps."""
import ctypes as C
import json
import os
import sys

import numpy as np
import torch

# the stage timeline needs a grid barrier at every stage boundary (the default trunk hands
# QKV -> attention -> RLN2 and FFN1 -> FFN2 over per-task flags instead)
os.environ.setdefault("PRLAB_SMALL_BARRIERS", "1")

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2603_28708_b200 as pg  # noqa: E402

NAMES = ["qkv", "attn+wo", "rln2", "ffn1", "ffn2", "rln1"]
PER = len(NAMES)  # stages per layer


def main():
    cfg = pg.ModelConfig.preset(sys.argv[1] if len(sys.argv) > 1 else "gpt2_small")
    B, S = int(os.environ.get("B", 1)), int(os.environ.get("S", 128))
    m = pg.DeviceModel(cfg, pg.build_model(cfg))
    ids = torch.from_numpy(pg.random_tokens(cfg.vocab, B, S, 3)).cuda()
    V = cfg.vocab
    ld = (V + 7) // 8 * 8
    out = torch.empty(B * S, ld, device="cuda", dtype=torch.float16)
    st = torch.cuda.current_stream().cuda_stream
    for _ in range(3):
        m.forward_device(ids.data_ptr(), B, S, "hybrid", out.data_ptr(), pg.OUT_F16, ld, st, False)
    torch.cuda.synchronize()
    nst = 1 + PER * cfg.num_layers
    dbg = torch.zeros(300000, dtype=torch.int64, device="cuda")
    pg._check(pg.lib().prlab_gpu_debug_small_stamps(C.c_void_p(dbg.data_ptr())))
    m.forward_device(ids.data_ptr(), B, S, "hybrid", out.data_ptr(), pg.OUT_F16, ld, st, False)
    torch.cuda.synchronize()
    pg._check(pg.lib().prlab_gpu_debug_small_stamps(None))
    raw = dbg.cpu().numpy().astype(np.float64)
    d = raw[: nst * 148 * 2].reshape(nst, 148, 2)  # (the pair grid is 148 CTAs too)
    rl = raw[200000:200000 + 8 * cfg.num_layers].reshape(cfg.num_layers, 8)
    arrive_max = d[:, :, 0].max(1)
    release_min = np.where(d[:, :, 1] > 0, d[:, :, 1], np.inf).min(1)
    release_max = d[:, :, 1].max(1)
    t0 = d[0, :, 0].min()
    prev_release = t0
    rows = []
    for k in range(nst - 1):
        name = "embed+ln1" if k == 0 else NAMES[(k - 1) % PER]
        rows.append({"stage": k, "name": name, "work_us": round((arrive_max[k] - prev_release) / 1e3, 2),
                     "barrier_us": round((release_max[k] - arrive_max[k]) / 1e3, 2)})
        prev_release = release_max[k]
    agg = {}
    for r in rows:
        a = agg.setdefault(r["name"], [0.0, 0.0, 0])
        a[0] += r["work_us"]
        a[1] += r["barrier_us"]
        a[2] += 1
    print(json.dumps({"total_us": round((release_max[nst - 2] - t0) / 1e3, 1),
                      "per_stage_type": {k: {"n": v[2], "work_us_avg": round(v[0] / v[2], 2),
                                             "barrier_us_avg": round(v[1] / v[2], 2)} for k, v in agg.items()}}))
    for r in rows[:9]:
        print(json.dumps(r))
    # per-CTA arrival spread inside each stage type (layers 1..L-1: warm L2), relative to
    # the previous barrier's last release: who is late, and by how much
    spread = {}
    for k in range(1 + PER, nst - 1):
        name = NAMES[(k - 1) % PER]
        arr = (d[k, :, 0] - release_max[k - 1]) / 1e3
        active = arr[arr > -1e3]
        spread.setdefault(name, []).append((np.percentile(active, 10), np.median(active), active.max(),
                                            int(np.argmax(arr))))
    print(json.dumps({"arrival_spread_us": {n: {"p10": round(float(np.mean([v[0] for v in vs])), 2),
                                                "median": round(float(np.mean([v[1] for v in vs])), 2),
                                                "max": round(float(np.mean([v[2] for v in vs])), 2),
                                                "latest_cta": [v[3] for v in vs][:6]}
                                            for n, vs in spread.items()}}))
    at = raw[210000:210000 + 8 * cfg.num_layers].reshape(cfg.num_layers, 8)
    for l in range(min(3, cfg.num_layers)):
        k = 1 + PER * l + 1  # attention stage index
        print(json.dumps({"layer": l, "attn_cta0": {"start_us": round((at[l, 0] - d[k - 1, 0, 1]) / 1e3, 2),
                                                    "tasks_us": round((at[l, 1] - at[l, 0]) / 1e3, 2),
                                                    "to_arrive_us": round((d[k, 0, 0] - at[l, 1]) / 1e3, 2)}}))
    ta = raw[230000:230000 + 8 * cfg.num_layers].reshape(cfg.num_layers, 8)
    for l in range(min(3, cfg.num_layers)):
        k = 1 + PER * l + 1
        t = ta[l]
        if t[0] == 0:
            continue
        print(json.dumps({"layer": l, "attn_task_last_qblock": {
            "start_after_release_us": round((t[0] - d[k - 1, :, 1].max()) / 1e3, 2),
            "stage_us": round((t[1] - t[0]) / 1e3, 2), "scores_us": round((t[2] - t[1]) / 1e3, 2),
            "softmax_us": round((t[3] - t[2]) / 1e3, 2), "softmax_max_us": round((t[7] - t[2]) / 1e3, 2), "pv_us": round((t[4] - t[3]) / 1e3, 2),
            "wo_wait_us": round((t[5] - t[4]) / 1e3, 2), "wo_mma_store_us": round((t[6] - t[5]) / 1e3, 2)}}))
    wt = raw[240000:240000 + 64].reshape(8, 8)  # last layer's task, per warp: clock64
    if wt[0, 0] != 0:
        print(json.dumps({"attn_task_warp_cycles": [
            {"scores": int(w[1] - w[0]), "sync1": int(w[2] - w[1]), "max": int(w[3] - w[2]),
             "exp_sum": int(w[4] - w[3]), "store_p": int(w[5] - w[4]), "sync2": int(w[6] - w[5])} for w in wt]}))
    gt = raw[220000:220000 + 64 * 8].reshape(64, 8)
    names = ["qkv", "ffn1", "ffn2"]
    for t in range(6):
        g = gt[t]
        if g[0] == 0:
            break
        print(json.dumps({"gemm_task_cta0": names[t % 3], "b_ready_us": round((g[1] - g[0]) / 1e3, 2),
                          "first_a_us": round((g[2] - g[0]) / 1e3, 2), "mma_issued_us": round((g[3] - g[0]) / 1e3, 2),
                          "acc_ready_us": round((g[4] - g[0]) / 1e3, 2), "epilogue_done_us": round((g[5] - g[0]) / 1e3, 2)}))
    # CTA 0 inside RLN2 of each layer: release -> start, loads+residual, LN
    for l in range(min(3, cfg.num_layers)):
        k = 1 + PER * l + 2  # the RLN2 stage index
        print(json.dumps({"layer": l, "rln2_cta0": {"start_after_release_us": round((rl[l, 0] - d[k - 1, 0, 1]) / 1e3, 2),
                                                    "loads_us": round((rl[l, 1] - rl[l, 0]) / 1e3, 2),
                                                    "ln_us": round((rl[l, 2] - rl[l, 1]) / 1e3, 2),
                                                    "to_arrive_us": round((d[k, 0, 0] - rl[l, 2]) / 1e3, 2)}}))


if __name__ == "__main__":
    main()
