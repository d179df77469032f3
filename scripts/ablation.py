#!/usr/bin/env python3
"""C5 precision ablation on the B200: fp32 vs full_fp16 (tensor-core fast path and the exact
per-MAC emulation) vs hybrid at seq 512 for
BERT-base and GPT-2 -- device latency (CUDA-graph replay, p50), fidelity against the
GPU fp32 forward (cosine / max abs), and the NaN rate over adversarial models
(make_adversarial_model restated in oracle/, target max score 30, 5 seeds).
Writes one JSON line per (model, policy) to stdout."""
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2603_28708_b200 as pg  # noqa: E402
from oracle.oracle import ModelConfig as OC, Oracle, compare_logits, make_adversarial_params  # noqa: E402


def p50(xs):
    s = sorted(xs)
    return s[max(1, (len(s) + 1) // 2) - 1]


def time_policy(model, cfg, B, S, policy, reps=10):
    ids = torch.from_numpy(pg.random_tokens(cfg.vocab, B, S, 1234)).cuda()
    out = torch.empty(B * S, cfg.vocab, device="cuda", dtype=torch.float32)
    st = torch.cuda.current_stream().cuda_stream
    for _ in range(2):
        model.forward_device(ids.data_ptr(), B, S, policy, out.data_ptr(), pg.OUT_F32, cfg.vocab, st, True)
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        model.forward_device(ids.data_ptr(), B, S, policy, out.data_ptr(), pg.OUT_F32, cfg.vocab, st, True)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return p50(ts)


def main():
    S = int(os.environ.get("ABL_SEQ", "512"))
    o = Oracle()
    for name in ["bert_base", "gpt2_small"]:
        cfg = pg.ModelConfig.preset(name)
        params = pg.build_model(cfg)
        model = pg.DeviceModel(cfg, params)
        ids = pg.random_tokens(cfg.vocab, 1, S, 77)
        base = model.forward(ids, 1, S, "fp32")
        # adversarial NaN rate: 5 seeds (acceptance_main.cpp:47 uses target 30)
        small = OC(**cfg.replace(num_layers=2).__dict__)
        adv_nan = {"fp32": 0, "full_fp16": 0, "hybrid": 0}
        for seed in range(5):
            c = small.replace(seed=seed)
            probe = o.random_tokens(c.vocab, 1, 32, 100 + seed)
            adv = make_adversarial_params(o, c, probe, 1, 32, 30.0)
            am = pg.DeviceModel(pg.ModelConfig(**c.__dict__), adv)
            for pol in adv_nan:
                adv_nan[pol] += int(not np.isfinite(am.forward(probe, 1, 32, pol)).all())
            am.close()
        for pol, exact in [("fp32", 0), ("full_fp16", 0), ("full_fp16", 1), ("hybrid", 0)]:
            # full_fp16: tensor-core FP16 accumulators (default) or the exact per-MAC emulation
            os.environ["PRLAB_FP16_EXACT"] = str(exact)
            ms = time_policy(model, cfg, 1, S, pol)
            got = model.forward(ids, 1, S, pol)
            r = compare_logits(base, got)
            tag = pol + ("_exact_emulation" if exact else "")
            print(json.dumps({"model": name, "seq": S, "batch": 1, "policy": tag, "p50_ms": round(ms, 4),
                              "kernels": model.kernel_count(1, S, pol),
                              "cosine_vs_gpu_fp32": r["cosine"], "max_abs_vs_gpu_fp32": r["max_abs_error"],
                              "nonfinite": r["candidate_nonfinite"],
                              "adversarial_nan_rate": adv_nan[pol] / 5.0 if not exact else None}), flush=True)
        os.environ.pop("PRLAB_FP16_EXACT", None)
        model.close()


if __name__ == "__main__":
    main()
