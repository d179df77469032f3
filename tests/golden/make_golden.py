#!/usr/bin/env python3
"""Generate tests/golden/ fixtures by running the REFERENCE itself.

The reference sources under /root/reference/proj/src are compiled unmodified by
oracle/Makefile into oracle/_ref/libprlab_ref.so; this script calls that library
(prlab::build_model, random_tokens, forward, the per-op kernels) and stores
small, size-bounded fixtures:

  toy_logits.npz     full logits of decoder_toy / encoder_toy, 3 policies, (B=2, S=16)
  preset_rows.npz    GPT-2 / BERT-base presets, batch 1, seq 32, fp32 + hybrid:
                     per-position argmax, max, sum (float64) and 2048 sampled entries
  ops.npz            per-operator outputs on seeded inputs (matmul / softmax /
                     layernorm / gelu / scores / embed) for every kernel config
  meta.json          configs, seeds, param counts, kernel_calls traces

Run (where /root/reference exists): python tests/golden/make_golden.py
"""
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
from oracle.oracle import PRESETS, Reference  # noqa: E402

POLICIES = ["fp32", "hybrid", "full_fp16"]
CFGS = [(0, 0), (1, 0), (0, 1), (1, 1)]  # (compute, accum) incl. invalid (0,1) skipped


def main():
    ref = Reference()
    meta = {"generator": "tests/golden/make_golden.py", "reference_lib": "oracle/_ref/libprlab_ref.so"}

    # ---- toy models, full logits
    toy = {}
    meta["toy"] = {}
    for name in ["decoder_toy", "encoder_toy"]:
        cfg = PRESETS[name].replace(seed=3)
        params = ref.build_model(cfg)
        ids = ref.random_tokens(cfg.vocab, 2, 16, 9)
        toy[f"{name}_ids"] = ids
        toy[f"{name}_param_sum"] = np.array([params.astype(np.float64).sum()])
        meta["toy"][name] = {"config": cfg.__dict__, "batch": 2, "seq": 16, "token_seed": 9,
                             "param_count": int(params.size)}
        for pol in POLICIES:
            logits, calls = ref.forward(cfg, params, ids, 2, 16, pol, want_calls=True)
            toy[f"{name}_{pol}"] = logits
            meta["toy"][name][f"calls_{pol}"] = calls.tolist()
    np.savez_compressed(os.path.join(HERE, "toy_logits.npz"), **toy)

    # ---- presets: bounded row statistics + sampled entries
    rows = {}
    meta["presets"] = {}
    rng = np.random.default_rng(2026)
    for name in ["gpt2_small", "bert_base"]:
        cfg = PRESETS[name]
        params = ref.build_model(cfg)
        ids = ref.random_tokens(cfg.vocab, 1, 32, 1234)
        rows[f"{name}_ids"] = ids
        rows[f"{name}_param_sum"] = np.array([params.astype(np.float64).sum()])
        idx = rng.integers(0, 32 * cfg.vocab, 2048)
        rows[f"{name}_sample_idx"] = idx
        meta["presets"][name] = {"config": cfg.__dict__, "batch": 1, "seq": 32, "token_seed": 1234,
                                 "param_count": int(params.size)}
        for pol in ["fp32", "hybrid"]:
            lg = ref.forward(cfg, params, ids, 1, 32, pol, threads=8).reshape(32, cfg.vocab)
            rows[f"{name}_{pol}_argmax"] = lg.argmax(1)
            rows[f"{name}_{pol}_max"] = lg.max(1)
            rows[f"{name}_{pol}_sum"] = lg.astype(np.float64).sum(1)
            rows[f"{name}_{pol}_sample"] = lg.ravel()[idx]
            top2 = np.sort(lg, 1)[:, -2:]
            rows[f"{name}_{pol}_gap"] = top2[:, 1] - top2[:, 0]
    np.savez_compressed(os.path.join(HERE, "preset_rows.npz"), **rows)

    # ---- per-operator outputs
    ops = {}
    r = np.random.default_rng(7)
    a = r.uniform(-1, 1, (17, 33)).astype(np.float32)
    b = r.uniform(-1, 1, (33, 9)).astype(np.float32)
    x = r.uniform(-6, 6, (8, 40)).astype(np.float32)
    xl = r.normal(0, 2, (6, 64)).astype(np.float32)
    g = r.normal(1, 0.1, 64).astype(np.float32)
    be = r.normal(0, 0.1, 64).astype(np.float32)
    q = r.normal(0, 1, (5, 16)).astype(np.float32)
    k = r.normal(0, 1, (7, 16)).astype(np.float32)
    xg = r.uniform(-5, 5, 1000).astype(np.float32)
    ops.update(a=a, b=b, x=x, xl=xl, g=g, be=be, q=q, k=k, xg=xg)
    for c, ac in [(0, 0), (1, 0), (1, 1)]:
        ops[f"matmul_{c}{ac}"] = ref.matmul(a, b, c, ac)
        ops[f"layernorm_{c}{ac}"] = ref.layernorm(xl, g, be, 1e-5, c, ac)
        ops[f"gelu_{c}{ac}"] = ref.gelu(xg, c, ac)
        s, tap = ref.attention_scores(q, k, 0.25, c, ac, capture=True)
        ops[f"scores_{c}{ac}"] = s
        ops[f"scores_tap_{c}{ac}"] = tap
        for st in (0, 1):
            ops[f"softmax_{c}{ac}{st}"] = ref.softmax(x, c, ac, bool(st))
    tok = r.normal(0, 1, (50, 12)).astype(np.float32)
    pos = r.normal(0, 1, (10, 12)).astype(np.float32)
    eids = r.integers(0, 50, 3 * 10).astype(np.int32)
    ops.update(tok=tok, pos=pos, eids=eids)
    for c in (0, 1):
        ops[f"embed_{c}"] = ref.embed(tok, pos, eids, 3, 10, c)
    np.savez_compressed(os.path.join(HERE, "ops.npz"), **ops)

    with open(os.path.join(HERE, "meta.json"), "w") as f:
        json.dump(meta, f, indent=1)
    print("golden fixtures written to", HERE)


if __name__ == "__main__":
    main()
