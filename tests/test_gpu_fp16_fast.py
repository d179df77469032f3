"""full_fp16 on the tensor cores -- the speed arm of the C5 precision ablation
(BASELINE.json configs[4]; reference policy src/policy.cpp:18,55: every op class
{F16E, F16E, unstabilised}).

The fast path keeps every op output and the residual stream on the binary16 lattice,
accumulates the GEMMs in FP16 TMEM accumulators (rounded once per 16-wide MMA step, not
after every product as the reference's emulation does, src/kernels.cpp:56-66) and runs
the softmax unstabilised (kernels.cpp:155).  The exact per-MAC emulation remains behind
PRLAB_FP16_EXACT=1 and reproduces the reference's known-answer tests (test_gpu_kernels,
test_gpu_forward toy cases).  Bars: finite on random weights, closer to fp32 than the
reference's own full_fp16 (cosine 0.99988 BERT / 0.99990 GPT-2 at s512),
NaN on the adversarial models exactly like the reference (tests/test_gpu_sweep.py).
"""
import json
import os

import numpy as np
import pytest

import paper_2603_28708_b200 as pg
from oracle.oracle import PRESETS, compare_logits
from prlab_testutil import model_params, oracle

pytestmark = pytest.mark.gpu
_MODELS = {}


def device_model(cfg):
    if cfg not in _MODELS:
        _MODELS[cfg] = pg.DeviceModel(pg.ModelConfig(**cfg.__dict__), model_params(cfg))
    return _MODELS[cfg]


def report(**kw):
    path = os.environ.get("PRLAB_PARITY_REPORT")
    if path:
        with open(path, "a") as f:
            f.write(json.dumps(kw) + "\n")


@pytest.mark.parametrize("name,S", [("bert_base", 512), ("gpt2_small", 512), ("gpt2_small", 128)])
def test_full_fp16_fast_vs_cpu(name, S):
    cfg = PRESETS[name]
    o = oracle()
    m = device_model(cfg)
    p = model_params(cfg)
    ids = o.random_tokens(cfg.vocab, 1, S, 77)
    fast = m.forward(ids, 1, S, "full_fp16")
    assert m.kernel_count(1, S, "full_fp16") > 2  # tensor-core multi-kernel path, not the SIMT emulator
    cpu32 = o.forward(cfg, p, ids, 1, S, "fp32")
    r32 = compare_logits(cpu32, fast)
    rec = {"test": "full_fp16_fast", "model": name, "S": S, "vs_cpu_fp32": r32}
    if S <= 128:  # the CPU per-MAC emulation is ~80 s per forward single-threaded at s128
        cpuf = o.forward(cfg, p, ids, 1, S, "full_fp16")
        rec["vs_cpu_full_fp16"] = compare_logits(cpuf, fast)
        rec["cpu_full_fp16_vs_cpu_fp32"] = compare_logits(cpu32, cpuf)
    report(**rec)
    assert r32["candidate_nonfinite"] == 0
    assert r32["cosine"] >= 0.9998, r32
    # rounding points are every op output: hybrid stays closer to fp32 than full_fp16
    rh = compare_logits(cpu32, m.forward(ids, 1, S, "hybrid"))
    assert rh["cosine"] >= r32["cosine"]


def test_full_fp16_exact_switch(monkeypatch):
    """PRLAB_FP16_EXACT=1 selects the per-MAC emulation (kernel_count of the SIMT path)."""
    cfg = PRESETS["gpt2_small"].replace(num_layers=2)
    m = pg.DeviceModel(pg.ModelConfig(**cfg.__dict__), oracle().build_model(cfg))
    fast_k = m.kernel_count(1, 64, "full_fp16")
    monkeypatch.setenv("PRLAB_FP16_EXACT", "1")
    exact_k = m.kernel_count(1, 64, "full_fp16")
    ids = oracle().random_tokens(cfg.vocab, 1, 64, 5)
    exact = m.forward(ids, 1, 64, "full_fp16")
    want = oracle().forward(cfg, oracle().build_model(cfg), ids, 1, 64, "full_fp16")
    monkeypatch.delenv("PRLAB_FP16_EXACT")
    fast = m.forward(ids, 1, 64, "full_fp16")
    m.close()
    assert fast_k == 1 + 7 * 2 + 2 and exact_k == 1 + 7 * 2 + 2  # same op graph, different kernels
    assert np.abs(exact - want).max() < 5e-2
    r = compare_logits(want, fast)
    report(test="full_fp16_fast_vs_exact", model="gpt2_2layer", S=64, **r)
    assert r["candidate_nonfinite"] == 0 and r["cosine"] >= 0.9995
