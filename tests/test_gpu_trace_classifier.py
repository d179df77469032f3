"""The drop-in's optional forward outputs and the encoder classifier head on the GPU,
checked against the CPU oracle (bit-identical to the reference: tests/test_oracle_golden.py).

  * retain_scores (src/model.cpp:393-427, kernels.cpp:108-118): per layer [B,H,S,S]
    fp32 pre-mask scaled scores, on the tensor-core path (GPT-2 / BERT head shape) and
    the generic SIMT path; the tap is an fp32 dot product, so the bar is the fp32
    accumulation-order drift (relative 1e-5 of the score range);
  * ForwardTrace.seconds: CUDA-event time per op class (model.cpp:55-62);
  * classifier_probs (model.cpp:484-526): fp32 policy within 1e-5 of the CPU fp32
    probabilities, hybrid within 2e-3 (logit drift of the fp16 lattice); decoder
    models raise invalid_argument like the reference.
"""
import numpy as np
import pytest

import paper_2603_28708_b200 as pg
from oracle.oracle import PRESETS, ModelConfig, compare_logits
from prlab_testutil import model_params, oracle

pytestmark = pytest.mark.gpu

# h = 768, 12 heads of 64 (the tcgen05 attention shape), 2 layers, small vocabulary
GPT2_SMALLV = ModelConfig(archetype=1, num_layers=2, hidden=768, heads=12, ffn=3072, vocab=4096,
                          max_positions=512, seed=0)
BERT_SMALLV = GPT2_SMALLV.replace(archetype=0)
_MODELS = {}


def device_model(cfg):
    if cfg not in _MODELS:
        _MODELS[cfg] = pg.DeviceModel(pg.ModelConfig(**cfg.__dict__), model_params(cfg))
    return _MODELS[cfg]


@pytest.mark.parametrize("cfg", [GPT2_SMALLV, BERT_SMALLV, PRESETS["decoder_toy"]],
                         ids=["gpt2_tc", "bert_tc", "toy_generic"])
@pytest.mark.parametrize("policy", ["hybrid", "fp32"])
@pytest.mark.parametrize("B,S", [(2, 96), (1, 300)])
def test_retain_scores_taps(cfg, policy, B, S):
    if S > cfg.max_positions:
        pytest.skip("sequence longer than the preset's positions")
    o = oracle()
    m = device_model(cfg)
    ids = o.random_tokens(cfg.vocab, B, S, 21)
    p = model_params(cfg)
    want_logits, want_tap = o.forward(cfg, p, ids, B, S, policy, retain_scores=True)
    logits, tr, tap = m.forward_ex(ids, B, S, policy, retain_scores=True)
    assert tap.shape == want_tap.shape == (cfg.num_layers, B, cfg.heads, S, S)
    assert np.isfinite(tap).all()
    scale = float(np.abs(want_tap).max())
    err = float(np.abs(tap.astype(np.float64) - want_tap).max())
    # layer 0 sees identical inputs up to LN/linear drift; later layers inherit it
    assert err <= 2e-2 * scale, (err, scale)
    l0 = float(np.abs(tap[0].astype(np.float64) - want_tap[0]).max())
    assert l0 <= (1e-3 if policy == "hybrid" else 1e-4) * scale, (l0, scale)
    # the logits of the tapped forward still meet the forward bars
    cpu32 = o.forward(cfg, p, ids, B, S, "fp32")
    cmp = compare_logits(cpu32, logits)
    assert cmp["candidate_nonfinite"] == 0 and cmp["cosine"] >= 0.9998


def test_timed_trace_seconds_and_calls():
    cfg = GPT2_SMALLV
    o = oracle()
    m = device_model(cfg)
    ids = o.random_tokens(cfg.vocab, 1, 128, 3)
    _, tr, _ = m.forward_ex(ids, 1, 128, "hybrid", timed=True)
    secs = np.array(tr.seconds[:])
    assert secs[0] > 0 and secs[1] > 0 and secs[3] > 0 and secs[5] > 0  # Linear, AttnMM, LN, Embedding
    _, calls = o.forward(cfg, model_params(cfg), ids, 1, 128, "hybrid", want_calls=True)
    got = np.array([[tr.kernel_calls[c][d] for d in range(2)] for c in range(7)])
    assert (got == calls).all()


@pytest.mark.parametrize("cfg", [BERT_SMALLV, PRESETS["encoder_toy"]], ids=["bert_tc", "toy_generic"])
@pytest.mark.parametrize("B,S", [(3, 48), (1, 128)])
def test_classifier_probs(cfg, B, S):
    o = oracle()
    m = device_model(cfg)
    p = model_params(cfg)
    ids = o.random_tokens(cfg.vocab, B, S, 5)
    want32 = o.classifier_probs(cfg, p, ids, B, S, "fp32")
    got32 = m.classifier_probs(ids, B, S, "fp32")
    assert np.abs(got32.astype(np.float64) - want32).max() <= 1e-5
    goth = m.classifier_probs(ids, B, S, "hybrid")
    assert np.isfinite(goth).all()
    assert np.abs(goth.astype(np.float64) - want32).max() <= 2e-3
    wanth = o.classifier_probs(cfg, p, ids, B, S, "hybrid")
    assert np.abs(goth.astype(np.float64) - wanth).max() <= 2e-3


def test_classifier_probs_rejects_decoder():
    cfg = PRESETS["decoder_toy"]
    m = device_model(cfg)
    ids = oracle().random_tokens(cfg.vocab, 1, 8, 1)
    with pytest.raises(ValueError, match="encoder_only"):
        m.classifier_probs(ids, 1, 8, "hybrid")


# policy_from_spec (src/policy.cpp:69-116) outcomes: per-class assignments beyond the
# three named policies run the generic per-class SIMT path with the same rounding points
CUSTOM = {
    # hybrid with an fp32 attention block (overrides.AttentionScoreMatmul + Softmax)
    "hybrid_fp32_attention": [(1, 0, 1), (0, 0, 1), (0, 0, 1), (0, 0, 1), (1, 0, 1), (0, 0, 1), (0, 0, 1)],
    # fp32 with fp16-lattice linears accumulating in fp32
    "fp32_f16_linears": [(1, 0, 1), (0, 0, 1), (0, 0, 1), (0, 0, 1), (0, 0, 1), (0, 0, 1), (0, 0, 1)],
    # hybrid with a narrow (F16E-accumulating) LayerNorm
    "hybrid_narrow_ln": [(1, 0, 1), (1, 0, 1), (0, 0, 1), (1, 1, 1), (1, 0, 1), (0, 0, 1), (0, 0, 1)],
}


@pytest.mark.parametrize("name", sorted(CUSTOM))
@pytest.mark.parametrize("cfg", [PRESETS["decoder_toy"], PRESETS["encoder_toy"]], ids=["dec", "enc"])
def test_custom_policy_matches_oracle(name, cfg):
    o = oracle()
    m = device_model(cfg)
    spec = CUSTOM[name]
    pol = pg.PrecisionPolicy()
    for i, (c_, a_, s_) in enumerate(spec):
        pol.cls[i] = pg.KernelConfig(c_, a_, s_)
    pg._check(pg.lib().prlab_gpu_validate_policy(pg.C.byref(pol)) if hasattr(pg, "C") else 0)
    ids = o.random_tokens(cfg.vocab, 2, 24, 8)
    p = model_params(cfg)
    want = o.forward(cfg, p, ids, 2, 24, spec)
    got = m.forward(ids, 2, 24, pol)
    cmp = compare_logits(want, got)
    assert cmp["candidate_nonfinite"] == 0
    assert cmp["max_abs_error"] <= 5e-3 * float(np.abs(want).max()) and cmp["cosine"] >= 0.99999, cmp
