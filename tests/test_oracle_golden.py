"""The oracle restatement against the reference itself:

* tests/golden/ fixtures produced by running the compiled reference
  (tests/golden/make_golden.py) -- these travel to the GPU box;
* bit-for-bit comparisons with oracle/_ref/libprlab_ref.so when it is built
  (this container), across policies, seeds and archetypes.
"""
import json
import os

import numpy as np
import pytest

from oracle.oracle import PRESETS
from prlab_testutil import have_reference_lib, oracle, reference

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
o = oracle()


def u32(a):
    return np.ascontiguousarray(a, np.float32).view(np.uint32)


@pytest.fixture(scope="module")
def meta():
    with open(os.path.join(GOLD, "meta.json")) as f:
        return json.load(f)


@pytest.mark.parametrize("name", ["decoder_toy", "encoder_toy"])
def test_toy_logits_bitexact_vs_golden(name, meta):
    g = np.load(os.path.join(GOLD, "toy_logits.npz"))
    cfg = PRESETS[name].replace(seed=3)
    params = o.build_model(cfg)
    assert np.float64(params.astype(np.float64).sum()) == g[f"{name}_param_sum"][0]
    ids = o.random_tokens(cfg.vocab, 2, 16, 9)
    assert np.array_equal(ids, g[f"{name}_ids"])
    for pol in ["fp32", "hybrid", "full_fp16"]:
        got, calls = o.forward(cfg, params, ids, 2, 16, pol, want_calls=True)
        assert np.array_equal(u32(got), u32(g[f"{name}_{pol}"])), pol
        assert calls.tolist() == meta["toy"][name][f"calls_{pol}"]


@pytest.mark.parametrize("name", ["gpt2_small", "bert_base"])
def test_preset_rows_vs_golden(name):
    g = np.load(os.path.join(GOLD, "preset_rows.npz"))
    cfg = PRESETS[name]
    params = o.build_model(cfg)
    assert np.float64(params.astype(np.float64).sum()) == g[f"{name}_param_sum"][0]
    ids = o.random_tokens(cfg.vocab, 1, 32, 1234)
    assert np.array_equal(ids, g[f"{name}_ids"])
    for pol in ["fp32", "hybrid"]:
        lg = o.forward(cfg, params, ids, 1, 32, pol).reshape(32, cfg.vocab)
        assert np.array_equal(lg.argmax(1), g[f"{name}_{pol}_argmax"])
        assert np.array_equal(u32(lg.max(1)), u32(g[f"{name}_{pol}_max"]))
        assert np.array_equal(lg.astype(np.float64).sum(1), g[f"{name}_{pol}_sum"])
        assert np.array_equal(u32(lg.ravel()[g[f"{name}_sample_idx"]]), u32(g[f"{name}_{pol}_sample"]))


def test_operators_bitexact_vs_golden():
    g = np.load(os.path.join(GOLD, "ops.npz"))
    for c, ac in [(0, 0), (1, 0), (1, 1)]:
        assert np.array_equal(u32(o.matmul(g["a"], g["b"], c, ac)), u32(g[f"matmul_{c}{ac}"]))
        assert np.array_equal(u32(o.layernorm(g["xl"], g["g"], g["be"], 1e-5, c, ac)),
                              u32(g[f"layernorm_{c}{ac}"]))
        assert np.array_equal(u32(o.gelu(g["xg"], c, ac)), u32(g[f"gelu_{c}{ac}"]))
        s, tap = o.attention_scores(g["q"], g["k"], 0.25, c, ac, capture=True)
        assert np.array_equal(u32(s), u32(g[f"scores_{c}{ac}"]))
        assert np.array_equal(u32(tap), u32(g[f"scores_tap_{c}{ac}"]))
        for st in (0, 1):
            got = o.softmax(g["x"], c, ac, bool(st))
            want = g[f"softmax_{c}{ac}{st}"]
            assert np.array_equal(np.isnan(got), np.isnan(want))
            ok = ~np.isnan(want)
            assert np.array_equal(u32(got[ok]), u32(want[ok]))
    for c in (0, 1):
        assert np.array_equal(u32(o.embed(g["tok"], g["pos"], g["eids"], 3, 10, c)), u32(g[f"embed_{c}"]))


needs_ref = pytest.mark.skipif(not have_reference_lib(), reason="oracle/_ref not built here")


@needs_ref
@pytest.mark.parametrize("name", ["decoder_toy", "encoder_toy"])
@pytest.mark.parametrize("seed", [0, 11])
@pytest.mark.parametrize("B,S", [(1, 1), (3, 23), (2, 160)])
def test_oracle_bitexact_vs_reference(name, seed, B, S):
    r = reference()
    cfg = PRESETS[name].replace(seed=seed)
    p = o.build_model(cfg)
    assert np.array_equal(u32(p), u32(r.build_model(cfg)))
    ids = o.random_tokens(cfg.vocab, B, S, seed + 1)
    assert np.array_equal(ids, r.random_tokens(cfg.vocab, B, S, seed + 1))
    for pol in ["fp32", "hybrid", "full_fp16"]:
        a, ca = o.forward(cfg, p, ids, B, S, pol, want_calls=True)
        b, cb = r.forward(cfg, p, ids, B, S, pol, want_calls=True)
        assert np.array_equal(u32(a), u32(b)), pol
        assert np.array_equal(ca, cb)


@needs_ref
def test_oracle_per_sequence_equals_batched_reference():
    """Batch consistency: per-sequence reference runs == batched oracle."""
    r = reference()
    cfg = PRESETS["decoder_toy"]
    p = o.build_model(cfg)
    ids = o.random_tokens(cfg.vocab, 4, 20, 3)
    a = o.forward(cfg, p, ids, 4, 20, "hybrid")
    b = r.forward(cfg, p, ids, 4, 20, "hybrid", threads=4)
    assert np.array_equal(u32(a), u32(b))


@needs_ref
def test_round16_matches_reference_on_random_bits():
    r = reference()
    rng = np.random.default_rng(1)
    for x in rng.integers(0, 2 ** 32, 20_000, dtype=np.uint64).astype(np.uint32).view(np.float32):
        a, b = o.round16(float(x)), r.lib.ref_round16(float(x))
        assert (np.isnan(a) and np.isnan(b)) or u32(a) == u32(b)


@needs_ref
@pytest.mark.parametrize("name", ["decoder_toy", "encoder_toy"])
def test_adversarial_construction_matches_reference(name):
    from oracle.oracle import make_adversarial_params
    r = reference()
    cfg = PRESETS[name].replace(seed=4)
    probe = o.random_tokens(cfg.vocab, 1, 32, 5)
    a = make_adversarial_params(o, cfg, probe, 1, 32, 30.0)
    b = r.make_adversarial_model(cfg, probe, 1, 32, 30.0)
    assert np.array_equal(u32(a), u32(b))
    # the NaN mechanism (test_fidelity.cpp:175-195): full_fp16 overflows, hybrid/fp32 stay finite
    ids = o.random_tokens(cfg.vocab, 1, 32, 5)
    assert not np.isfinite(o.forward(cfg, a, ids, 1, 32, "full_fp16")).all()
    assert np.isfinite(o.forward(cfg, a, ids, 1, 32, "hybrid")).all()
    assert np.isfinite(o.forward(cfg, a, ids, 1, 32, "fp32")).all()


@pytest.mark.skipif(not have_reference_lib(), reason="oracle/_ref not built (needs /root/reference)")
@pytest.mark.parametrize("policy", ["fp32", "hybrid", "full_fp16"])
def test_oracle_classifier_and_taps_bit_identical_to_reference(policy):
    """classifier_probs (model.cpp:484-526) and the retain_scores taps (model.cpp:393-427)
    of the restatement equal the compiled reference bit for bit."""
    from oracle.oracle import ModelConfig
    o, r = oracle(), reference()
    enc = ModelConfig(archetype=0, num_layers=2, hidden=128, heads=4, ffn=256, vocab=320,
                      max_positions=160, seed=3)
    p = o.build_model(enc)
    ids = o.random_tokens(enc.vocab, 3, 40, 5)
    a = o.classifier_probs(enc, p, ids, 3, 40, policy)
    b = r.classifier_probs(enc, p, ids, 3, 40, policy)
    assert np.array_equal(a.view(np.uint32), b.view(np.uint32))
    dec = enc.replace(archetype=1)
    p = o.build_model(dec)
    lo, to = o.forward(dec, p, ids, 3, 40, policy, retain_scores=True)
    lr, tr = r.forward_scores(dec, p, ids, 3, 40, policy)
    assert np.array_equal(to.view(np.uint32), tr.view(np.uint32))
    assert np.array_equal(np.nan_to_num(lo).view(np.uint32), np.nan_to_num(lr).view(np.uint32))


@pytest.mark.skipif(not have_reference_lib(), reason="oracle/_ref not built (needs /root/reference)")
@pytest.mark.parametrize("policy", ["fp32", "hybrid"])
def test_perplexity_restatement_matches_reference(policy):
    """perplexity / window_nll_sum (fidelity.cpp:213-279) restated over the oracle's
    forward equals the compiled reference (double-precision log-softmax; numpy's exp may
    differ from glibc's in the last ulp)."""
    from oracle.oracle import perplexity_windows
    o, r = oracle(), reference()
    cfg = PRESETS["decoder_toy"]
    p = o.build_model(cfg)
    stream = o.random_tokens(cfg.vocab, 1, 150, 9)
    want = r.perplexity(cfg, p, stream, 64, policy)
    got = perplexity_windows(lambda w, n: o.forward(cfg, p, w, 1, n, policy), stream, 64)
    assert abs(got - want) <= 1e-12 * want
