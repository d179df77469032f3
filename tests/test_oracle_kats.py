"""The CPU oracle (oracle/prlab_oracle.c) against the reference's own known-answer
tests -- restated from tests/test_float16.cpp, test_kernels.cpp, test_model.cpp and
test_policy.cpp of the reference -- plus an independent binary16 check (numpy).

These pin the oracle before it is trusted as the checker of the CUDA path."""
import numpy as np
import pytest

from oracle.oracle import F16E, F32, PRESETS
from prlab_testutil import oracle

o = oracle()


def bits(x):
    return np.float32(x).view(np.uint32)


def same_value(a, b):
    if np.isnan(a) or np.isnan(b):
        return np.isnan(a) and np.isnan(b)
    return bits(a) == bits(b)


# ---------------------------------------------------------------------------
# binary16 lattice (reference tests/test_float16.cpp)
# ---------------------------------------------------------------------------
FROZEN = [  # test_float16.cpp:34-52
    (0.1, 0x2E66, 0.0999755859375), (1.0, 0x3C00, 1.0), (65504.0, 0x7BFF, 65504.0),
    (65505.0, 0x7BFF, 65504.0), (65519.99609375, 0x7BFF, 65504.0), (65520.0, 0x7C00, 0.0),
    (2.0 ** -25, 0x0000, 0.0), (float.fromhex("0x1.000002p-25"), 0x0001, 2.0 ** -24),
    (2.0 ** -24, 0x0001, 2.0 ** -24), (1.00048828125, 0x3C00, 1.0),
    (1.00146484375, 0x3C02, 1.001953125), (-1.0 / 3.0, 0xB555, -0.333251953125),
    (3.14159265, 0x4248, 3.140625), (2.0 ** -14, 0x0400, 2.0 ** -14),
    (6.097555160522461e-05, 0x03FF, 6.097555160522461e-05), (1e-7, 0x0002, 2.0 ** -23),
    (5e-7, 0x0008, 2.0 ** -21),
]


@pytest.mark.parametrize("x,hb,hv", FROZEN)
def test_frozen_conversions(x, hb, hv):
    x = float(np.float32(x))
    assert o.f16_encode(x) == hb
    if (hb & 0x7C00) != 0x7C00:
        assert same_value(o.round16(x), np.float32(hv))
        assert same_value(o.f16_decode(hb), np.float32(hv))


def test_overflow_and_nan():
    assert np.isinf(o.round16(65520.0)) and np.isinf(o.round16(1e30))
    assert o.round16(-65520.0) == -np.inf
    assert o.f16_encode(float("nan")) == 0x7E00
    assert np.isnan(o.round16(float("nan")))
    assert bits(o.f16_decode(0x7E01)) == 0x7FC00000


def test_exhaustive_half_lattice():  # test_float16.cpp:69-87
    for b in range(0x10000):
        v = o.f16_decode(b)
        ref = np.uint16(b).view(np.float16).astype(np.float32)
        assert same_value(v, ref), hex(b)
        if not np.isnan(v):
            assert same_value(o.round16(v), v)
            assert o.f16_encode(v) == b
        else:
            assert o.f16_encode(v) == 0x7E00


def test_random_floats_match_ieee_binary16():
    """Independent check: numpy's IEEE binary16 conversion (RNE, overflow to inf)
    on 200k random fp32 bit patterns, plus the values around every half ulp midpoint."""
    rng = np.random.default_rng(12345)
    xs = rng.integers(0, 2 ** 32, 200_000, dtype=np.uint64).astype(np.uint32).view(np.float32)
    got = o.round16_array(xs)
    with np.errstate(over="ignore", invalid="ignore"):
        want = xs.astype(np.float16).astype(np.float32)
    nan = np.isnan(want)
    assert np.array_equal(np.isnan(got), nan)
    assert np.array_equal(got[~nan].view(np.uint32), want[~nan].view(np.uint32))


def test_rounding_properties():  # test_float16.cpp:102-141
    rng = np.random.default_rng(99)
    xs = rng.uniform(-65504, 65504, 5000).astype(np.float32)
    r = o.round16_array(xs)
    assert np.array_equal(o.round16_array(r), r)
    assert np.array_equal(o.round16_array(-xs), -r)
    e = np.maximum(np.floor(np.log2(np.abs(xs.astype(np.float64)))), -14)
    assert np.all(np.abs(r.astype(np.float64) - xs) <= 2.0 ** (e - 11))


# ---------------------------------------------------------------------------
# operators (reference tests/test_kernels.cpp)
# ---------------------------------------------------------------------------
def test_long_reductions():  # test_kernels.cpp:37-60
    for n, want in [(2049, (2048.0, 2048.0, 2049.0)), (2050, (2048.0, 2050.0, 2050.0))]:
        a = np.ones((1, n), np.float32)
        b = np.ones((n, 1), np.float32)
        assert o.matmul(a, b, F16E, F16E)[0, 0] == want[0]
        assert o.matmul(a, b, F16E, F32)[0, 0] == want[1]
        assert o.matmul(a, b, F32, F32)[0, 0] == want[2]


def test_fp32_matmul_vs_fp64():  # test_kernels.cpp:62-75
    rng = np.random.default_rng(3)
    a = rng.uniform(-1, 1, (17, 33)).astype(np.float32)
    b = rng.uniform(-1, 1, (33, 9)).astype(np.float32)
    c = o.matmul(a, b, F32, F32)
    ref = a.astype(np.float64) @ b.astype(np.float64)
    assert np.abs(ref - c).max() <= 33 * 1.2e-7 * 33


def test_invalid_config_rejected():
    with pytest.raises(ValueError):
        o.matmul(np.ones((2, 2), np.float32), np.ones((2, 2), np.float32), F32, F16E)


def test_softmax_stable_and_unstable():  # test_kernels.cpp:82-98
    x = np.array([[12.0, 0.0]], np.float32)
    y = o.softmax(x, F16E, F16E, True)
    assert y[0, 0] == 1.0 and y[0, 1] == np.float32(6.139278411865234e-06)
    y = o.softmax(x, F16E, F16E, False)
    assert np.isnan(y[0, 0]) and y[0, 1] == 0.0


def test_softmax_rows_sum_to_one():  # test_kernels.cpp:100-117
    rng = np.random.default_rng(11)
    x = rng.uniform(-4, 4, (8, 16)).astype(np.float32)
    y32 = o.softmax(x, F32, F32)
    y16 = o.softmax(x, F16E, F16E)
    assert np.allclose(y32.astype(np.float64).sum(1), 1.0, atol=1e-6)
    assert np.allclose(y16.astype(np.float64).sum(1), 1.0, atol=0.01)


def test_scores_fold_scale():  # test_kernels.cpp:119-135
    q = np.array([[1, 2, 3], [4, 5, 6]], np.float32)
    k = np.array([[7, 8, 9], [10, 11, 12]], np.float32)
    s, tap = o.attention_scores(q, k, 0.125, F16E, F16E, capture=True)
    ref = (q.astype(np.float64) @ k.T.astype(np.float64)).astype(np.float32)
    assert np.array_equal(tap, ref * np.float32(0.125))
    assert np.array_equal(s, o.round16_array(ref * np.float32(0.125)))
    s32 = o.attention_scores(q, k, 0.125, F32, F32)
    assert np.array_equal(s32, ref * np.float32(0.125))


def test_layernorm():  # test_kernels.cpp:137-160
    y = o.layernorm(np.full((1, 6), 3.0, np.float32), np.ones(6, np.float32),
                    np.full(6, 0.25, np.float32), 1e-5, F32, F32)
    assert np.allclose(y, 0.25, rtol=1e-6)
    rng = np.random.default_rng(5)
    x = rng.uniform(-2, 2, (4, 64)).astype(np.float32)
    z = o.layernorm(x, np.ones(64, np.float32), np.zeros(64, np.float32), 1e-5, F32, F32)
    assert np.allclose(z.mean(1), 0, atol=1e-4) and np.allclose(z.var(1), 1, atol=1e-3)


def test_gelu_add_embed():  # test_kernels.cpp:162-191
    g = o.gelu(np.array([0.0, 1.0, -1.0], np.float32), F32, F32)
    assert g[0] == 0.0 and abs(g[1] - 0.8413447460685429) < 1e-6
    assert abs(g[2] + 0.15865525393145707) < 1e-6
    assert o.add(np.array([2048.0], np.float32), np.array([1.0], np.float32), F16E, F16E)[0] == 2048.0
    assert o.add(np.array([2048.0], np.float32), np.array([1.0], np.float32), F32, F32)[0] == 2049.0
    tok = np.array([[0, 0], [10, 20], [30, 40]], np.float32)
    pos = np.array([[1, 2], [3, 4]], np.float32)
    assert o.embed(tok, pos, [2, 1], 1, 2, F32).ravel().tolist() == [31.0, 42.0, 13.0, 24.0]
    with pytest.raises(IndexError):
        o.embed(tok, pos, [3, 0], 1, 2, F32)
    with pytest.raises(IndexError):
        o.embed(tok, pos, [0, 0, 0], 1, 3, F32)


# ---------------------------------------------------------------------------
# model (reference tests/test_model.cpp, tests/test_policy.cpp)
# ---------------------------------------------------------------------------
def test_param_counts():  # test_model.cpp:34-37
    assert o.param_count(PRESETS["bert_base"]) == 109_482_242
    assert o.param_count(PRESETS["gpt2_small"]) == 124_439_808


def test_init_deterministic_and_profile():  # test_model.cpp:66-112
    from oracle.oracle import split_params
    cfg = PRESETS["decoder_toy"].replace(seed=7)
    a, b = o.build_model(cfg), o.build_model(cfg)
    c = o.build_model(cfg.replace(seed=8))
    assert np.array_equal(a, b) and not np.array_equal(a, c)
    for name, t in split_params(cfg, a):
        if name.endswith("gamma"):
            assert np.all(t == 1.0)
        elif t.ndim == 2:
            if t.size >= 10_000:
                assert 0.015 < float(np.sqrt((t.astype(np.float64) ** 2).mean())) < 0.025
        else:
            assert np.all(t == 0.0)


def test_random_tokens():  # test_model.cpp:136-147
    t1 = o.random_tokens(320, 2, 16, 5)
    assert np.array_equal(t1, o.random_tokens(320, 2, 16, 5))
    assert not np.array_equal(t1, o.random_tokens(320, 2, 16, 6))
    assert t1.size == 32 and t1.min() >= 0 and t1.max() < 320


def test_decoder_causality_encoder_bidirectional():  # test_model.cpp:169-203
    cfg = PRESETS["decoder_toy"].replace(num_layers=2)
    p = o.build_model(cfg)
    a = o.random_tokens(cfg.vocab, 1, 8, 1)
    b = a.copy()
    b[7] = (b[7] + 1) % cfg.vocab
    la, lb = o.forward(cfg, p, a, 1, 8, "fp32"), o.forward(cfg, p, b, 1, 8, "fp32")
    assert np.array_equal(la[0, :7], lb[0, :7])
    ecfg = PRESETS["encoder_toy"].replace(num_layers=2)
    ep = o.build_model(ecfg)
    ea = o.random_tokens(ecfg.vocab, 1, 8, 2)
    eb = ea.copy()
    eb[7] = (eb[7] + 1) % ecfg.vocab
    assert not np.array_equal(o.forward(ecfg, ep, ea, 1, 8, "fp32")[0, 0],
                              o.forward(ecfg, ep, eb, 1, 8, "fp32")[0, 0])


def test_zero_layer_model_is_embedding():  # test_model.cpp:242-271
    cfg = PRESETS["decoder_toy"].replace(num_layers=0)
    p = o.build_model(cfg)
    ids = o.random_tokens(cfg.vocab, 2, 5, 7)
    out, calls = o.forward(cfg, p, ids, 2, 5, "fp32", want_calls=True)
    tok = p[:cfg.vocab * cfg.hidden].reshape(cfg.vocab, cfg.hidden)
    pos = p[cfg.vocab * cfg.hidden:(cfg.vocab + cfg.max_positions) * cfg.hidden].reshape(-1, cfg.hidden)
    want = tok[ids.reshape(2, 5)] + pos[:5][None]
    assert out.shape == (2, 5, cfg.hidden) and np.array_equal(out, want)
    assert calls[0][0] == 0 and calls[3][0] == 0  # no Linear, no LayerNorm


def test_policy_routing():  # test_policy.cpp:77-109
    cfg = PRESETS["decoder_toy"]
    p = o.build_model(cfg)
    ids = o.random_tokens(cfg.vocab, 1, 8, 42)
    _, h = o.forward(cfg, p, ids, 1, 8, "hybrid", want_calls=True)
    assert h[0][1] > 0 and h[0][0] == 0          # Linear on F16E only
    assert h[1][1] > 0                           # AttentionScoreMatmul F16E
    assert h[2][1] == 0 and h[2][0] > 0          # Softmax F32
    assert h[3][1] == 0 and h[6][1] == 0 and h[5][1] == 0
    assert h[4][1] > 0                           # Activation F16E
    _, f = o.forward(cfg, p, ids, 1, 8, "full_fp16", want_calls=True)
    assert all(f[c][0] == 0 for c in range(7))
    _, s = o.forward(cfg, p, ids, 1, 8, "fp32", want_calls=True)
    assert all(s[c][1] == 0 for c in range(7))
    assert np.array_equal(s.sum(1), f.sum(1))


def test_unknown_policy():
    with pytest.raises(ValueError, match="fp32"):
        o.policy("mixed")
