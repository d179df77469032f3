"""Device-side logits reductions (src/fidelity.cpp) against the
host restatements:

  * row NLL / argmax (window_nll_sum, fidelity.cpp:213-240): per-row NLL within 2e-6
    absolute of the numpy double computation (the device uses fp32 exponentials with
    double accumulation), argmax = numpy's first maximum, NaN/+inf rows poison;
  * compare_logits (fidelity.cpp:11-37) on device tensors = oracle.compare_logits on the
    host (double sums in a different order: 1e-9 relative);
  * perplexity (fidelity.cpp:248-279) with the NLL reduced on the device: fp32 policy
    within 1e-5 relative of the compiled reference, hybrid within 2e-3 of the CPU fp32
    value; the reference's validation errors.
"""
import numpy as np
import torch
import pytest

import paper_2603_28708_b200 as pg
from oracle.oracle import PRESETS, ModelConfig, compare_logits, window_nll_sum
from prlab_testutil import have_reference_lib, model_params, oracle, reference

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


@pytest.mark.parametrize("dtype", ["float32", "float16"])
@pytest.mark.parametrize("rows,n,ld", [(7, 1000, 1000), (33, 50257, 50264), (1, 3, 8)])
def test_row_nll_and_argmax(dtype, rows, n, ld):
    g = torch.Generator().manual_seed(rows * 7 + n)
    x = (torch.randn(rows, ld, generator=g) * 3.0).to(getattr(torch, dtype))
    if rows > 2:
        x[1, 5] = float("nan")          # poisoned row
        x[2, 0] = x[2, :n].max() + 1.0  # argmax at 0
        x[2, n - 1] = x[2, 0]           # tie: first index wins
    tg = torch.randint(0, n, (rows,), generator=g, dtype=torch.int32)
    tg[0] = -1                          # no target
    xd, tgd = x.cuda(), tg.cuda()
    nll = torch.empty(rows, dtype=torch.float64, device="cuda")
    am = torch.empty(rows, dtype=torch.int32, device="cuda")
    pg.row_nll_device(xd, tgd, nll, am, rows=rows, n=n, ld=ld)
    torch.cuda.synchronize()
    xh = x[:, :n].double().numpy()
    got, gam = nll.cpu().numpy(), am.cpu().numpy()
    for r in range(rows):
        row = xh[r]
        if np.isnan(row).any():
            assert np.isnan(got[r]) or tg[r] < 0
            continue
        want_am = int(np.argmax(row))
        assert gam[r] == want_am
        if tg[r] < 0:
            assert got[r] == 0.0
            continue
        mx = row.max()
        want = -((row[int(tg[r])] - mx) - np.log(np.exp(row - mx).sum()))
        assert abs(got[r] - want) <= 2e-6 * max(1.0, abs(want)), (r, got[r], want)


@pytest.mark.parametrize("cdtype", ["float32", "float16"])
def test_compare_logits_device(cdtype):
    g = torch.Generator().manual_seed(3)
    base = torch.randn(64, 1032, generator=g)
    cand = (base + 1e-3 * torch.randn(64, 1032, generator=g)).to(getattr(torch, cdtype))
    cand[3, 7] = float("inf")
    n = 1025
    r = pg.compare_logits_device(base.cuda(), cand.cuda(), 64, n)
    want = compare_logits(base[:, :n].numpy(), cand[:, :n].float().numpy())
    for k in ("max_abs_error", "mean_abs_error", "cosine"):
        assert abs(r[k] - want[k]) <= 1e-9 * max(1.0, abs(want[k])), (k, r[k], want[k])
    assert r["candidate_nonfinite"] == want["candidate_nonfinite"] == 1
    assert r["nan_affected"]


GPT2_SMALLV = ModelConfig(archetype=1, num_layers=2, hidden=768, heads=12, ffn=3072, vocab=4096,
                          max_positions=512, seed=0)


@pytest.mark.parametrize("cfg", [PRESETS["decoder_toy"], GPT2_SMALLV], ids=["toy", "gpt2_tc"])
def test_perplexity_on_device(cfg):
    o = oracle()
    p = model_params(cfg)
    m = pg.DeviceModel(pg.ModelConfig(**cfg.__dict__), p)
    stream = o.random_tokens(cfg.vocab, 1, 3 * 128 + 37, 17)
    ctx = 128
    if have_reference_lib() and cfg.num_layers * cfg.hidden <= 512:
        want32 = reference().perplexity(cfg, p, stream, ctx, "fp32")
    else:
        from oracle.oracle import perplexity_windows
        want32 = perplexity_windows(lambda w, n: o.forward(cfg, p, w, 1, n, "fp32"), stream, ctx)
    got32 = m.perplexity(stream, ctx, "fp32")
    assert abs(got32 - want32) <= 1e-5 * want32, (got32, want32)
    goth = m.perplexity(stream, ctx, "hybrid")
    assert abs(goth - want32) <= 2e-3 * want32, (goth, want32)
    with pytest.raises(ValueError, match="too short"):
        m.perplexity(stream[:ctx], ctx, "hybrid")
    with pytest.raises(ValueError, match="context_len must be >= 2"):
        m.perplexity(stream, 1, "hybrid")
    m.close()


def test_perplexity_rejects_encoder():
    cfg = PRESETS["encoder_toy"]
    m = pg.DeviceModel(pg.ModelConfig(**cfg.__dict__), model_params(cfg))
    with pytest.raises(ValueError, match="decoder_only"):
        m.perplexity(np.zeros(100, np.int32), 16, "hybrid")
    m.close()


def test_window_nll_restatement_uniform():
    """fidelity tests: uniform logits give perplexity equal to the vocabulary size
    (test_fidelity.cpp:139-147), through the device kernel."""
    V, S = 1000, 9
    x = torch.zeros(S, V, device="cuda")
    tg = torch.arange(1, S + 1, dtype=torch.int32, device="cuda")
    tg[-1] = -1
    nll = torch.empty(S, dtype=torch.float64, device="cuda")
    pg.row_nll_device(x, tg, nll)
    torch.cuda.synchronize()
    ppl = float(np.exp(nll.cpu().numpy()[:-1].sum() / (S - 1)))
    assert abs(ppl - V) <= 1e-9 * V
    assert abs(window_nll_sum(np.zeros((1, S, V), np.float32), np.arange(S)) / (S - 1) - np.log(V)) < 1e-12


@pytest.mark.parametrize("B,S", [(4, 128), (3, 200), (1, 64)])
def test_forward_nll_fused_head_matches_logits_path(B, S):
    """forward_nll_device: the LM head's log-softmax statistics fused
    into its GEMM epilogue (CTA-pair head, B*S >= 512 rows) give the same argmax as the
    logits + row_nll path bit for bit and the same NLL within 2e-6 absolute (fp32 partial
    sums of expf per 128 columns, folded in double); small shapes fall back to the logits
    path (identical results).  Odd vocabulary tail, targets in the last partial tile, -1
    targets (0 NLL)."""
    cfg = PRESETS["gpt2_small"].replace(num_layers=1)
    m = pg.DeviceModel(pg.ModelConfig(**cfg.__dict__), model_params(cfg))
    o = oracle()
    M, V = B * S, cfg.vocab
    ids = torch.from_numpy(o.random_tokens(V, B, S, 5)).cuda()
    rng = np.random.default_rng(7)
    tg = rng.integers(0, V, M).astype(np.int32)
    tg[::S] = -1
    tg[1::17] = V - 1 - rng.integers(0, 80, tg[1::17].size)  # inside the last (partial) n-tile
    tgd = torch.from_numpy(tg).cuda()
    nll = torch.full((M,), -7.0, dtype=torch.float64, device="cuda")
    am = torch.full((M,), -7, dtype=torch.int32, device="cuda")
    fused = m.forward_nll_device(ids.data_ptr(), tgd.data_ptr(), B, S, "hybrid", nll.data_ptr(), am.data_ptr())
    assert fused == (M >= 512)
    ld = (V + 7) // 8 * 8
    logits = torch.empty(M, ld, dtype=torch.float16, device="cuda")
    m.forward_device(ids.data_ptr(), B, S, "hybrid", logits.data_ptr(), pg.OUT_F16, ld)
    nll_ref = torch.empty(M, dtype=torch.float64, device="cuda")
    am_ref = torch.empty(M, dtype=torch.int32, device="cuda")
    pg.row_nll_device(logits, tgd, nll_ref, am_ref, rows=M, n=V, ld=ld)
    torch.cuda.synchronize()
    m.sync_status()
    assert np.array_equal(am.cpu().numpy(), am_ref.cpu().numpy())
    a, b = nll.cpu().numpy(), nll_ref.cpu().numpy()
    assert np.all(a[tg < 0] == 0.0) and np.all(np.isfinite(a))
    assert np.max(np.abs(a - b)) <= 2e-6, np.max(np.abs(a - b))
    # argmax only (no NLL buffer, no targets)
    am2 = torch.full((M,), -7, dtype=torch.int32, device="cuda")
    m.forward_nll_device(ids.data_ptr(), 0, B, S, "hybrid", 0, am2.data_ptr())
    torch.cuda.synchronize()
    assert np.array_equal(am2.cpu().numpy(), am_ref.cpu().numpy())
    m.close()


def test_perplexity_fused_head_matches_unfused(monkeypatch):
    """perplexity (fidelity.cpp:248-279) with >= 512 rows per batch of windows runs the
    head's fused log-softmax epilogue; the same stream through a model whose plans were
    made with PRLAB_NO_FUSED_NLL=1 (logits + row kernel) agrees within 1e-6 relative."""
    cfg = PRESETS["gpt2_small"].replace(num_layers=1)
    p = model_params(cfg)
    o = oracle()
    stream = o.random_tokens(cfg.vocab, 1, 6 * 128 + 5, 23)
    fused = pg.DeviceModel(pg.ModelConfig(**cfg.__dict__), p)
    a = fused.perplexity(stream, 128, "hybrid")
    monkeypatch.setenv("PRLAB_NO_FUSED_NLL", "1")
    plain = pg.DeviceModel(pg.ModelConfig(**cfg.__dict__), p)
    b = plain.perplexity(stream, 128, "hybrid")
    monkeypatch.delenv("PRLAB_NO_FUSED_NLL")
    assert np.isfinite(a) and abs(a - b) <= 1e-6 * b, (a, b)
    fused.close()
    plain.close()


@pytest.mark.parametrize("policy", ["full_fp16", "hybrid"])
def test_forward_nll_fused_nonfinite_rows(policy, monkeypatch):
    """The fused statistics epilogue on an adversarial model (fidelity.cpp:282-312): full_fp16's
    unstabilised softmax poisons rows with NaN / inf; the fused head must flag exactly the rows
    the logits + row_nll path flags (NaN NLL), give the same argmax and the same NLL elsewhere.
    The NaN / inf tests are folded into the running sum / max there, not done per element."""
    from oracle.oracle import make_adversarial_params
    cfg = PRESETS["gpt2_small"].replace(num_layers=1, seed=3)
    o = oracle()
    probe = o.random_tokens(cfg.vocab, 1, 32, 5)
    adv = make_adversarial_params(o, cfg, probe, 1, 32, 30.0)
    B, S = 16, 32
    M, V = B * S, cfg.vocab
    ids = np.tile(probe, (B, 1)).astype(np.int32).ravel()
    ids[32:] = o.random_tokens(V, B - 1, S, 9).ravel()  # first sequence = the probe itself
    tg = np.roll(ids, -1).astype(np.int32)
    d_ids, d_tg = torch.from_numpy(ids).cuda(), torch.from_numpy(tg).cuda()
    res = []
    for fused_on in (True, False):
        if not fused_on:
            monkeypatch.setenv("PRLAB_NO_FUSED_NLL", "1")
        m = pg.DeviceModel(pg.ModelConfig(**cfg.__dict__), adv)
        nll = torch.full((M,), -7.0, dtype=torch.float64, device="cuda")
        am = torch.full((M,), -7, dtype=torch.int32, device="cuda")
        f = m.forward_nll_device(d_ids.data_ptr(), d_tg.data_ptr(), B, S, policy, nll.data_ptr(), am.data_ptr())
        torch.cuda.synchronize()
        m.sync_status()
        assert f == fused_on
        res.append((nll.cpu().numpy(), am.cpu().numpy()))
        m.close()
    monkeypatch.delenv("PRLAB_NO_FUSED_NLL")
    (a, am_a), (b, am_b) = res
    bad_a, bad_b = ~np.isfinite(a), ~np.isfinite(b)
    assert np.array_equal(bad_a, bad_b)
    if policy == "full_fp16":
        assert bad_a.any()  # the mechanism fired
    else:
        assert not bad_a.any()
    assert np.array_equal(am_a[~bad_a], am_b[~bad_b])
    assert np.max(np.abs(a[~bad_a] - b[~bad_b]), initial=0.0) <= 2e-6
