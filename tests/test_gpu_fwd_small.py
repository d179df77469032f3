"""The batch-1 persistent forward (fwd_small.cu: forward_hidden as one cooperative
kernel with grid barriers, used for B*S <= 128, and on CTA pairs for 128 < B*S <= 256)
against the multi-kernel tensor-core path and the CPU oracle, decoder (causal) and encoder
shapes, including ragged M."""
import os

import numpy as np
import pytest

import paper_2603_28708_b200 as pg
from oracle.oracle import ModelConfig, compare_logits
from prlab_testutil import model_params, oracle

pytestmark = pytest.mark.gpu

GPT2_SMALLV = ModelConfig(archetype=1, num_layers=2, hidden=768, heads=12, ffn=3072, vocab=4096,
                          max_positions=512, seed=0)
BERT_SMALLV = GPT2_SMALLV.replace(archetype=0, seed=1)
# GPT-2-medium-shaped (h 1024, 16 heads, ffn 4096): the largest hidden size the trunk takes
GPT2_MEDIUMV = GPT2_SMALLV.replace(hidden=1024, heads=16, ffn=4096, seed=2)


@pytest.mark.parametrize("cfg", [GPT2_SMALLV, BERT_SMALLV], ids=["gpt2", "bert"])
@pytest.mark.parametrize("B,S", [(1, 128), (1, 1), (1, 37), (2, 64), (4, 32), (3, 17),
                                 # 128 < B*S <= 256: the CTA-pair kernel (2-CTA clusters, M = 256 MMAs)
                                 (2, 128), (4, 64), (8, 32), (3, 77), (2, 65)])
def test_fwd_small_matches_multikernel_and_oracle(cfg, B, S, monkeypatch):
    _check_small(cfg, B, S, monkeypatch)


@pytest.mark.parametrize("B,S", [(128, 1), (200, 1), (37, 3)], ids=["single-128x1", "pair-200x1", "pair-37x3"])
def test_fwd_small_many_short_sequences(B, S, monkeypatch):
    """Many one-to-three-token sequences: the most attention tasks / per-task flags the
    barrier-free trunk has to track (B * heads * query blocks)."""
    _check_small(GPT2_SMALLV, B, S, monkeypatch)


@pytest.mark.parametrize("B,S", [(1, 128), (2, 100)], ids=["single", "pair"])
def test_fwd_small_h1024(B, S, monkeypatch):
    """h = 1024 (16 heads, ffn 4096): 16 k-block weight slabs, 16-query attention tasks and
    one-row stages in the pair kernel (the 32-query / two-row variants are h = 768 only)."""
    _check_small(GPT2_MEDIUMV, B, S, monkeypatch)


def _check_small(cfg, B, S, monkeypatch):
    o = oracle()
    p = model_params(cfg)
    ids = o.random_tokens(cfg.vocab, B, S, 5 + B + S)
    small = pg.DeviceModel(pg.ModelConfig(**cfg.__dict__), p)
    assert small.kernel_count(B, S, "hybrid") == 2  # the cooperative kernel + the LM head
    got = small.forward(ids, B, S, "hybrid")
    monkeypatch.setenv("PRLAB_NO_FWD_SMALL", "1")
    multi = pg.DeviceModel(pg.ModelConfig(**cfg.__dict__), p)
    assert multi.kernel_count(B, S, "hybrid") > 2
    ref = multi.forward(ids, B, S, "hybrid")
    monkeypatch.delenv("PRLAB_NO_FWD_SMALL")
    r = compare_logits(ref, got)
    assert r["candidate_nonfinite"] == 0 and r["cosine"] >= 0.99999, r
    cpu32 = o.forward(cfg, p, ids, B, S, "fp32")
    r32 = compare_logits(cpu32, got)
    assert r32["cosine"] >= 0.9998, r32
    small.close()
    multi.close()


def test_fwd_small_bad_token_reported():
    cfg = GPT2_SMALLV
    m = pg.DeviceModel(pg.ModelConfig(**cfg.__dict__), model_params(cfg))
    import torch
    ids = torch.zeros(64, dtype=torch.int32, device="cuda")
    ids[5] = cfg.vocab + 3
    out = torch.empty(64, (cfg.vocab + 7) // 8 * 8, dtype=torch.float16, device="cuda")
    st = torch.cuda.current_stream().cuda_stream
    m.forward_device(ids.data_ptr(), 1, 64, "hybrid", out.data_ptr(), pg.OUT_F16, out.shape[1], st, True)
    with pytest.raises(IndexError):
        m.sync_status(st)
    m.close()


@pytest.mark.parametrize("B,S", [(1, 128), (2, 128)], ids=["single", "pair"])
def test_fwd_small_repeatable_under_back_to_back_launches(B, S):
    """Race detector for the grid-barrier protocol (release/acquire + the TMA thread's
    proxy fence) and, at B*S > 128, the CTA-pair protocol (remote arrivals, multicast
    commits): 200 back-to-back forwards of a 12-layer model on one stream must give
    bit-identical logits -- a stale operand read in any of the ~85 stages would not."""
    import torch
    cfg = GPT2_SMALLV.replace(num_layers=12)
    o = oracle()
    m = pg.DeviceModel(pg.ModelConfig(**cfg.__dict__), model_params(cfg))
    ids = torch.as_tensor(o.random_tokens(cfg.vocab, B, S, 11).reshape(-1), dtype=torch.int32, device="cuda")
    width = (cfg.vocab + 7) // 8 * 8
    outs = torch.empty(200, B * S, width, dtype=torch.float16, device="cuda")
    st = torch.cuda.current_stream().cuda_stream
    for i in range(outs.shape[0]):
        m.forward_device(ids.data_ptr(), B, S, "hybrid", outs[i].data_ptr(), pg.OUT_F16, width, st, True)
    torch.cuda.synchronize()
    m.sync_status(st)
    ref = outs[0]
    assert torch.isfinite(ref.float()).all()
    bad = [(i) for i in range(1, outs.shape[0]) if not torch.equal(outs[i], ref)]
    assert not bad, f"{len(bad)} of {outs.shape[0] - 1} repeats differ (first {bad[:5]})"
    m.close()


@pytest.mark.parametrize("B,S", [(1, 128), (2, 96), (5, 13)], ids=["single", "pair", "ragged"])
def test_fwd_small_counter_handoffs_match_grid_barriers(B, S, monkeypatch):
    """The barrier-free trunk (per-task release counters) and the same kernel with a grid
    barrier at every stage boundary (PRLAB_SMALL_BARRIERS=1) compute the same logits bit for
    bit: only the synchronisation differs."""
    cfg = GPT2_SMALLV
    p = model_params(cfg)
    ids = oracle().random_tokens(cfg.vocab, B, S, 17 + B)
    flags = pg.DeviceModel(pg.ModelConfig(**cfg.__dict__), p)
    a = flags.forward(ids, B, S, "hybrid")
    # (read when the launch is recorded: a fresh model captures its forward graph with it set)
    monkeypatch.setenv("PRLAB_SMALL_BARRIERS", "1")
    barriers = pg.DeviceModel(pg.ModelConfig(**cfg.__dict__), p)
    b = barriers.forward(ids, B, S, "hybrid")
    b2 = barriers.forward(ids, B, S, "hybrid")
    monkeypatch.delenv("PRLAB_SMALL_BARRIERS")
    assert np.isfinite(a).all()
    assert np.array_equal(a, b) and np.array_equal(b, b2)
    flags.close()
    barriers.close()
