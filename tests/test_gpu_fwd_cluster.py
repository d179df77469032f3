"""The cluster batch-1 trunk (fwd_cluster.cu; opt-in with PRLAB_FWD_CLUSTER=1, DESIGN.md
section 5.3): 16-CTA clusters owning 32-row blocks, per-CTA pre-tiled weight streams,
cross-cluster k/v flags.  Held to the same bars as the default trunk: bit-exact embedding
gather against the reference's embed(), hybrid logits within the GPU<->CPU drift of the
other tensor-core paths, on causal and bidirectional models and on row blocks that split
or merge sequences (B > 1, S not a multiple of 32)."""
import numpy as np
import pytest

import paper_2603_28708_b200 as pg
from oracle.oracle import PRESETS, compare_logits, split_params
from prlab_testutil import have_reference_lib, model_params, oracle, reference

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


@pytest.fixture(autouse=True)
def cluster_on(monkeypatch):
    monkeypatch.setenv("PRLAB_FWD_CLUSTER", "1")


@pytest.mark.parametrize("name,B,S", [("gpt2_small", 1, 128), ("bert_base", 1, 128), ("gpt2_small", 4, 32),
                                      ("bert_base", 3, 40), ("gpt2_small", 2, 48), ("gpt2_small", 1, 7)])
def test_cluster_trunk_vs_cpu_hybrid(name, B, S):
    cfg = PRESETS[name]
    o = oracle()
    m = pg.DeviceModel(pg.ModelConfig(**cfg.__dict__), model_params(cfg))
    ids = o.random_tokens(cfg.vocab, B, S, 4242)
    got = m.forward(ids, B, S, "hybrid")
    r = compare_logits(o.forward(cfg, model_params(cfg), ids, B, S, "hybrid"), got)
    m.close()
    assert r["candidate_nonfinite"] == 0 and r["cosine"] >= 0.9999 and r["max_abs_error"] <= 5e-3, r


def test_cluster_embedding_bitexact():
    cfg = PRESETS["gpt2_small"]
    m = pg.DeviceModel(pg.ModelConfig(**cfg.__dict__), model_params(cfg))
    ids = oracle().random_tokens(cfg.vocab, 1, 128, 77)
    p = dict(split_params(cfg, model_params(cfg)))
    src = reference() if have_reference_lib() else oracle()
    want = src.embed(p["token_embedding"], p["position_embedding"], ids, 1, 128, 0)
    d_ids = torch.from_numpy(ids).cuda()
    out = torch.full((128, cfg.hidden), float("nan"), device="cuda")
    st = torch.cuda.current_stream().cuda_stream
    m.embedding_device(d_ids.data_ptr(), 1, 128, 2, out.data_ptr(), st)
    m.sync_status(st)
    m.close()
    assert np.array_equal(out.cpu().numpy().view(np.uint32), want.view(np.uint32))


def test_cluster_trunk_repeatable():
    """200 back-to-back forwards bit-identical (cluster syncs, ring and k/v flags reused)."""
    cfg = PRESETS["gpt2_small"]
    m = pg.DeviceModel(pg.ModelConfig(**cfg.__dict__), model_params(cfg))
    ids = torch.from_numpy(oracle().random_tokens(cfg.vocab, 1, 128, 5)).cuda()
    ld = (cfg.vocab + 7) // 8 * 8
    out = torch.empty(128, ld, dtype=torch.float16, device="cuda")
    st = torch.cuda.current_stream().cuda_stream
    m.forward_device(ids.data_ptr(), 1, 128, "hybrid", out.data_ptr(), pg.OUT_F16, ld, st, True)
    first = out.clone()
    for _ in range(200):
        m.forward_device(ids.data_ptr(), 1, 128, "hybrid", out.data_ptr(), pg.OUT_F16, ld, st, True)
    m.sync_status(st)
    m.close()
    assert torch.equal(out, first)
