"""Concurrency contract of the drop-in (include/prlab_gpu.h "Threading / streams"; the
reference's functions are safe concurrently on distinct data):

  * one model driven from two CUDA streams with no host synchronisation in between:
    every call orders itself after the previous call's work (the workspace, split-K
    scratch and the persistent kernel's grid-barrier counter are shared), so results
    equal the single-stream ones bit for bit;
  * two models driven from two host threads at once (ctypes drops the GIL): the batch-1
    persistent kernel's 28 KB launch arguments are per thread, so neither launch sees the
    other model's tensor maps or weights.
"""
import threading

import numpy as np
import pytest

import paper_2603_28708_b200 as pg
from oracle.oracle import PRESETS
from prlab_testutil import model_params, oracle

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


def _logits(out, B, S, V):
    return out[:, :V].float().cpu().numpy().reshape(B, S, V)


@pytest.mark.parametrize("B,S", [(1, 128), (4, 200)])   # persistent kernel / multi-kernel path
def test_one_model_two_streams(B, S):
    cfg = PRESETS["gpt2_small"].replace(num_layers=4)
    m = pg.DeviceModel(pg.ModelConfig(**cfg.__dict__), model_params(cfg))
    V, ld = cfg.vocab, (cfg.vocab + 7) // 8 * 8
    ids = [oracle().random_tokens(V, B, S, 10 + i) for i in range(2)]
    d_ids = [torch.from_numpy(x).cuda() for x in ids]
    want = [m.forward(x, B, S, "hybrid") for x in ids]
    streams = [torch.cuda.Stream(), torch.cuda.Stream()]
    outs = [torch.empty(B * S, ld, dtype=torch.float16, device="cuda") for _ in range(2)]
    torch.cuda.synchronize()
    for rep in range(6):
        for i in range(2):  # alternate streams, no host sync: only the library's ordering
            m.forward_device(d_ids[i].data_ptr(), B, S, "hybrid", outs[i].data_ptr(), pg.OUT_F16, ld,
                             streams[i].cuda_stream, rep % 2 == 0)
    torch.cuda.synchronize()
    m.sync_status(0)
    for i in range(2):
        assert np.array_equal(_logits(outs[i], B, S, V), want[i])
    m.close()


def test_two_models_two_threads():
    cfgs = [PRESETS["gpt2_small"].replace(num_layers=3, seed=s) for s in (0, 9)]
    models = [pg.DeviceModel(pg.ModelConfig(**c.__dict__), oracle().build_model(c)) for c in cfgs]
    V, ld, B, S = cfgs[0].vocab, (cfgs[0].vocab + 7) // 8 * 8, 1, 128
    ids = oracle().random_tokens(V, B, S, 3)
    want = [m.forward(ids, B, S, "hybrid") for m in models]
    assert not np.array_equal(want[0], want[1])
    errors, results = [], [None, None]

    def run(i):
        try:
            st = torch.cuda.Stream()
            d_ids = torch.from_numpy(ids).cuda()
            out = torch.empty(B * S, ld, dtype=torch.float16, device="cuda")
            with torch.cuda.stream(st):
                for _ in range(40):
                    models[i].forward_device(d_ids.data_ptr(), B, S, "hybrid", out.data_ptr(), pg.OUT_F16, ld,
                                             st.cuda_stream, False)
                st.synchronize()
            results[i] = _logits(out, B, S, V)
        except Exception as e:  # surfaced below
            errors.append(e)

    th = [threading.Thread(target=run, args=(i,)) for i in range(2)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    assert not errors, errors
    for i in range(2):
        assert np.array_equal(results[i], want[i])
        models[i].close()


@pytest.mark.parametrize("B,S", [(1, 128), (2, 64)])
def test_one_model_concurrent_host_callers(B, S):
    """prlab_gpu_forward from three host threads on one model (the overlapped two-phase path:
    compute under the model lock into one of two logits slots, copy-out outside it): every
    call returns exactly the logits of its own ids, equal to a serial call's, while the
    copy-outs of one call overlap another call's compute."""
    cfg = PRESETS["gpt2_small"].replace(num_layers=2)
    m = pg.DeviceModel(pg.ModelConfig(**cfg.__dict__), model_params(cfg))
    V = cfg.vocab
    ids = [oracle().random_tokens(V, B, S, 40 + i) for i in range(3)]
    want = [m.forward(x, B, S, "hybrid") for x in ids]  # first call calibrates the copy-out
    assert m.host_copy_mode(B, S, "hybrid") in (1, 2)
    errors, bad = [], []

    def run(i):
        try:
            for rep in range(12):
                got = m.forward(ids[i], B, S, "hybrid")
                if not np.array_equal(got, want[i]):
                    bad.append((i, rep))
        except Exception as e:  # pragma: no cover
            errors.append(e)
    ths = [threading.Thread(target=run, args=(i,)) for i in range(3)]
    for t in ths:
        t.start()
    for t in ths:
        t.join()
    assert not errors, errors
    assert not bad, bad
    m.close()
