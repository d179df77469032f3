"""fp32 logits from the device forward come straight out of the head GEMM's epilogue
(EPI_F16_F32: the widened binary16 values) -- they must equal the fp16 logits of the same
forward widened, bit for bit, for 16-byte-aligned and unaligned row pitches, on the
persistent-trunk, CTA-pair-trunk and multi-kernel paths and on the full_fp16 fast path,
and leave the pitch padding past the 16-byte chunk alone."""
import numpy as np
import pytest
import torch

import paper_2603_28708_b200 as pg
from oracle.oracle import ModelConfig
from prlab_testutil import model_params

pytestmark = pytest.mark.gpu

CFG = ModelConfig(archetype=1, num_layers=2, hidden=768, heads=12, ffn=3072, vocab=4093,
                  max_positions=512, seed=4)


@pytest.fixture(scope="module")
def model():
    m = pg.DeviceModel(pg.ModelConfig(**CFG.__dict__), model_params(CFG))
    yield m
    m.close()


@pytest.mark.parametrize("B,S", [(1, 128), (2, 96), (3, 200)], ids=["trunk", "pair-trunk", "multi-kernel"])
@pytest.mark.parametrize("policy", ["hybrid", "full_fp16"])
@pytest.mark.parametrize("ld32", [4100, 4095], ids=["aligned", "unaligned"])
def test_f32_logits_equal_widened_f16(model, B, S, policy, ld32):
    V, M = CFG.vocab, B * S
    ids = torch.from_numpy(np.random.default_rng(B * S).integers(0, V, M).astype(np.int32)).cuda()
    ld16 = (V + 7) // 8 * 8
    o16 = torch.empty(M, ld16, device="cuda", dtype=torch.float16)
    model.forward_device(ids.data_ptr(), B, S, policy, o16.data_ptr(), pg.OUT_F16, ld16)
    o32 = torch.full((M, ld32), float("nan"), device="cuda", dtype=torch.float32)
    for graph in (True, False):
        model.forward_device(ids.data_ptr(), B, S, policy, o32.data_ptr(), pg.OUT_F32, ld32, 0, graph)
        torch.cuda.synchronize()
        model.sync_status()
        assert torch.equal(o32[:, :V], o16[:, :V].float())
        # TMA stores (16-byte rows) may fill the row's 16-byte chunk; per-thread stores stop at V
        assert torch.isnan(o32[:, (V + 3) // 4 * 4 if ld32 % 4 == 0 else V:]).all()
