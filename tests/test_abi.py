"""CPU-side checks of the drop-in boundary: the C-ABI library loads, exports every
symbol include/prlab_gpu.h declares, mirrors the reference's host-side semantics
(policies, fixture generators, validation messages) and -- with no GPU -- fails
loudly instead of falling back to the CPU."""
import ctypes as C
import os
import re
import subprocess

import numpy as np
import pytest

import paper_2603_28708_b200 as pg
from oracle.oracle import PRESETS
from prlab_testutil import gpu_available, oracle


def test_library_exports_every_header_symbol():
    lib = pg.lib()
    declared = pg.header_symbols()
    assert len(declared) >= 20
    for name in declared:
        assert hasattr(lib, name), name
    # and the ctypes table binds exactly the declared surface
    assert sorted(n for n, _, _ in pg.EXPORTS) == declared


def test_library_is_sm100a_native():
    out = subprocess.run(["cuobjdump", "-lelf", pg.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    sass = subprocess.run(["cuobjdump", "-sass", pg.LIB_PATH], capture_output=True, text=True).stdout
    for mnemonic in ["UTCHMMA", "UTMALDG", "LDTM"]:  # tcgen05.mma / TMA / tcgen05.ld
        assert mnemonic in sass, mnemonic


def test_no_cpu_fallback_in_product():
    """The product never links or loads the oracle."""
    src_dir = os.path.dirname(pg.LIB_PATH) + "/../csrc"
    for f in os.listdir(src_dir):
        text = open(os.path.join(src_dir, f)).read()
        assert "oracle" not in text.lower(), f
    init = open(pg.__file__).read()
    assert "import oracle" not in init and "from oracle" not in init


def test_policies_mirror_reference():
    hyb = pg.resolve_policy("hybrid")
    for c in ["Linear", "AttentionScoreMatmul", "Activation"]:
        k = hyb.config_for(c)
        assert (k.compute, k.accum) == (pg.F16E, pg.F32)
    for c in ["Softmax", "LayerNorm", "Embedding", "Residual"]:
        k = hyb.config_for(c)
        assert (k.compute, k.accum) == (pg.F32, pg.F32)
    assert hyb.config_for("Softmax").stabilized
    full = pg.resolve_policy("full_fp16")
    assert all(full.cls[i].compute == pg.F16E and full.cls[i].accum == pg.F16E for i in range(7))
    assert not full.config_for("Softmax").stabilized
    with pytest.raises(ValueError, match="valid: fp32, full_fp16, hybrid"):
        pg.resolve_policy("mixed")
    p = pg.policy_from_classes("hybrid", {"Softmax": {"compute": "f16e", "accum": "f16e",
                                                      "stabilized": False}})
    assert p.config_for("Softmax").compute == pg.F16E and not p.config_for("Softmax").stabilized
    with pytest.raises(ValueError, match="f32 compute with f16e"):
        pg.policy_from_classes("fp32", {"Linear": {"compute": "f32", "accum": "f16e"}})


@pytest.mark.parametrize("name", ["decoder_toy", "encoder_toy"])
def test_fixture_generators_match_reference_streams(name):
    cfg = PRESETS[name].replace(seed=5)
    pcfg = pg.ModelConfig(**cfg.__dict__)
    assert pg.param_count(pcfg) == oracle().param_count(cfg)
    a = pg.build_model(pcfg)
    b = oracle().build_model(cfg)
    assert np.array_equal(a.view(np.uint32), b.view(np.uint32))
    assert np.array_equal(pg.random_tokens(cfg.vocab, 3, 7, 9), oracle().random_tokens(cfg.vocab, 3, 7, 9))


def test_preset_param_counts():
    assert pg.param_count(pg.ModelConfig.bert_base()) == 109_482_242
    assert pg.param_count(pg.ModelConfig.gpt2_small()) == 124_439_808


def test_config_validation_messages():
    bad = pg.ModelConfig.decoder_toy().replace(heads=3)
    with pytest.raises(ValueError, match="heads"):
        pg.build_model(bad)
    with pytest.raises(ValueError, match="ffn"):
        pg.build_model(pg.ModelConfig.decoder_toy().replace(ffn=64))
    with pytest.raises(ValueError):
        pg.ModelConfig.preset("bert_huge")


def test_flop_count_matches_reference_formula():  # test_model.cpp:114-134
    cfg = pg.ModelConfig(1, 1, 2, 1, 4, 7, 8)
    fc = pg.flop_count(cfg, 1, 2)
    assert (fc["linear"], fc["attention"], fc["output_projection"], fc["total"]) == (128, 32, 56, 216)
    g = pg.ModelConfig.gpt2_small()
    lin = 12 * 2 * (4 * 768 ** 2 + 2 * 768 * 3072) * 128
    att = 12 * 4 * 128 ** 2 * 768
    out = 2 * 128 * 768 * 50257
    assert pg.flop_count(g, 1, 128)["total"] == lin + att + out  # ~32.23 GFLOP


@pytest.mark.skipif(gpu_available(), reason="checks the no-GPU failure mode")
def test_fails_loudly_without_gpu():
    cfg = pg.ModelConfig.decoder_toy()
    with pytest.raises(pg.CudaError, match="no CPU fallback"):
        pg.DeviceModel(cfg, pg.build_model(cfg))
    with pytest.raises(pg.CudaError):
        pg.matmul(np.ones((2, 2), np.float32), np.ones((2, 2), np.float32),
                  pg.KernelConfig(pg.F32, pg.F32, True))


def test_header_is_plain_c():
    """include/prlab_gpu.h compiles as C (no torch / C++ types at the boundary)."""
    src = '#include "prlab_gpu.h"\nint main(void){prlab_policy p; return prlab_gpu_resolve_policy("hybrid", &p);}\n'
    path = "/tmp/prlab_abi_check.c"
    with open(path, "w") as f:
        f.write(src)
    inc = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "include")
    r = subprocess.run(["gcc", "-std=c99", "-Wall", "-Werror", "-c", path, "-I", inc, "-o", "/tmp/prlab_abi_check.o"],
                       capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
