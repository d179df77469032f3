"""PRLABCKP loader (load_checkpoint, src/checkpoint.cpp:133-162) straight into the
device arena.

CPU part: the format checks run before any device work and raise the reference's
messages (runtime_error -> RuntimeError); the checkpoints are written by the compiled
reference (serialize_checkpoint).  GPU part: loading an f32 checkpoint gives logits
bit-identical to uploading the same parameters; an f16 checkpoint equals uploading the
reference's own load_checkpoint() result.
"""
import os
import struct

import numpy as np
import pytest

import paper_2603_28708_b200 as pg
from oracle.oracle import PRESETS
from prlab_testutil import have_reference_lib, model_params, oracle, reference

needs_ref = pytest.mark.skipif(not have_reference_lib(), reason="oracle/_ref not built here")


def _write(tmp_path, cfg, f16=False, name="m.ckp"):
    path = str(tmp_path / name)
    reference().serialize_checkpoint(cfg, model_params(cfg), path, f16=f16)
    return path


@needs_ref
def test_checkpoint_format_errors(tmp_path):
    cfg = PRESETS["decoder_toy"]
    good = open(_write(tmp_path, cfg), "rb").read()
    cases = {
        "bad magic": (b"NOTACKPT" + good[8:], "not a checkpoint \\(bad magic\\)"),
        "version": (good[:8] + struct.pack("<I", 7) + good[12:], "unsupported checkpoint version 7"),
        "truncated": (good[: len(good) // 2], "checkpoint truncated while reading tensor payload"),
    }
    for name, (blob, msg) in cases.items():
        p = tmp_path / f"{name.replace(' ', '_')}.ckp"
        p.write_bytes(blob)
        with pytest.raises(RuntimeError, match=msg):
            pg.DeviceModel.from_checkpoint(str(p))
    with pytest.raises(RuntimeError, match="cannot open checkpoint"):
        pg.DeviceModel.from_checkpoint(str(tmp_path / "missing.ckp"))
    # a record out of canonical order (the reference names both tensors)
    cfg_len = struct.unpack_from("<I", good, 12)[0]
    off = 16 + cfg_len
    n0 = struct.unpack_from("<I", good, off)[0]
    assert good[off + 4: off + 4 + n0] == b"token_embedding"
    bad = bytearray(good)
    bad[off + 4: off + 4 + n0] = b"token_embeddinX"
    (tmp_path / "order.ckp").write_bytes(bytes(bad))
    with pytest.raises(RuntimeError, match="unexpected tensor 'token_embeddinX' \\(wanted 'token_embedding'\\)"):
        pg.DeviceModel.from_checkpoint(str(tmp_path / "order.ckp"))


@needs_ref
@pytest.mark.gpu
@pytest.mark.parametrize("cfg", [PRESETS["decoder_toy"], PRESETS["encoder_toy"]], ids=["dec", "enc"])
@pytest.mark.parametrize("f16", [False, True], ids=["f32", "f16"])
def test_checkpoint_loads_into_arena(tmp_path, cfg, f16):
    path = _write(tmp_path, cfg, f16=f16)
    loaded = pg.DeviceModel.from_checkpoint(path)
    assert loaded.config == pg.ModelConfig(**cfg.__dict__)
    params = reference().load_checkpoint(path, cfg) if f16 else model_params(cfg)
    direct = pg.DeviceModel(pg.ModelConfig(**cfg.__dict__), params)
    ids = oracle().random_tokens(cfg.vocab, 2, 33, 4)
    for pol in ("hybrid", "fp32"):
        a = loaded.forward(ids, 2, 33, pol)
        b = direct.forward(ids, 2, 33, pol)
        assert np.array_equal(a.view(np.uint32), b.view(np.uint32)), pol
    loaded.close()
    direct.close()
