"""ctypes bindings for the prlab CPU oracle -- TEST INFRASTRUCTURE ONLY.

Two checkers live behind this module:

* ``Oracle`` -- the plain-C restatement of the reference hot path
  (``oracle/prlab_oracle.c`` -> ``oracle/build/liboracle.so``);
* ``Reference`` -- the unmodified reference sources compiled by
  ``oracle/Makefile`` into ``oracle/_ref/libprlab_ref.so``.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
reference arm may import this module, and only as the checker or the CPU
baseline.  The product package (``paper_2603_28708_b200``) never imports it.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "build", "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libprlab_ref.so")

F32, F16E = 0, 1
CLASSES = ["Linear", "AttentionScoreMatmul", "Softmax", "LayerNorm", "Activation",
           "Embedding", "Residual"]


@dataclass(frozen=True)
class ModelConfig:
    """Reference ModelConfig (include/prlab/model.hpp:21-52); archetype 0 encoder, 1 decoder."""
    archetype: int
    num_layers: int
    hidden: int
    heads: int
    ffn: int
    vocab: int
    max_positions: int
    seed: int = 0

    def replace(self, **kw) -> "ModelConfig":
        d = self.__dict__.copy()
        d.update(kw)
        return ModelConfig(**d)


# src/model.cpp:122-136
PRESETS = {
    "bert_base": ModelConfig(0, 12, 768, 12, 3072, 30522, 512),
    "gpt2_small": ModelConfig(1, 12, 768, 12, 3072, 50257, 1024),
    "encoder_toy": ModelConfig(0, 4, 128, 4, 256, 320, 160),
    "decoder_toy": ModelConfig(1, 4, 128, 4, 256, 320, 160),
}


class _Kcfg(C.Structure):
    _fields_ = [("compute", C.c_int), ("accum", C.c_int), ("stabilized", C.c_int)]


class _Policy(C.Structure):
    _fields_ = [("cls", _Kcfg * 7)]


class _ModelCfg(C.Structure):
    _fields_ = [("archetype", C.c_int), ("num_layers", C.c_int64), ("hidden", C.c_int64),
                ("heads", C.c_int64), ("ffn", C.c_int64), ("vocab", C.c_int64),
                ("max_positions", C.c_int64), ("seed", C.c_uint64)]


def _fp(a):
    return a.ctypes.data_as(C.POINTER(C.c_float)) if a is not None else None


def _ip(a):
    return a.ctypes.data_as(C.POINTER(C.c_int32))


def _up(a):
    return a.ctypes.data_as(C.POINTER(C.c_uint64)) if a is not None else None


def _mcfg(c: ModelConfig) -> _ModelCfg:
    return _ModelCfg(c.archetype, c.num_layers, c.hidden, c.heads, c.ffn, c.vocab,
                     c.max_positions, c.seed)


def param_shapes(c: ModelConfig):
    """(name, shape) in canonical order: Model::for_each_param, src/model.cpp:178-209."""
    h, f = c.hidden, c.ffn
    out = [("token_embedding", (c.vocab, h)), ("position_embedding", (c.max_positions, h))]
    for l in range(c.num_layers):
        p = f"layers.{l}."
        out += [(p + "ln1.gamma", (h,)), (p + "ln1.beta", (h,)),
                (p + "attn.wq", (h, h)), (p + "attn.bq", (h,)),
                (p + "attn.wk", (h, h)), (p + "attn.bk", (h,)),
                (p + "attn.wv", (h, h)), (p + "attn.bv", (h,)),
                (p + "attn.wo", (h, h)), (p + "attn.bo", (h,)),
                (p + "ln2.gamma", (h,)), (p + "ln2.beta", (h,)),
                (p + "ffn.w1", (h, f)), (p + "ffn.b1", (f,)),
                (p + "ffn.w2", (f, h)), (p + "ffn.b2", (h,))]
    out += [("final_ln.gamma", (h,)), ("final_ln.beta", (h,))]
    if c.archetype == 0:
        out += [("pooler.weight", (h, h)), ("pooler.bias", (h,)),
                ("classifier.weight", (h, 2)), ("classifier.bias", (2,))]
    return out


def split_params(c: ModelConfig, flat: np.ndarray):
    """Views of a flat canonical buffer, one per parameter tensor."""
    views, off = [], 0
    for name, shape in param_shapes(c):
        n = int(np.prod(shape))
        views.append((name, flat[off:off + n].reshape(shape)))
        off += n
    assert off == flat.size
    return views


class Oracle:
    """The C restatement (oracle/prlab_oracle.c)."""

    def __init__(self, path: str = ORACLE_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing: run `make -C oracle`")
        L = self.lib = C.CDLL(path)
        L.or_round16.restype = C.c_float
        L.or_round16.argtypes = [C.c_float]
        L.or_f16_encode.restype = C.c_uint16
        L.or_f16_encode.argtypes = [C.c_float]
        L.or_f16_decode.restype = C.c_float
        L.or_f16_decode.argtypes = [C.c_uint16]
        L.or_param_count.restype = C.c_uint64
        L.or_param_count.argtypes = [C.POINTER(_ModelCfg)]
        L.or_build_model.argtypes = [C.POINTER(_ModelCfg), C.POINTER(C.c_float)]
        L.or_random_tokens.argtypes = [C.c_int64, C.c_int64, C.c_int64, C.c_uint64,
                                       C.POINTER(C.c_int32)]
        L.or_resolve_policy.argtypes = [C.c_char_p, C.POINTER(_Policy)]
        L.or_forward.argtypes = [C.POINTER(_ModelCfg), C.POINTER(C.c_float), C.POINTER(C.c_int32),
                                 C.c_int64, C.c_int64, C.POINTER(_Policy), C.POINTER(C.c_float),
                                 C.POINTER(C.c_uint64), C.POINTER(C.c_float)]
        L.or_matmul.argtypes = [C.POINTER(C.c_float), C.POINTER(C.c_float), C.c_int64, C.c_int64,
                                C.c_int64, _Kcfg, C.POINTER(C.c_float)]
        L.or_attention_scores.argtypes = [C.POINTER(C.c_float), C.POINTER(C.c_float), C.c_int64,
                                          C.c_int64, C.c_int64, C.c_float, _Kcfg,
                                          C.POINTER(C.c_float), C.POINTER(C.c_float)]
        L.or_softmax.argtypes = [C.POINTER(C.c_float), C.c_int64, C.c_int64, _Kcfg,
                                 C.POINTER(C.c_float)]
        L.or_layernorm.argtypes = [C.POINTER(C.c_float), C.c_int64, C.c_int64,
                                   C.POINTER(C.c_float), C.POINTER(C.c_float), C.c_float, _Kcfg,
                                   C.POINTER(C.c_float)]
        L.or_gelu.argtypes = [C.POINTER(C.c_float), C.c_int64, _Kcfg, C.POINTER(C.c_float)]
        L.or_add.argtypes = [C.POINTER(C.c_float), C.POINTER(C.c_float), C.c_int64, _Kcfg,
                             C.POINTER(C.c_float)]
        L.or_tanh.argtypes = [C.POINTER(C.c_float), C.c_int64, _Kcfg, C.POINTER(C.c_float)]
        L.or_embed.argtypes = [C.POINTER(C.c_float), C.c_int64, C.POINTER(C.c_float), C.c_int64,
                               C.c_int64, C.POINTER(C.c_int32), C.c_int64, C.c_int64, _Kcfg,
                               C.POINTER(C.c_float)]
        L.or_set_threads.argtypes = [C.c_int]
        L.or_classifier_probs.argtypes = [C.POINTER(_ModelCfg), C.POINTER(C.c_float),
                                          C.POINTER(C.c_int32), C.c_int64, C.c_int64,
                                          C.POINTER(_Policy), C.POINTER(C.c_float)]

    # --- lattice
    def round16(self, x: float) -> float:
        return self.lib.or_round16(x)

    def round16_array(self, x: np.ndarray) -> np.ndarray:
        f = np.vectorize(self.lib.or_round16, otypes=[np.float32])
        return f(np.asarray(x, dtype=np.float32))

    def f16_encode(self, x: float) -> int:
        return self.lib.or_f16_encode(x)

    def f16_decode(self, h: int) -> float:
        return self.lib.or_f16_decode(h)

    def set_threads(self, n: int):
        self.lib.or_set_threads(n)

    # --- policies
    def policy(self, name) -> _Policy:
        """A named policy (resolve_policy, src/policy.cpp:49-67) or a custom per-class
        assignment given as 7 (compute, accum, stabilized) triples in OpClass order
        (the outcome of policy_from_spec, src/policy.cpp:69-116)."""
        p = _Policy()
        if not isinstance(name, str):
            for i, (cmp_, acc, stab) in enumerate(name):
                p.cls[i] = _Kcfg(int(cmp_), int(acc), int(stab))
            return p
        if self.lib.or_resolve_policy(name.encode(), C.byref(p)) != 0:
            raise ValueError(f"unknown policy '{name}' (valid: fp32, full_fp16, hybrid)")
        return p

    # --- model
    def param_count(self, c: ModelConfig) -> int:
        m = _mcfg(c)
        return int(self.lib.or_param_count(C.byref(m)))

    def build_model(self, c: ModelConfig) -> np.ndarray:
        m = _mcfg(c)
        out = np.empty(self.param_count(c), dtype=np.float32)
        if self.lib.or_build_model(C.byref(m), _fp(out)) != 0:
            raise ValueError("invalid model config")
        return out

    def random_tokens(self, vocab: int, batch: int, seq: int, seed: int) -> np.ndarray:
        ids = np.empty(batch * seq, dtype=np.int32)
        self.lib.or_random_tokens(vocab, batch, seq, seed, _ip(ids))
        return ids

    def forward(self, c: ModelConfig, params: np.ndarray, ids: np.ndarray, batch: int, seq: int,
                policy: str, want_calls=False, retain_scores=False):
        m = _mcfg(c)
        pol = self.policy(policy)
        width = c.vocab if c.num_layers > 0 else c.hidden
        logits = np.empty((batch, seq, width), dtype=np.float32)
        calls = np.zeros(14, dtype=np.uint64)
        tap = (np.empty((c.num_layers, batch, c.heads, seq, seq), dtype=np.float32)
               if retain_scores else None)
        ids = np.ascontiguousarray(ids, dtype=np.int32)
        rc = self.lib.or_forward(C.byref(m), _fp(params), _ip(ids), batch, seq, C.byref(pol),
                                 _fp(logits), _up(calls), _fp(tap))
        if rc == -1:
            raise ValueError("invalid forward arguments")
        if rc == -2:
            raise IndexError("token id or sequence out of range")
        out = [logits]
        if want_calls:
            out.append(calls.reshape(7, 2))
        if retain_scores:
            out.append(tap)
        return out[0] if len(out) == 1 else tuple(out)

    # --- operators
    def classifier_probs(self, c: ModelConfig, params: np.ndarray, ids: np.ndarray, batch: int,
                         seq: int, policy: str) -> np.ndarray:
        """classifier_probs, src/model.cpp:484-526 (encoder_only)."""
        out = np.empty(batch, dtype=np.float32)
        pol = self.policy(policy)
        ids = np.ascontiguousarray(ids, dtype=np.int32)
        if self.lib.or_classifier_probs(C.byref(_mcfg(c)), _fp(params), _ip(ids), batch, seq,
                                        C.byref(pol), _fp(out)):
            raise ValueError("or_classifier_probs failed (encoder_only model, valid config)")
        return out

    @staticmethod
    def _k(compute, accum, stabilized=True):
        return _Kcfg(compute, accum, int(stabilized))

    def matmul(self, a, b, compute, accum):
        a = np.ascontiguousarray(a, np.float32)
        b = np.ascontiguousarray(b, np.float32)
        m, k = a.shape
        n = b.shape[1]
        out = np.empty((m, n), np.float32)
        if self.lib.or_matmul(_fp(a), _fp(b), m, k, n, self._k(compute, accum), _fp(out)):
            raise ValueError("invalid kernel config")
        return out

    def attention_scores(self, q, k, scale, compute, accum, capture=False):
        q = np.ascontiguousarray(q, np.float32)
        k = np.ascontiguousarray(k, np.float32)
        out = np.empty((q.shape[0], k.shape[0]), np.float32)
        tap = np.empty_like(out) if capture else None
        self.lib.or_attention_scores(_fp(q), _fp(k), q.shape[0], k.shape[0], q.shape[1], scale,
                                     self._k(compute, accum), _fp(out), _fp(tap))
        return (out, tap) if capture else out

    def softmax(self, x, compute, accum, stabilized=True):
        x = np.ascontiguousarray(x, np.float32)
        out = np.empty_like(x)
        n = x.shape[-1]
        self.lib.or_softmax(_fp(x), x.size // n, n, self._k(compute, accum, stabilized), _fp(out))
        return out

    def layernorm(self, x, gamma, beta, eps, compute, accum):
        x = np.ascontiguousarray(x, np.float32)
        out = np.empty_like(x)
        n = x.shape[-1]
        self.lib.or_layernorm(_fp(x), x.size // n, n, _fp(np.ascontiguousarray(gamma, np.float32)),
                              _fp(np.ascontiguousarray(beta, np.float32)), eps,
                              self._k(compute, accum), _fp(out))
        return out

    def gelu(self, x, compute, accum):
        x = np.ascontiguousarray(x, np.float32)
        out = np.empty_like(x)
        self.lib.or_gelu(_fp(x), x.size, self._k(compute, accum), _fp(out))
        return out

    def add(self, a, b, compute, accum):
        a = np.ascontiguousarray(a, np.float32)
        b = np.ascontiguousarray(b, np.float32)
        out = np.empty_like(a)
        self.lib.or_add(_fp(a), _fp(b), a.size, self._k(compute, accum), _fp(out))
        return out

    def tanh(self, x, compute, accum):
        x = np.ascontiguousarray(x, np.float32)
        out = np.empty_like(x)
        self.lib.or_tanh(_fp(x), x.size, self._k(compute, accum), _fp(out))
        return out

    def embed(self, tok, pos, ids, batch, seq, compute):
        tok = np.ascontiguousarray(tok, np.float32)
        pos = np.ascontiguousarray(pos, np.float32)
        ids = np.ascontiguousarray(ids, np.int32)
        h = tok.shape[1]
        out = np.empty((batch * seq, h), np.float32)
        rc = self.lib.or_embed(_fp(tok), tok.shape[0], _fp(pos), pos.shape[0], h, _ip(ids), batch,
                               seq, self._k(compute, compute), _fp(out))
        if rc == -2:
            raise IndexError("token id or sequence out of range")
        return out


def make_adversarial_params(orc: "Oracle", c: ModelConfig, probe_ids, batch: int, seq: int,
                            target: float = 30.0) -> np.ndarray:
    """Restatement of make_adversarial_model (src/fidelity.cpp:282-312) on the oracle:
    rescale layer-0 Wq/bq/Wk/bk by sqrt(target / max|layer-0 fp32 score|)."""
    if c.num_layers < 1:
        raise ValueError("adversarial construction needs >= 1 layer")
    p = orc.build_model(c)
    _, tap = orc.forward(c, p, probe_ids, batch, seq, "fp32", retain_scores=True)
    max_score = float(np.abs(tap[0].astype(np.float64)).max())
    if max_score == 0.0:
        raise ValueError("probe produced all-zero layer-0 scores; cannot rescale")
    s = np.float32(np.sqrt(target / max_score))
    views = dict(split_params(c, p))
    for name in ("layers.0.attn.wq", "layers.0.attn.bq", "layers.0.attn.wk", "layers.0.attn.bk"):
        views[name][...] = views[name] * s
    return p


class Reference:
    """The unmodified reference, compiled by oracle/Makefile (oracle/_ref/libprlab_ref.so)."""

    def __init__(self, path: str = REF_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing: run `make -C oracle ref` where "
                                    "/root/reference exists")
        L = self.lib = C.CDLL(path)
        L.ref_last_error.restype = C.c_char_p
        L.ref_round16.restype = C.c_float
        L.ref_round16.argtypes = [C.c_float]
        L.ref_f16_encode.restype = C.c_uint16
        L.ref_f16_encode.argtypes = [C.c_float]
        L.ref_param_count.restype = C.c_uint64
        L.ref_param_count.argtypes = [C.c_int] + [C.c_int64] * 6
        L.ref_build_model.argtypes = [C.c_int] + [C.c_int64] * 6 + [C.c_uint64, C.POINTER(C.c_float)]
        L.ref_random_tokens.argtypes = [C.c_int64, C.c_int64, C.c_int64, C.c_uint64,
                                        C.POINTER(C.c_int32)]
        L.ref_forward.argtypes = ([C.c_int] + [C.c_int64] * 6 +
                                  [C.POINTER(C.c_float), C.POINTER(C.c_int32), C.c_int64,
                                   C.c_int64, C.c_char_p, C.POINTER(C.c_float),
                                   C.POINTER(C.c_uint64), C.c_int])
        L.ref_matmul.argtypes = [C.POINTER(C.c_float), C.POINTER(C.c_float), C.c_int64, C.c_int64,
                                 C.c_int64, C.c_int, C.c_int, C.POINTER(C.c_float)]
        L.ref_softmax.argtypes = [C.POINTER(C.c_float), C.c_int64, C.c_int64, C.c_int, C.c_int,
                                  C.c_int, C.POINTER(C.c_float)]
        L.ref_layernorm.argtypes = [C.POINTER(C.c_float), C.c_int64, C.c_int64,
                                    C.POINTER(C.c_float), C.POINTER(C.c_float), C.c_float,
                                    C.c_int, C.c_int, C.POINTER(C.c_float)]
        L.ref_gelu.argtypes = [C.POINTER(C.c_float), C.c_int64, C.c_int, C.c_int,
                               C.POINTER(C.c_float)]
        L.ref_attention_scores.argtypes = [C.POINTER(C.c_float), C.POINTER(C.c_float), C.c_int64,
                                           C.c_int64, C.c_int64, C.c_float, C.c_int, C.c_int,
                                           C.POINTER(C.c_float), C.POINTER(C.c_float)]
        L.ref_embed.argtypes = [C.POINTER(C.c_float), C.c_int64, C.POINTER(C.c_float), C.c_int64,
                                C.c_int64, C.POINTER(C.c_int32), C.c_int64, C.c_int64, C.c_int,
                                C.POINTER(C.c_float)]

    @staticmethod
    def _c(c: ModelConfig):
        return (c.archetype, c.num_layers, c.hidden, c.heads, c.ffn, c.vocab, c.max_positions)

    def param_count(self, c: ModelConfig) -> int:
        return int(self.lib.ref_param_count(*self._c(c)))

    def build_model(self, c: ModelConfig) -> np.ndarray:
        out = np.empty(self.param_count(c), dtype=np.float32)
        if self.lib.ref_build_model(*self._c(c), c.seed, _fp(out)):
            raise ValueError(self.lib.ref_last_error().decode())
        return out

    def random_tokens(self, vocab, batch, seq, seed) -> np.ndarray:
        ids = np.empty(batch * seq, dtype=np.int32)
        self.lib.ref_random_tokens(vocab, batch, seq, seed, _ip(ids))
        return ids

    def forward(self, c: ModelConfig, params, ids, batch, seq, policy, want_calls=False,
                threads=1):
        width = c.vocab if c.num_layers > 0 else c.hidden
        logits = np.empty((batch, seq, width), dtype=np.float32)
        calls = np.zeros(14, dtype=np.uint64)
        ids = np.ascontiguousarray(ids, dtype=np.int32)
        rc = self.lib.ref_forward(*self._c(c), _fp(params), _ip(ids), batch, seq,
                                  policy.encode(), _fp(logits), _up(calls), threads)
        if rc:
            msg = self.lib.ref_last_error().decode()
            raise (IndexError if rc == -2 else ValueError)(msg)
        return (logits, calls.reshape(7, 2)) if want_calls else logits

    # ---- prebuilt reference Model (built once, outside any timed region) ----
    def model_build(self, c: ModelConfig):
        """prlab::build_model(config) held on the C++ side (src/model.cpp:217-265); returns a handle."""
        L = self.lib
        L.ref_model_build.restype = C.c_void_p
        L.ref_model_build.argtypes = [C.c_int] + [C.c_int64] * 6 + [C.c_uint64]
        h = L.ref_model_build(*self._c(c), c.seed)
        if not h:
            raise ValueError(L.ref_last_error().decode())
        return h

    def model_free(self, h):
        self.lib.ref_model_free.argtypes = [C.c_void_p]
        self.lib.ref_model_free(h)

    def benchmark_forward(self, h, ids, batch, seq, policy, warmup, measure):
        """The reference's own prlab::benchmark_forward (src/bench.cpp:47-106), single thread:
        dict(mean_s, p50_s, p95_s, throughput_sps, samples_s)."""
        L = self.lib
        L.ref_benchmark_forward.argtypes = [C.c_void_p, C.POINTER(C.c_int32), C.c_int64, C.c_int64,
                                            C.c_char_p, C.c_int64, C.c_int64, C.POINTER(C.c_double),
                                            C.POINTER(C.c_double)]
        out = np.zeros(4, dtype=np.float64)
        smp = np.zeros(max(1, measure), dtype=np.float64)
        ids = np.ascontiguousarray(ids, dtype=np.int32)
        if L.ref_benchmark_forward(h, _ip(ids), batch, seq, policy.encode(), warmup, measure,
                                   out.ctypes.data_as(C.POINTER(C.c_double)),
                                   smp.ctypes.data_as(C.POINTER(C.c_double))):
            raise ValueError(L.ref_last_error().decode())
        return {"mean_s": out[0], "p50_s": out[1], "p95_s": out[2], "throughput_sps": out[3],
                "samples_s": smp.tolist()}

    def forward_threads(self, h, ids, batch, seq, policy, threads, want_logits=False, width=None):
        """`batch` independent batch-1 prlab::forward calls on `threads` host threads over the
        prebuilt Model; returns (seconds of the forwards only, logits or None)."""
        L = self.lib
        L.ref_forward_threads.argtypes = [C.c_void_p, C.POINTER(C.c_int32), C.c_int64, C.c_int64,
                                          C.c_char_p, C.c_int, C.POINTER(C.c_float),
                                          C.POINTER(C.c_double)]
        ids = np.ascontiguousarray(ids, dtype=np.int32)
        logits = np.empty((batch, seq, width), dtype=np.float32) if want_logits else None
        sec = C.c_double(0.0)
        if L.ref_forward_threads(h, _ip(ids), batch, seq, policy.encode(), threads, _fp(logits),
                                 C.byref(sec)):
            raise ValueError(L.ref_last_error().decode())
        return sec.value, logits

    def forward_scores(self, c: ModelConfig, params, ids, batch, seq, policy):
        """prlab::forward(..., retain_scores=true): (logits, [L,B,H,S,S] fp32 taps)."""
        L = self.lib
        L.ref_forward_scores.argtypes = ([C.c_int] + [C.c_int64] * 6 +
                                         [C.POINTER(C.c_float), C.POINTER(C.c_int32), C.c_int64,
                                          C.c_int64, C.c_char_p, C.POINTER(C.c_float),
                                          C.POINTER(C.c_float)])
        width = c.vocab if c.num_layers > 0 else c.hidden
        logits = np.empty((batch, seq, width), dtype=np.float32)
        taps = np.empty((c.num_layers, batch, c.heads, seq, seq), dtype=np.float32)
        ids = np.ascontiguousarray(ids, dtype=np.int32)
        if L.ref_forward_scores(*self._c(c), _fp(params), _ip(ids), batch, seq, policy.encode(),
                                _fp(logits), _fp(taps)):
            raise ValueError(L.ref_last_error().decode())
        return logits, taps

    def classifier_probs(self, c: ModelConfig, params, ids, batch, seq, policy):
        """prlab::classifier_probs (src/model.cpp:484-526)."""
        L = self.lib
        L.ref_classifier_probs.argtypes = ([C.c_int] + [C.c_int64] * 6 +
                                           [C.POINTER(C.c_float), C.POINTER(C.c_int32), C.c_int64,
                                            C.c_int64, C.c_char_p, C.POINTER(C.c_float)])
        out = np.empty(batch, dtype=np.float32)
        ids = np.ascontiguousarray(ids, dtype=np.int32)
        if L.ref_classifier_probs(*self._c(c), _fp(params), _ip(ids), batch, seq, policy.encode(),
                                  _fp(out)):
            raise ValueError(L.ref_last_error().decode())
        return out

    def perplexity(self, c: ModelConfig, params, stream, context_len, policy) -> float:
        """prlab::perplexity (src/fidelity.cpp:248-279)."""
        L = self.lib
        L.ref_perplexity.argtypes = ([C.c_int] + [C.c_int64] * 6 +
                                     [C.POINTER(C.c_float), C.POINTER(C.c_int32), C.c_int64, C.c_int64,
                                      C.c_char_p, C.POINTER(C.c_double)])
        out = C.c_double()
        stream = np.ascontiguousarray(stream, dtype=np.int32)
        if L.ref_perplexity(*self._c(c), _fp(params), _ip(stream), stream.size, context_len,
                            policy.encode(), C.byref(out)):
            raise ValueError(L.ref_last_error().decode())
        return out.value

    def serialize_checkpoint(self, c: ModelConfig, params, path: str, f16: bool = False):
        """prlab::serialize_checkpoint (src/checkpoint.cpp:104-121)."""
        L = self.lib
        L.ref_serialize_checkpoint.argtypes = ([C.c_int] + [C.c_int64] * 6 +
                                               [C.c_uint64, C.POINTER(C.c_float), C.c_int, C.c_char_p])
        if L.ref_serialize_checkpoint(*self._c(c), c.seed, _fp(params), int(f16), path.encode()):
            raise ValueError(L.ref_last_error().decode())

    def load_checkpoint(self, path: str, c: ModelConfig) -> np.ndarray:
        """prlab::load_checkpoint (src/checkpoint.cpp:133-162) -> flat canonical params."""
        L = self.lib
        L.ref_load_checkpoint.argtypes = [C.c_char_p, C.POINTER(C.c_float), C.c_int64]
        out = np.empty(self.param_count(c), dtype=np.float32)
        if L.ref_load_checkpoint(path.encode(), _fp(out), out.size):
            raise ValueError(L.ref_last_error().decode())
        return out

    def make_adversarial_model(self, c: ModelConfig, probe_ids, batch, seq, target=30.0):
        L = self.lib
        L.ref_make_adversarial_model.argtypes = ([C.c_int] + [C.c_int64] * 6 +
                                                 [C.c_uint64, C.POINTER(C.c_int32), C.c_int64,
                                                  C.c_int64, C.c_float, C.POINTER(C.c_float)])
        out = np.empty(self.param_count(c), dtype=np.float32)
        ids = np.ascontiguousarray(probe_ids, np.int32)
        if L.ref_make_adversarial_model(*self._c(c), c.seed, _ip(ids), batch, seq, target, _fp(out)):
            raise ValueError(L.ref_last_error().decode())
        return out

    def matmul(self, a, b, compute, accum):
        a = np.ascontiguousarray(a, np.float32)
        b = np.ascontiguousarray(b, np.float32)
        out = np.empty((a.shape[0], b.shape[1]), np.float32)
        if self.lib.ref_matmul(_fp(a), _fp(b), a.shape[0], a.shape[1], b.shape[1], compute,
                               accum, _fp(out)):
            raise ValueError(self.lib.ref_last_error().decode())
        return out

    def softmax(self, x, compute, accum, stabilized=True):
        x = np.ascontiguousarray(x, np.float32)
        out = np.empty_like(x)
        n = x.shape[-1]
        self.lib.ref_softmax(_fp(x), x.size // n, n, compute, accum, int(stabilized), _fp(out))
        return out

    def layernorm(self, x, gamma, beta, eps, compute, accum):
        x = np.ascontiguousarray(x, np.float32)
        out = np.empty_like(x)
        n = x.shape[-1]
        self.lib.ref_layernorm(_fp(x), x.size // n, n, _fp(np.ascontiguousarray(gamma, np.float32)),
                               _fp(np.ascontiguousarray(beta, np.float32)), eps, compute, accum,
                               _fp(out))
        return out

    def gelu(self, x, compute, accum):
        x = np.ascontiguousarray(x, np.float32)
        out = np.empty_like(x)
        self.lib.ref_gelu(_fp(x), x.size, compute, accum, _fp(out))
        return out

    def attention_scores(self, q, k, scale, compute, accum, capture=False):
        q = np.ascontiguousarray(q, np.float32)
        k = np.ascontiguousarray(k, np.float32)
        out = np.empty((q.shape[0], k.shape[0]), np.float32)
        tap = np.empty_like(out) if capture else None
        self.lib.ref_attention_scores(_fp(q), _fp(k), q.shape[0], k.shape[0], q.shape[1], scale,
                                      compute, accum, _fp(out), _fp(tap))
        return (out, tap) if capture else out

    def embed(self, tok, pos, ids, batch, seq, compute):
        tok = np.ascontiguousarray(tok, np.float32)
        pos = np.ascontiguousarray(pos, np.float32)
        ids = np.ascontiguousarray(ids, np.int32)
        out = np.empty((batch * seq, tok.shape[1]), np.float32)
        rc = self.lib.ref_embed(_fp(tok), tok.shape[0], _fp(pos), pos.shape[0], tok.shape[1],
                                _ip(ids), batch, seq, compute, _fp(out))
        if rc == -2:
            raise IndexError(self.lib.ref_last_error().decode())
        return out


def compare_logits(baseline: np.ndarray, candidate: np.ndarray) -> dict:
    """Restatement of compare_logits (src/fidelity.cpp:11-37), in float64."""
    b = np.asarray(baseline, np.float64).ravel()
    c = np.asarray(candidate, np.float64).ravel()
    if b.shape != c.shape:
        raise ValueError("logit shapes differ")
    cand_nonfinite = int((~np.isfinite(c)).sum())
    ok = np.isfinite(b) & np.isfinite(c)
    b, c = b[ok], c[ok]
    r = {"max_abs_error": 0.0, "mean_abs_error": 0.0, "cosine": None,
         "finite_pairs": int(ok.sum()), "candidate_nonfinite": cand_nonfinite,
         "nan_affected": cand_nonfinite > 0}
    if b.size:
        d = np.abs(b - c)
        r["max_abs_error"] = float(d.max())
        r["mean_abs_error"] = float(d.mean())
        na, nb = float((b * b).sum()), float((c * c).sum())
        if na > 0 and nb > 0:
            r["cosine"] = float((b * c).sum() / (np.sqrt(na) * np.sqrt(nb)))
    return r


def window_nll_sum(logits: np.ndarray, window: np.ndarray) -> float:
    """window_nll_sum (src/fidelity.cpp:213-240) restated in numpy double: positions
    0..S-2 predict their successors; max-stabilised log-softmax; a non-finite row max
    poisons the sum with NaN."""
    seq, vocab = logits.shape[-2], logits.shape[-1]
    rows = logits.reshape(seq, vocab)
    nll = 0.0
    for t in range(seq - 1):
        row = rows[t].astype(np.float64)
        mx = np.max(row) if not np.isnan(row).all() else np.nan
        if not np.isfinite(mx):
            return float("nan")
        denom = float(np.sum(np.exp(row - mx)))
        nll -= (row[int(window[t + 1])] - mx) - np.log(denom)
    return float(nll)


def perplexity_windows(forward_fn, stream: np.ndarray, context_len: int) -> float:
    """perplexity (src/fidelity.cpp:248-279) over a forward_fn(ids, seq) -> [1, seq, V]."""
    nll, predicted = 0.0, 0
    for off in range(0, len(stream), context_len):
        n = min(context_len, len(stream) - off)
        if n < 2:
            break
        w = stream[off:off + n]
        nll += window_nll_sum(forward_fn(w, n), w)
        predicted += n - 1
    return float(np.exp(nll / predicted))
