"""B200-native prlab forward: Python mirror of the reference operator API.

The product is the C-ABI library ``_lib/libprlab_gpu.so`` (hand-written sm_100a
CUDA kernels + C++ runtime, declared in ``include/prlab_gpu.h``).  This module
is a thin ctypes binding that mirrors the reference's C++ API
(``include/prlab/{kernels,model,policy}.hpp``) with the same names, argument
meaning and error behaviour (``std::invalid_argument`` -> ``ValueError``,
``std::out_of_range`` -> ``IndexError``, ``std::runtime_error`` ->
``RuntimeError``), so tests read like the reference's own tests.

There is no CPU fallback: importing works anywhere, but every compute call
goes through the CUDA library and fails loudly without it or without a GPU.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass
from typing import Optional, Sequence

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# PRLAB_GPU_LIB: an alternative build of the same library (A/B timing of kernel variants)
LIB_PATH = os.environ.get("PRLAB_GPU_LIB") or os.path.join(_HERE, "_lib", "libprlab_gpu.so")
HEADER_PATH = os.path.join(os.path.dirname(_HERE), "include", "prlab_gpu.h")

F32, F16E = 0, 1
OP_CLASSES = ["Linear", "AttentionScoreMatmul", "Softmax", "LayerNorm", "Activation",
              "Embedding", "Residual"]
OUT_F32, OUT_F16 = 0, 1
FWD_RETAIN_SCORES, FWD_TIMED = 1, 2

PRLAB_OK, PRLAB_EINVAL, PRLAB_ERANGE, PRLAB_ERUNTIME, PRLAB_ECUDA = range(5)


class CudaError(RuntimeError):
    """A CUDA failure inside the library (PRLAB_ECUDA) -- std::runtime_error in the reference."""


class KernelConfig(C.Structure):
    """Reference KernelConfig (include/prlab/kernels.hpp:16-22)."""
    _fields_ = [("compute", C.c_int32), ("accum", C.c_int32), ("stabilized", C.c_int32)]

    def __init__(self, compute=F32, accum=F32, stabilized=True):
        super().__init__(compute, accum, int(bool(stabilized)))

    def __repr__(self):
        n = ["f32", "f16e"]
        return f"KernelConfig({n[self.compute]}, {n[self.accum]}, stabilized={bool(self.stabilized)})"


class PrecisionPolicy(C.Structure):
    """Reference PrecisionPolicy assignment (include/prlab/policy.hpp:43-56)."""
    _fields_ = [("cls", KernelConfig * 7)]

    def config_for(self, op_class) -> KernelConfig:
        i = OP_CLASSES.index(op_class) if isinstance(op_class, str) else int(op_class)
        return self.cls[i]


class _ModelDesc(C.Structure):
    _fields_ = [("archetype", C.c_int32), ("num_layers", C.c_int64), ("hidden", C.c_int64),
                ("heads", C.c_int64), ("ffn", C.c_int64), ("vocab", C.c_int64),
                ("max_positions", C.c_int64), ("seed", C.c_uint64)]


class LogitComparison(C.Structure):
    """compare_logits result (include/prlab/fidelity.hpp:20-27)."""
    _fields_ = [("max_abs_error", C.c_double), ("mean_abs_error", C.c_double), ("cosine", C.c_double),
                ("has_cosine", C.c_int32), ("finite_pairs", C.c_uint64),
                ("candidate_nonfinite", C.c_uint64), ("nan_affected", C.c_int32)]

    def as_dict(self):
        return {"max_abs_error": self.max_abs_error, "mean_abs_error": self.mean_abs_error,
                "cosine": self.cosine if self.has_cosine else None,
                "finite_pairs": int(self.finite_pairs),
                "candidate_nonfinite": int(self.candidate_nonfinite),
                "nan_affected": bool(self.nan_affected)}


class MemoryReport(C.Structure):
    _fields_ = [("weights_fast", C.c_uint64), ("weights_fp32", C.c_uint64), ("workspace", C.c_uint64),
                ("logits", C.c_uint64), ("scratch", C.c_uint64), ("total", C.c_uint64)]

    def as_dict(self):
        return {k: int(getattr(self, k)) for k, _ in self._fields_}


class Trace(C.Structure):
    """Reference ForwardTrace instrumentation (include/prlab/model.hpp:113-125)."""
    _fields_ = [("seconds", C.c_double * 7), ("kernel_calls", (C.c_uint64 * 2) * 7)]

    def calls(self, op_class, dtype) -> int:
        i = OP_CLASSES.index(op_class) if isinstance(op_class, str) else int(op_class)
        return int(self.kernel_calls[i][dtype])


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

    @property
    def head_dim(self) -> int:
        return self.hidden // self.heads

    def replace(self, **kw) -> "ModelConfig":
        d = dict(self.__dict__)
        d.update(kw)
        return ModelConfig(**d)

    # presets, src/model.cpp:122-136
    @staticmethod
    def bert_base():
        return ModelConfig(0, 12, 768, 12, 3072, 30522, 512)

    @staticmethod
    def gpt2_small():
        return ModelConfig(1, 12, 768, 12, 3072, 50257, 1024)

    @staticmethod
    def encoder_toy():
        return ModelConfig(0, 4, 128, 4, 256, 320, 160)

    @staticmethod
    def decoder_toy():
        return ModelConfig(1, 4, 128, 4, 256, 320, 160)

    @staticmethod
    def preset(name: str) -> "ModelConfig":
        table = {"bert_base": ModelConfig.bert_base, "gpt2_small": ModelConfig.gpt2_small,
                 "encoder_toy": ModelConfig.encoder_toy, "decoder_toy": ModelConfig.decoder_toy}
        if name not in table:
            raise ValueError(f"unknown model preset '{name}' (valid: bert_base, gpt2_small, "
                             "encoder_toy, decoder_toy)")
        return table[name]()

    def _desc(self) -> _ModelDesc:
        return _ModelDesc(self.archetype, self.num_layers, self.hidden, self.heads, self.ffn,
                          self.vocab, self.max_positions, self.seed)


_lib: Optional[C.CDLL] = None

# (name, restype, argtypes) for every entry point of include/prlab_gpu.h
_P = C.c_void_p
_FP = C.POINTER(C.c_float)
_IP = C.POINTER(C.c_int32)
EXPORTS = [
    ("prlab_gpu_last_error", C.c_char_p, []),
    ("prlab_gpu_abi_version", C.c_int, []),
    ("prlab_gpu_resolve_policy", C.c_int, [C.c_char_p, C.POINTER(PrecisionPolicy)]),
    ("prlab_gpu_validate_policy", C.c_int, [C.POINTER(PrecisionPolicy)]),
    ("prlab_gpu_model_create", C.c_int, [C.POINTER(_ModelDesc), C.POINTER(_FP), C.c_int64,
                                         C.c_int, C.POINTER(_P)]),
    ("prlab_gpu_model_create_flat", C.c_int, [C.POINTER(_ModelDesc), _FP, C.c_int, C.POINTER(_P)]),
    ("prlab_gpu_model_destroy", None, [_P]),
    ("prlab_gpu_model_memory", C.c_int, [_P, C.POINTER(C.c_uint64), C.POINTER(C.c_uint64)]),
    ("prlab_gpu_model_memory_ex", C.c_int, [_P, C.POINTER(MemoryReport)]),
    ("prlab_gpu_build_model", C.c_int, [C.POINTER(_ModelDesc), _FP, C.c_int64]),
    ("prlab_gpu_param_count", C.c_uint64, [C.POINTER(_ModelDesc)]),
    ("prlab_gpu_random_tokens", C.c_int, [C.c_int64, C.c_int64, C.c_int64, C.c_uint64, _IP]),
    ("prlab_gpu_argmax_device", C.c_int, [_P, C.c_int32, C.c_int64, C.c_int64, C.c_int64, _P, _P]),
    ("prlab_gpu_forward", C.c_int, [_P, _IP, C.c_int64, C.c_int64, C.POINTER(PrecisionPolicy),
                                    _FP, C.POINTER(Trace)]),
    ("prlab_gpu_forward_ex", C.c_int, [_P, _IP, C.c_int64, C.c_int64, C.POINTER(PrecisionPolicy),
                                       C.c_int32, _FP, C.POINTER(Trace), _FP]),
    ("prlab_gpu_row_nll_device", C.c_int, [_P, C.c_int32, C.c_int64, C.c_int64, C.c_int64, _P, _P,
                                           _P, _P]),
    ("prlab_gpu_compare_logits_device", C.c_int, [_P, C.c_int32, C.c_int64, _P, C.c_int32, C.c_int64,
                                                  C.c_int64, C.c_int64, _P, C.POINTER(LogitComparison)]),
    ("prlab_gpu_perplexity", C.c_int, [_P, _IP, C.c_int64, C.c_int64, C.POINTER(PrecisionPolicy),
                                       C.POINTER(C.c_double)]),
    ("prlab_gpu_model_load_checkpoint", C.c_int, [C.c_char_p, C.c_int, _P, C.POINTER(C.c_void_p)]),
    ("prlab_gpu_classifier_probs", C.c_int, [_P, _IP, C.c_int64, C.c_int64,
                                             C.POINTER(PrecisionPolicy), _FP]),
    ("prlab_gpu_forward_device", C.c_int, [_P, _P, C.c_int64, C.c_int64,
                                           C.POINTER(PrecisionPolicy), _P, C.c_int32, C.c_int64,
                                           _P, C.c_int32]),
    ("prlab_gpu_forward_trunk_device", C.c_int, [_P, _P, C.c_int64, C.c_int64,
                                                 C.POINTER(PrecisionPolicy), _P, C.POINTER(C.c_int64)]),
    ("prlab_gpu_forward_nll_device", C.c_int, [_P, _P, _P, C.c_int64, C.c_int64, C.POINTER(PrecisionPolicy),
                                               _P, _P, _P, C.POINTER(C.c_int32)]),
    ("prlab_gpu_sync_status", C.c_int, [_P, _P]),
    ("prlab_gpu_forward_kernel_count", C.c_int, [_P, C.c_int64, C.c_int64,
                                                 C.POINTER(PrecisionPolicy),
                                                 C.POINTER(C.c_int64)]),
    ("prlab_gpu_forward_kernel_count_ex", C.c_int, [_P, C.c_int64, C.c_int64,
                                                    C.POINTER(PrecisionPolicy), C.c_int32,
                                                    C.POINTER(C.c_int64)]),
    ("prlab_gpu_debug_embedding_device", C.c_int, [_P, _P, C.c_int64, C.c_int64, C.c_int32, _P, _P]),
    ("prlab_gpu_host_copy_mode", C.c_int, [_P, C.c_int64, C.c_int64, C.POINTER(PrecisionPolicy),
                                           C.POINTER(C.c_int32)]),
    ("prlab_gpu_matmul", C.c_int, [_FP, _FP, C.c_int64, C.c_int64, C.c_int64, KernelConfig, _FP]),
    ("prlab_gpu_attention_scores", C.c_int, [_FP, _FP, C.c_int64, C.c_int64, C.c_int64, C.c_float,
                                             KernelConfig, _FP, _FP]),
    ("prlab_gpu_softmax", C.c_int, [_FP, C.c_int64, C.c_int64, KernelConfig, _FP]),
    ("prlab_gpu_layernorm", C.c_int, [_FP, C.c_int64, C.c_int64, _FP, _FP, C.c_float,
                                      KernelConfig, _FP]),
    ("prlab_gpu_gelu", C.c_int, [_FP, C.c_int64, KernelConfig, _FP]),
    ("prlab_gpu_add", C.c_int, [_FP, _FP, C.c_int64, KernelConfig, _FP]),
    ("prlab_gpu_tanh", C.c_int, [_FP, C.c_int64, KernelConfig, _FP]),
    ("prlab_gpu_embed", C.c_int, [_FP, C.c_int64, _FP, C.c_int64, C.c_int64, _IP, C.c_int64,
                                  C.c_int64, KernelConfig, _FP]),
    ("prlab_gpu_linear_f16_device", C.c_int, [_P, _P, _P, _P, C.c_int64, C.c_int64, C.c_int64,
                                              C.c_int64, C.c_int32, _P]),
    ("prlab_gpu_linear_f16_device_ex", C.c_int, [_P, _P, _P, _P, C.c_int64, C.c_int64, C.c_int64,
                                                 C.c_int64, C.c_int32, C.c_int32, C.c_int32,
                                                 C.c_int32, _P]),
    ("prlab_gpu_linear_f32_device", C.c_int, [_P, _P, _P, _P, C.c_int64, C.c_int64, C.c_int64,
                                              C.c_int32, _P, _P]),
    ("prlab_gpu_attention_f16_device", C.c_int, [_P, _P, C.c_int64, C.c_int64, C.c_int64,
                                                 C.c_int64, C.c_int32, _P]),
    ("prlab_gpu_debug_gemm_stamps", C.c_int, [_P]),
    ("prlab_gpu_debug_small_stamps", C.c_int, [_P]),
    ("prlab_gpu_debug_cluster_stamps", C.c_int, [_P]),
    ("prlab_gpu_attention_f16_device_dbg", C.c_int, [_P, _P, C.c_int64, C.c_int64, C.c_int64,
                                                     C.c_int64, C.c_int32, _P, _P]),
]


def lib() -> C.CDLL:
    """Load the CUDA library (raises if it was not built -- there is no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"{LIB_PATH} is missing: build it with "
                               "`make -C paper_2603_28708_b200` (or __graft_entry__.build())")
        L = C.CDLL(LIB_PATH)
        for name, res, args in EXPORTS:
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def _check(rc: int):
    if rc == PRLAB_OK:
        return
    msg = lib().prlab_gpu_last_error().decode()
    if rc == PRLAB_EINVAL:
        raise ValueError(msg)
    if rc == PRLAB_ERANGE:
        raise IndexError(msg)
    if rc == PRLAB_ECUDA:
        raise CudaError(msg)
    raise RuntimeError(msg)


def _f(a):
    return a.ctypes.data_as(_FP) if a is not None else None


def _arr(x, dtype=np.float32):
    return np.ascontiguousarray(x, dtype=dtype)


# ---------------------------------------------------------------------------
# policies (src/policy.cpp)
# ---------------------------------------------------------------------------
def resolve_policy(name: str) -> PrecisionPolicy:
    p = PrecisionPolicy()
    _check(lib().prlab_gpu_resolve_policy(name.encode(), C.byref(p)))
    return p


def policy_from_classes(base: str = "hybrid", overrides: Optional[dict] = None) -> PrecisionPolicy:
    """policy_from_spec (src/policy.cpp:69-116) for {"base": ..., "overrides": {...}} specs."""
    p = resolve_policy(base)
    for key, entry in (overrides or {}).items():
        if key not in OP_CLASSES:
            raise ValueError(f"policy overrides names unknown op class '{key}'")
        c = p.cls[OP_CLASSES.index(key)]
        names = {"f32": F32, "f16e": F16E}
        if "compute" in entry:
            c.compute = names[entry["compute"]]
        if "accum" in entry:
            c.accum = names[entry["accum"]]
        if "stabilized" in entry:
            c.stabilized = int(bool(entry["stabilized"]))
    _check(lib().prlab_gpu_validate_policy(C.byref(p)))
    return p


def _policy(p) -> PrecisionPolicy:
    return resolve_policy(p) if isinstance(p, str) else p


# ---------------------------------------------------------------------------
# fixture generators (src/model.cpp:217-296), host side of the library
# ---------------------------------------------------------------------------
def param_count(cfg: ModelConfig) -> int:
    d = cfg._desc()
    return int(lib().prlab_gpu_param_count(C.byref(d)))


def build_model(cfg: ModelConfig) -> np.ndarray:
    """Flat canonical-order parameters, bit-identical to the reference build_model()."""
    d = cfg._desc()
    out = np.empty(param_count(cfg), np.float32)
    _check(lib().prlab_gpu_build_model(C.byref(d), _f(out), out.size))
    return out


def random_tokens(vocab: int, batch: int, seq: int, seed: int) -> np.ndarray:
    ids = np.empty(batch * seq, np.int32)
    _check(lib().prlab_gpu_random_tokens(vocab, batch, seq, seed, ids.ctypes.data_as(_IP)))
    return ids


def argmax_device(d_logits: int, dtype: int, rows: int, n: int, ld: int, d_tokens: int,
                  stream: int = 0):
    _check(lib().prlab_gpu_argmax_device(C.c_void_p(d_logits), dtype, rows, n, ld,
                                         C.c_void_p(d_tokens), C.c_void_p(stream)))


def _check_ids(ids: np.ndarray, batch: int, seq: int):
    if batch < 0 or seq < 0 or ids.size != batch * seq:
        raise ValueError(f"token batch holds {ids.size} ids, expected batch*seq = {batch}*{seq}")


# ---------------------------------------------------------------------------
# model + forward (src/model.cpp)
# ---------------------------------------------------------------------------
class DeviceModel:
    """A model uploaded into the device arena (fp16 K-major linears, fp32 LN/bias/tables)."""

    def __init__(self, config: ModelConfig, params: np.ndarray, device: int = 0):
        self.config = config
        flat = _arr(params)
        want = param_count(config)
        if flat.size != want:  # the C entry point walks param_sizes(desc) over the pointer
            raise ValueError(f"expected {want} parameters for this config, got {flat.size}")
        h = C.c_void_p()
        d = config._desc()
        _check(lib().prlab_gpu_model_create_flat(C.byref(d), _f(flat), device, C.byref(h)))
        self._h = h

    @classmethod
    def from_checkpoint(cls, path: str, device: int = 0) -> "DeviceModel":
        """load_checkpoint (src/checkpoint.cpp:133-162) straight into the device arena."""
        self = cls.__new__(cls)
        h = C.c_void_p()
        d = _ModelDesc()
        _check(lib().prlab_gpu_model_load_checkpoint(path.encode(), device, C.byref(d), C.byref(h)))
        self._h = h
        self.config = ModelConfig(archetype=d.archetype, num_layers=d.num_layers, hidden=d.hidden,
                                  heads=d.heads, ffn=d.ffn, vocab=d.vocab,
                                  max_positions=d.max_positions, seed=d.seed)
        return self

    def close(self):
        if getattr(self, "_h", None):
            lib().prlab_gpu_model_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def memory(self):
        w, ws = C.c_uint64(), C.c_uint64()
        _check(lib().prlab_gpu_model_memory(self._h, C.byref(w), C.byref(ws)))
        return int(w.value), int(ws.value)

    def memory_report(self) -> dict:
        """Device bytes by purpose (prlab_gpu_model_memory_ex)."""
        r = MemoryReport()
        _check(lib().prlab_gpu_model_memory_ex(self._h, C.byref(r)))
        return r.as_dict()

    def forward(self, ids, batch: int, seq: int, policy="hybrid", want_trace=False):
        """Drop-in forward (src/model.cpp:456-482): host ids -> host fp32 logits [B,S,V]."""
        cfg = self.config
        ids = _arr(ids, np.int32)
        _check_ids(ids, batch, seq)
        width = cfg.vocab if cfg.num_layers > 0 else cfg.hidden
        logits = np.empty((batch, seq, width), np.float32)
        tr = Trace()
        pol = _policy(policy)
        _check(lib().prlab_gpu_forward(self._h, ids.ctypes.data_as(_IP), batch, seq,
                                       C.byref(pol), _f(logits), C.byref(tr)))
        return (logits, tr) if want_trace else logits

    def forward_ex(self, ids, batch: int, seq: int, policy="hybrid", retain_scores=False,
                   timed=False):
        """forward with the reference's optional outputs: (logits, Trace, layer_scores or None);
        layer_scores [L,B,H,S,S] fp32 pre-mask taps (ForwardTrace::layer_scores)."""
        cfg = self.config
        ids = _arr(ids, np.int32)
        _check_ids(ids, batch, seq)
        width = cfg.vocab if cfg.num_layers > 0 else cfg.hidden
        logits = np.empty((batch, seq, width), np.float32)
        scores = (np.empty((cfg.num_layers, batch, cfg.heads, seq, seq), np.float32)
                  if retain_scores else None)
        tr = Trace()
        pol = _policy(policy)
        flags = (FWD_RETAIN_SCORES if retain_scores else 0) | (FWD_TIMED if timed else 0)
        _check(lib().prlab_gpu_forward_ex(self._h, ids.ctypes.data_as(_IP), batch, seq,
                                          C.byref(pol), flags, _f(logits), C.byref(tr),
                                          _f(scores) if scores is not None else None))
        return logits, tr, scores

    def classifier_probs(self, ids, batch: int, seq: int, policy="hybrid") -> np.ndarray:
        """classifier_probs (src/model.cpp:484-526): positive-class probability per row."""
        ids = _arr(ids, np.int32)
        _check_ids(ids, batch, seq)
        out = np.empty(batch, np.float32)
        pol = _policy(policy)
        _check(lib().prlab_gpu_classifier_probs(self._h, ids.ctypes.data_as(_IP), batch, seq,
                                                C.byref(pol), _f(out)))
        return out

    def perplexity(self, tokens, context_len: int, policy="hybrid") -> float:
        """perplexity (src/fidelity.cpp:248-279) with the NLL reduced on the device."""
        tokens = _arr(tokens, np.int32)
        out = C.c_double()
        pol = _policy(policy)
        _check(lib().prlab_gpu_perplexity(self._h, tokens.ctypes.data_as(_IP), tokens.size, context_len,
                                          C.byref(pol), C.byref(out)))
        return float(out.value)

    def forward_device(self, d_ids: int, batch: int, seq: int, policy, d_out: int,
                       out_dtype: int, ld: int, stream: int = 0, use_graph: bool = True):
        """Device-resident forward: raw device pointers (e.g. torch .data_ptr())."""
        pol = _policy(policy)
        _check(lib().prlab_gpu_forward_device(self._h, C.c_void_p(d_ids), batch, seq,
                                              C.byref(pol), C.c_void_p(d_out), out_dtype, ld,
                                              C.c_void_p(stream), int(use_graph)))

    def forward_trunk_device(self, d_ids: int, batch: int, seq: int, policy="hybrid", stream: int = 0) -> int:
        """The trunk alone (embeddings .. final LN, model.cpp:350 forward_hidden) on
        `stream`; returns the number of kernels launched (timing helper)."""
        n = C.c_int64()
        _check(lib().prlab_gpu_forward_trunk_device(self._h, C.c_void_p(d_ids), batch, seq,
                                                    C.byref(_policy(policy)), C.c_void_p(stream),
                                                    C.byref(n)))
        return int(n.value)

    def forward_nll_device(self, d_ids: int, d_targets: int, batch: int, seq: int, policy, d_nll: int,
                           d_argmax: int, stream: int = 0) -> bool:
        """Per-row next-token NLL (double) and first argmax (int32) with the head's
        log-softmax fused into its GEMM epilogue (no logits written); raw device pointers
        (0 = NULL).  Returns True when the fused epilogue ran."""
        fused = C.c_int32()
        _check(lib().prlab_gpu_forward_nll_device(self._h, C.c_void_p(d_ids), C.c_void_p(d_targets or None),
                                                  batch, seq, C.byref(_policy(policy)),
                                                  C.c_void_p(d_nll or None), C.c_void_p(d_argmax or None),
                                                  C.c_void_p(stream), C.byref(fused)))
        return bool(fused.value)

    def sync_status(self, stream: int = 0):
        _check(lib().prlab_gpu_sync_status(self._h, C.c_void_p(stream)))

    def host_copy_mode(self, batch, seq, policy="hybrid") -> int:
        """How forward() moves this key's logits to the host: 0 undecided, 1 fp16 rows
        widened on host threads, 2 fp32 copy (decided by timing on the first call)."""
        mode = C.c_int32()
        _check(lib().prlab_gpu_host_copy_mode(self._h, batch, seq, C.byref(_policy(policy)), C.byref(mode)))
        return int(mode.value)

    def kernel_count(self, batch, seq, policy="hybrid", out_dtype=None) -> int:
        """Kernels one forward_device launch issues (fp16 logits unless out_dtype given)."""
        n = C.c_int64()
        pol = _policy(policy)
        _check(lib().prlab_gpu_forward_kernel_count_ex(self._h, batch, seq, C.byref(pol),
                                                       OUT_F16 if out_dtype is None else out_dtype,
                                                       C.byref(n)))
        return int(n.value)

    def embedding_device(self, d_ids: int, batch: int, seq: int, path: int, d_out: int, stream: int = 0):
        """Parity probe: the hot path's embedding gather alone into d_out fp32 [B*S, h]
        (path 0 = embed_f32_kernel of the multi-kernel path, 1 = stage 0 of the batch-1
        persistent kernel)."""
        _check(lib().prlab_gpu_debug_embedding_device(self._h, C.c_void_p(d_ids), batch, seq, path,
                                                      C.c_void_p(d_out), C.c_void_p(stream)))


# ---------------------------------------------------------------------------
# per-operator API (include/prlab/kernels.hpp:30-70) -- host fp32 arrays
# ---------------------------------------------------------------------------
def matmul(a, b, cfg: KernelConfig):
    a, b = _arr(a), _arr(b)
    if a.ndim != 2 or b.ndim != 2:
        raise ValueError("matmul operands must be 2-D")
    if a.shape[1] != b.shape[0]:
        raise ValueError(f"matmul inner extents differ: {list(a.shape)} x {list(b.shape)}")
    out = np.empty((a.shape[0], b.shape[1]), np.float32)
    _check(lib().prlab_gpu_matmul(_f(a), _f(b), a.shape[0], a.shape[1], b.shape[1], cfg, _f(out)))
    return out


def attention_scores(q, k, scale: float, cfg: KernelConfig, capture: bool = False):
    q, k = _arr(q), _arr(k)
    if q.shape[1] != k.shape[1]:
        raise ValueError(f"attention head extents differ: {list(q.shape)} vs {list(k.shape)}")
    out = np.empty((q.shape[0], k.shape[0]), np.float32)
    tap = np.empty_like(out) if capture else None
    _check(lib().prlab_gpu_attention_scores(_f(q), _f(k), q.shape[0], k.shape[0], q.shape[1],
                                            scale, cfg, _f(out), _f(tap)))
    return (out, tap) if capture else out


def softmax_lastdim(x, cfg: KernelConfig):
    x = _arr(x)
    if x.ndim == 0 or x.shape[-1] == 0:
        raise ValueError(f"softmax needs a non-empty last axis, got shape {list(x.shape)}")
    out = np.empty_like(x)
    n = x.shape[-1]
    _check(lib().prlab_gpu_softmax(_f(x), x.size // n, n, cfg, _f(out)))
    return out


def layernorm_lastdim(x, gamma, beta, eps: float, cfg: KernelConfig):
    x, g, b = _arr(x), _arr(gamma), _arr(beta)
    if x.ndim == 0 or x.shape[-1] == 0:
        raise ValueError(f"layernorm needs a non-empty last axis, got shape {list(x.shape)}")
    n = x.shape[-1]
    if g.size != n or b.size != n:
        raise ValueError(f"layernorm scale/shift extents {g.size}/{b.size} do not match axis {n}")
    out = np.empty_like(x)
    _check(lib().prlab_gpu_layernorm(_f(x), x.size // n, n, _f(g), _f(b), eps, cfg, _f(out)))
    return out


def gelu(x, cfg: KernelConfig):
    x = _arr(x)
    out = np.empty_like(x)
    _check(lib().prlab_gpu_gelu(_f(x), x.size, cfg, _f(out)))
    return out


def tanh_op(x, cfg: KernelConfig):
    x = _arr(x)
    out = np.empty_like(x)
    _check(lib().prlab_gpu_tanh(_f(x), x.size, cfg, _f(out)))
    return out


def add(a, b, cfg: KernelConfig):
    a, b = _arr(a), _arr(b)
    if a.shape != b.shape:
        raise ValueError(f"add shapes differ: {list(a.shape)} vs {list(b.shape)}")
    out = np.empty_like(a)
    _check(lib().prlab_gpu_add(_f(a), _f(b), a.size, cfg, _f(out)))
    return out


def embed(tok_table, pos_table, ids, batch: int, seq: int, cfg: KernelConfig):
    tok, pos = _arr(tok_table), _arr(pos_table)
    ids = _arr(ids, np.int32)
    if tok.shape[1] != pos.shape[1]:
        raise ValueError(f"embedding widths differ: {list(tok.shape)} vs {list(pos.shape)}")
    if ids.size != batch * seq:
        raise ValueError(f"expected {batch * seq} token ids, got {ids.size}")
    out = np.empty((batch * seq, tok.shape[1]), np.float32)
    _check(lib().prlab_gpu_embed(_f(tok), tok.shape[0], _f(pos), pos.shape[0], tok.shape[1],
                                 ids.ctypes.data_as(_IP), batch, seq, cfg, _f(out)))
    return out


# ---------------------------------------------------------------------------
# device building blocks (torch tensors or raw pointers)
# ---------------------------------------------------------------------------
def _ptr(t) -> int:
    return t if isinstance(t, int) else (t.data_ptr() if t is not None else 0)


def linear_f16_device(A, Wt, bias, out, M, N, K, ldo, epi, stream=0):
    _check(lib().prlab_gpu_linear_f16_device(C.c_void_p(_ptr(A)), C.c_void_p(_ptr(Wt)),
                                             C.c_void_p(_ptr(bias)), C.c_void_p(_ptr(out)), M, N,
                                             K, ldo, epi, C.c_void_p(stream)))


def linear_f16_device_ex(A, Wt, bias, out, M, N, K, ldo, epi, bn=0, splits=0, lean=0, stream=0):
    _check(lib().prlab_gpu_linear_f16_device_ex(C.c_void_p(_ptr(A)), C.c_void_p(_ptr(Wt)),
                                                C.c_void_p(_ptr(bias)), C.c_void_p(_ptr(out)), M,
                                                N, K, ldo, epi, bn, splits, lean,
                                                C.c_void_p(stream)))


def linear_f32_device(A, Wt, bias, out, M, N, K, epi=0, resid=None, stream=0):
    """fp32-policy linear on the tensor cores (3xTF32): out = epi(A . Wt^T)."""
    _check(lib().prlab_gpu_linear_f32_device(C.c_void_p(_ptr(A)), C.c_void_p(_ptr(Wt)), C.c_void_p(_ptr(bias)),
                                             C.c_void_p(_ptr(out)), M, N, K, epi, C.c_void_p(_ptr(resid)),
                                             C.c_void_p(stream)))


def attention_f16_device(qkv, ctx, B, S, H, hd, causal, stream=0):
    _check(lib().prlab_gpu_attention_f16_device(C.c_void_p(_ptr(qkv)), C.c_void_p(_ptr(ctx)), B,
                                                S, H, hd, int(causal), C.c_void_p(stream)))


def flop_count(cfg: ModelConfig, batch: int, seq: int) -> dict:
    """flop_count (src/model.cpp:528-543)."""
    b, s, h, f, L = batch, seq, cfg.hidden, cfg.ffn, cfg.num_layers
    lin = L * 2 * (4 * h * h + 2 * h * f) * s * b
    att = L * 4 * s * s * h * b
    out = 2 * s * h * cfg.vocab * b if L > 0 else 0
    return {"linear": lin, "attention": att, "output_projection": out, "total": lin + att + out}


def header_symbols(path: str = HEADER_PATH) -> Sequence[str]:
    """Every function declared in include/prlab_gpu.h."""
    import re
    src = open(path).read()
    return sorted(set(re.findall(r"\b(prlab_gpu_[a-z0-9_]+)\s*\(", src)))


def row_nll_device(logits, targets, nll, argmax=None, rows=None, n=None, ld=None, stream=0):
    """Per-row next-token NLL / argmax over device logits (torch tensors on cuda)."""
    import torch  # noqa: F401  (device tensors)
    dtype = OUT_F16 if str(logits.dtype) == "torch.float16" else OUT_F32
    rows = logits.shape[0] if rows is None else rows
    ld = logits.shape[1] if ld is None else ld
    n = ld if n is None else n
    _check(lib().prlab_gpu_row_nll_device(C.c_void_p(logits.data_ptr()), dtype, rows, n, ld,
                                          C.c_void_p(targets.data_ptr()) if targets is not None else None,
                                          C.c_void_p(nll.data_ptr()) if nll is not None else None,
                                          C.c_void_p(argmax.data_ptr()) if argmax is not None else None,
                                          C.c_void_p(stream)))


def compare_logits_device(base, cand, rows, n, stream=0) -> dict:
    """compare_logits (src/fidelity.cpp:11-37) of two device logit tensors [rows, ld]."""
    def dt(t):
        return OUT_F16 if str(t.dtype) == "torch.float16" else OUT_F32
    r = LogitComparison()
    _check(lib().prlab_gpu_compare_logits_device(C.c_void_p(base.data_ptr()), dt(base), base.shape[1],
                                                 C.c_void_p(cand.data_ptr()), dt(cand), cand.shape[1],
                                                 rows, n, C.c_void_p(stream), C.byref(r)))
    return r.as_dict()
