"""Test helpers shared by the suites (oracle handles, cached build_model params)."""
import functools
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


@functools.lru_cache(maxsize=None)
def oracle():
    from oracle.oracle import Oracle
    return Oracle()


@functools.lru_cache(maxsize=None)
def reference():
    from oracle.oracle import Reference
    return Reference()


def have_reference_lib() -> bool:
    from oracle.oracle import REF_SO
    return os.path.exists(REF_SO)


_PARAM_CACHE = {}


def model_params(cfg):
    """build_model() output for cfg (oracle restatement; bit-identical to the reference)."""
    key = cfg
    if key not in _PARAM_CACHE:
        _PARAM_CACHE[key] = oracle().build_model(cfg)
    return _PARAM_CACHE[key]


def gpu_available() -> bool:
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False
